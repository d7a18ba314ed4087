// sweep_internal.h — data shared between the host setup (sweep_host.cpp) and
// the sm_100a kernels (sweep_kernels.cu).  Not part of the public ABI.
#pragma once
#include <cstddef>
#include <cstdint>

namespace sweepk {

// compile-time kernel options (template parameter OPT)
constexpr int OPT_SIGMA = 1;   // append sum_g sigma_g phi_g, sum_g sigma_g J_g
constexpr int OPT_FIXUP = 2;   // zero-and-scale negative flux fixup inside the sweep (NEXT-2)
constexpr int OPT_HALF = 4;    // 1-D: also the untraced P_xx row of each half-range stream (NEXT-3);
                               // 2-D takes this at run time (Sweep2DParams::half)

// Per (folded) direction, in sweep coordinates (every direction is mapped to
// the (+,+) quadrant by mirroring the element order and the nodes).
struct DirConst {
    double cx, cy;     // |Omega_x|/hx, |Omega_y|/hy   (1-D: cx = |mu|/h, cy = 0)
    double mom[6];     // moment weights with the SIGNED direction:
                       //  2-D: w, w Ox, w Oy, w(Ox^2-1/3), w Ox Oy, w(Oy^2-1/3)
                       //  1-D: w, w mu, w(mu^2-1/3), 0, 0, 0
    double bw[4];      // beta weights per physical face x-,x+,y-,y+: w(|Omega.n| - alpha_n)
    double jw[4];      // J+ weights per physical face: w max(Omega.n, 0)
    double pw[2];      // untraced second-moment weights w Omega_x^2, w Omega_y^2 (half-range P+, NEXT-3)
};

// One work stream = (quadrant, group block, direction set): the lanes of one CTA.
struct StreamDesc {
    int quadrant;      // 2-D: bit0 = (Omega_x < 0), bit1 = (Omega_y < 0); 1-D: bit0 = (mu < 0)
    int g0, ng;        // local groups [g0, g0+ng)
    int d0, nd;        // directions [d0, d0+nd) of the quadrant-sorted table
};

// Modal constants of the p = 2 reference operator A^ = V Lambda W (W = V^-1),
// A^ = [[3,4,-1],[-1,0,1],[1,-4,3]] (derived in DESIGN.md §4 from the lumped
// weak form).  Mode 0 real (lambda0), mode 1 = mu + i nu, mode 2 = conj.
struct ModalConsts {
    double lam0, mu, nu;
    double W0[3];          // real row of W
    double W1re[3], W1im[3];
    double V0[3];          // real column of V (V[a][0])
    double V1re[3], V1im[3];   // V[a][1]  (V[2][0] = V[2][1] = 1: scaled at the outflow node)
    double V1re2[3], V1im2n[3];  // 2 Re V[a][1], -2 Im V[a][1] (separable modal -> nodal map)
    // real 9x9 maps between nodal (k = a + 3b, sweep coordinates) and the 9 modal
    // reals m = [u00, u01r, u01i, u10r, u10i, u11r, u11i, u12r, u12i]
    double fwd[9][9];      // modal = fwd * nodal   (W (x) W)
    double bck[9][9];      // nodal = bck * modal   (V (x) V)
};

struct Sweep2DParams {
    int nx, ny, G;                 // G = groups on this rank
    int nx_pad;                    // n_chunks * C (trace ring row length)
    int n_streams, n_strips, n_chunks, n_tasks;
    int gb;                        // lanes per direction (power of 2)
    int kpl;                       // groups per lane
    int dset;                      // directions per CTA
    int nbnode;
    int bulk_ok;                   // q / sigma rows are 16-byte aligned (G even): 1-D bulk copies
    int half;                      // SWEEP_HALF_RANGE: write the P_xx, P_yy rows at hr_off of the slab
    size_t hr_off;
    double inv_c_dt;
    const double* sigma;           // [N_el][G]
    const double* q;               // [N_el][n][G]
    const double* inflow;          // [N_bnode][G]
    const DirConst* dirs;          // quadrant-sorted
    const StreamDesc* streams;
    int* progress;                 // [n_streams][n_strips] chunks completed (per-chunk flag protocol)
    int* epoch;                    // LL ring protocol: launches completed on this handle (device counter,
                                   // read at kernel start, bumped by the last CTA: graph replays too)
    int* task_counter;
    double* ytr;                   // [n_streams][2][nx][K][NT][NL]
    size_t ring_len;               // doubles in ytr
    int* ytag;                     // debug builds: [n_streams][2][nx_pad] strip that wrote the ring column
    double* slabs;                 // [n_streams][out_size]
    size_t out_size;
    size_t nodes;                  // N_el * n
    int* err;
    const int* in_ready;           // sweep_run_host: per band of in_band_rows physical rows, the generation
    int in_gen, in_band_rows;      // whose inputs have landed (nullptr: inputs resident at launch)
};

struct Sweep1DParams {
    int nx, G, n_streams, gb, nseg, seglen;
    size_t hr_off;                 // OPT_HALF: slab offset of the P_xx row
    double inv_c_dt;
    const double* sigma;
    const double* q;
    const double* inflow;
    const DirConst* dirs;
    const StreamDesc* streams;
    double* slabs;
    size_t out_size;
    size_t nodes;
    int* err;
};

// 1-D warp-scan sweep (k_1d.cu): one warp per chain (direction, group), one lane per segment
struct Sweep1DScanParams {
    int nx, G, seglen;             // seglen = ceil(nx / 32) elements per lane
    size_t nodes, out_size, sum_size, hr_off;
    double inv_c_dt;
    const double* sigma;
    const double* q;
    const double* inflow;
    const DirConst* dirs;
    const StreamDesc* streams;     // per CTA: quadrant = half-range, d0 = its first direction,
                                   // g0 / ng = first chain / chain count (chain j: d0 + j / G, group j % G)
    double* slabs;                 // [grid][out_size]
    int* err;
    int* done_counter;             // fused_out: CTAs finished (the last one resets it)
    double* fused_out;             // non-null: the last CTA sums the slabs' [0, sum_size) here
    int single;                    // one CTA, both half-ranges (streams[0], streams[1]); fields
    int nw0;                       // accumulated in shared memory, written to fused_out
};
int scan1d_smem_bytes(int p, int opt, int warps, size_t single_nodes);
int raise_smem_cap(const void* f);  // dynamic smem cap of f := opt-in max - static smem
int launch_sweep1d_scan(int p, int opt, const Sweep1DScanParams& prm, int grid, int block, size_t smem, void* stream);
int upload_modal_1d(const ModalConsts& mc);

// launchers (k_common.cu); return cudaError_t as int.  opt = OPT_* bits.
int upload_modal(const ModalConsts& mc);
int launch_sweep2d(int p, int log2lg, int k, int opt, const Sweep2DParams& prm, int grid, int block, size_t smem,
                   void* stream);
int launch_sweep1d(int p, int log2gb, int opt, const Sweep1DParams& prm, int grid, int block, size_t smem, void* stream);
// grid caps (SMs x resident blocks per SM) of the grid-stride reduction kernels, per handle
struct ReduceCaps {
    int finalize, finalize_modal, halfrange;
};
int reduce_caps(int n_sm, ReduceCaps* caps);
int launch_finalize(const double* slabs, int n_slabs, size_t stride, size_t n, double* out, int* err, int cap,
                    void* stream);
int launch_halfrange(const double* slabs, int n_slabs, size_t stride, const StreamDesc* streams, size_t nodes,
                     size_t hr_off, int dim, int modal, double* out, int cap, void* stream);
// 2-D p = 2: back transform + fixed-order sum of the modal node-field rows [row0, row0 + nrows*nel*9)
int launch_finalize_modal(const double* slabs, int n_slabs, size_t stride, const StreamDesc* streams, size_t row0,
                          int nrows, size_t nel, double* out, int* err, int cap, void* stream);
int sweep2d_smem_bytes(int p, int k, int gbk, int dset, int opt);
int sweep2d_occupancy(int p, int log2lg, int k, int opt, int block, size_t smem, int* blocks_per_sm);
int sweep2d_rows_per_strip(int p, int k);
int sweep2d_cols_per_chunk(int p, int k, int opt);
int sweep2d_ring_record(int p, int k, int log2lg, int opt);  // trace-ring doubles per lane and column
const char* cuda_err_string(int e);
int fp64_probe(int device, double* tflops);
int launch_floor(int device, int reps, double* us);
int selfcheck_solves(int device, int p, int n, unsigned long long seed, double* max_rel);
int debug_build();  // 1 in -DSWEEP_DEBUG builds (bounds checks + trace-ring tags)

// unaccelerated TRT iteration (k_trt.cu)
int trt_blocks(int n_sm);
int launch_trt_emission(const double* T, const double* sigma, const double* Iprev, const double* nu, int G, int n,
                        size_t nodes, double inv_dt, double* q, int n_sm, void* stream);
int launch_trt_e0(const double* Iprev, int G, size_t nodes, double* E, int n_sm, void* stream);
int launch_trt_update(const double* Tk, double* T, const double* sphi, const double* phi, double* E,
                      const double* sigma, const double* nu, int G, int n, size_t nodes, double cv_dt, double* partial,
                      double* norms, int* err, int n_sm, void* stream);

// per translation unit (k2d_*.cu): kernel pointer for (log2lg, k, opt), or nullptr;
// and the upload of that unit's copy of the modal constants
const void* pick2d_p1(int log2lg, int k);
const void* pick2d_p2(int log2lg, int k);
const void* pick2d_opt_p1(int log2lg, int k, int opt);
const void* pick2d_opt_p2(int log2lg, int k, int opt);
int upload_modal_p1(const ModalConsts& mc);
int upload_modal_p2(const ModalConsts& mc);
int upload_modal_opt_p1(const ModalConsts& mc);
int upload_modal_opt_p2(const ModalConsts& mc);

}  // namespace sweepk
