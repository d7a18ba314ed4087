// sweep_host.cpp — the C ABI (include/sweep.h): validation, setup tables (a1),
// schedule (a2), device workspace, launches, NCCL all-reduce of the gray output.
//
// PAPER.md references: alpha (eq:alpha, :173-176), closures T and beta
// (:163-171), moments (:156-162), sigma~ (:239), weak form (:332-336).
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <new>
#include <string>
#include <utility>
#include <vector>

#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3 (ranges are no-ops without a profiler attached)

#include "../../include/sweep.h"
#include "sweep_internal.h"

using sweepk::DirConst;
using sweepk::ModalConsts;
using sweepk::StreamDesc;
using cplx = std::complex<double>;

// ---------------------------------------------------------------- NCCL (dlopen)
namespace {
typedef struct ncclComm* ncclComm_t;
typedef struct {
    char internal[128];
} ncclUniqueId_t;
typedef int (*pf_getUniqueId)(ncclUniqueId_t*);
typedef int (*pf_commInitRank)(ncclComm_t*, int, ncclUniqueId_t, int);
typedef int (*pf_allReduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t);
typedef int (*pf_commDestroy)(ncclComm_t);
typedef const char* (*pf_getErrorString)(int);

struct NcclApi {
    void* lib = nullptr;
    pf_getUniqueId getUniqueId = nullptr;
    pf_commInitRank commInitRank = nullptr;
    pf_allReduce allReduce = nullptr;
    pf_commDestroy commDestroy = nullptr;
    pf_getErrorString getErrorString = nullptr;
    bool load(std::string& err) {
        if (lib) return true;
        // the copy torch already loaded (same soname) is reused by the dynamic loader
        const char* names[] = {"libnccl.so.2", "libnccl.so"};
        for (const char* n : names) {
            lib = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
            if (lib) break;
        }
        if (!lib) {
            err = std::string("dlopen libnccl.so.2 failed: ") + dlerror();
            return false;
        }
        getUniqueId = (pf_getUniqueId)dlsym(lib, "ncclGetUniqueId");
        commInitRank = (pf_commInitRank)dlsym(lib, "ncclCommInitRank");
        allReduce = (pf_allReduce)dlsym(lib, "ncclAllReduce");
        commDestroy = (pf_commDestroy)dlsym(lib, "ncclCommDestroy");
        getErrorString = (pf_getErrorString)dlsym(lib, "ncclGetErrorString");
        if (!getUniqueId || !commInitRank || !allReduce || !commDestroy) {
            err = "libnccl: missing symbols";
            return false;
        }
        return true;
    }
};
NcclApi g_nccl;
thread_local std::string g_setup_error;
constexpr int kNcclFloat64 = 8, kNcclSum = 0;

// NVTX range for the lifetime of a scope (setup, run, all-reduce, closures, TRT iterations)
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

struct DeviceGuard {
    int prev = -1;
    bool ok = false;
    explicit DeviceGuard(int dev) {
        if (cudaGetDevice(&prev) == cudaSuccess && cudaSetDevice(dev) == cudaSuccess) ok = true;
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};
}  // namespace

// ---------------------------------------------------------------- handle
struct sweep_handle {
    int dim, nx, ny, p, n, np1, nbnode, G, device, nranks, rank;
    double lx, ly, hx, hy;
    unsigned flags;
    size_t nodes, out_size, off[8];
    size_t sum_size = 0;  // leading part of the output summed over slabs (all but the half-range rows)
    int opt = 0;  // sweepk::OPT_* bits from the flags
    int n_dir_in, n_dir_eff;
    // schedule
    int log2gb, gb, kpl, block, dset, n_streams, n_strips, n_chunks, n_tasks, grid, nseg, seglen;
    size_t smem;
    int n_sm = 0;                 // SMs of the handle's device (queried at setup)
    bool scan1d = false;          // 1-D: warp-scan kernel (k_1d.cu); the fixup keeps the sequential kernel
    bool fused1d = false;         // 1-D scan: the last CTA sums the slabs (no finalize launch)
    bool single1d = false;        // 1-D scan, tiny problem: one CTA for both half-ranges
    int single_nw0 = 0;
    sweepk::ReduceCaps caps{};    // grid caps of the reduction kernels
    // device workspace
    DirConst* d_dirs = nullptr;
    StreamDesc* d_streams = nullptr;
    int* d_progress = nullptr;  // [n_streams*n_strips] + task counter + err flag
    double* d_ytr = nullptr;
    size_t ring_len = 0;
    int* d_ytag = nullptr;  // debug builds: trace-ring tags
    double* d_slabs = nullptr;
    double* d_out = nullptr;
    int* d_err = nullptr;
    int* d_counter = nullptr;
    size_t progress_ints = 0;
    // host-API staging; 2-D: the copy stream, its order / join events and the per-band
    // input-ready flags of the overlapped copy (sweep_run_host)
    double *d_in_sigma = nullptr, *d_in_q = nullptr, *d_in_inflow = nullptr;
    cudaStream_t cp_stream = nullptr;
    cudaEvent_t cp_ev[2] = {nullptr, nullptr};
    int* d_in_ready = nullptr;
    int in_gen = 0;
    // unaccelerated TRT iteration workspace (trt_step)
    double *d_trt_q = nullptr, *d_trt_nu = nullptr, *d_trt_part = nullptr, *d_trt_norm = nullptr;
    double* d_trt_E = nullptr;  // E^l of the outer iteration (eq:relative_tol, u = [T, E])
    int trt_nu_len = 0;
    ncclComm_t comm = nullptr;
    long long launches = 0;
    // timing ring
    static constexpr int kRing = 1024;
    bool timing = false;
    std::vector<cudaEvent_t> ev;  // kRing * 4
    long long runs_recorded = 0;
    std::string err;
};

static int fail(sweep_handle* h, int code, const std::string& msg) {
    if (h)
        h->err = msg;
    else
        g_setup_error = msg;
    return code;
}

static int cuda_fail(sweep_handle* h, cudaError_t e, const char* where) {
    return fail(h, SWEEP_E_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

// ---------------------------------------------------------------- modal constants (p = 2)
// A^ = [[3,4,-1],[-1,0,1],[1,-4,3]] is the scaled lumped element operator of
// one axis for Omega > 0.  A^ = V diag(lam0, lam1, conj lam1) W.
static bool build_modal(ModalConsts& mc, std::string& err) {
    const double A[3][3] = {{3, 4, -1}, {-1, 0, 1}, {1, -4, 3}};
    // characteristic polynomial l^3 - tr l^2 + c1 l - det
    const double tr = A[0][0] + A[1][1] + A[2][2];
    const double c1 = (A[0][0] * A[1][1] - A[0][1] * A[1][0]) + (A[0][0] * A[2][2] - A[0][2] * A[2][0]) +
                      (A[1][1] * A[2][2] - A[1][2] * A[2][1]);
    const double det = A[0][0] * (A[1][1] * A[2][2] - A[1][2] * A[2][1]) -
                       A[0][1] * (A[1][0] * A[2][2] - A[1][2] * A[2][0]) +
                       A[0][2] * (A[1][0] * A[2][1] - A[1][1] * A[2][0]);
    double l = tr;  // Newton from above the real root
    for (int it = 0; it < 200; ++it) {
        const double f = ((l - tr) * l + c1) * l - det;
        const double df = (3 * l - 2 * tr) * l + c1;
        const double dl = f / df;
        l -= dl;
        if (std::fabs(dl) < 1e-16 * std::fabs(l)) break;
    }
    const double lam0 = l;
    const double mu = 0.5 * (tr - lam0);
    const double nu2 = det / lam0 - mu * mu;
    if (!(nu2 > 0)) {
        err = "modal: expected a complex eigenpair";
        return false;
    }
    const double nu = std::sqrt(nu2);
    const cplx lam[3] = {cplx(lam0, 0), cplx(mu, nu), cplx(mu, -nu)};
    cplx V[3][3];
    for (int k = 0; k < 2; ++k) {
        cplx M[3][3];
        for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b) M[a][b] = cplx(A[a][b], 0) - (a == b ? lam[k] : cplx(0, 0));
        // null vector = cross product of the two rows with the largest cross product
        cplx best[3];
        double bn = -1;
        const int pr[3][2] = {{0, 1}, {0, 2}, {1, 2}};
        for (auto& pq : pr) {
            const cplx* r0 = M[pq[0]];
            const cplx* r1 = M[pq[1]];
            cplx v[3] = {r0[1] * r1[2] - r0[2] * r1[1], r0[2] * r1[0] - r0[0] * r1[2], r0[0] * r1[1] - r0[1] * r1[0]};
            double nrm = std::sqrt(std::norm(v[0]) + std::norm(v[1]) + std::norm(v[2]));
            if (nrm > bn) {
                bn = nrm;
                for (int a = 0; a < 3; ++a) best[a] = v[a] / nrm;
            }
        }
        for (int a = 0; a < 3; ++a) V[a][k] = best[a];
    }
    // real eigenvector: remove any global phase
    {
        int im = 0;
        for (int a = 1; a < 3; ++a)
            if (std::abs(V[a][0]) > std::abs(V[im][0])) im = a;
        const cplx ph = std::abs(V[im][0]) / V[im][0];
        for (int a = 0; a < 3; ++a) V[a][0] = cplx((V[a][0] * ph).real(), 0.0);
    }
    // scale each eigenvector to 1 at the outflow node (a = 2): the outflow traces of a
    // modal solution are then plain sums of modal coefficients (traces_p2)
    for (int k = 0; k < 2; ++k) {
        const cplx piv = V[2][k];
        if (!(std::abs(piv) > 1e-3)) {
            err = "modal: eigenvector vanishes at the outflow node";
            return false;
        }
        for (int a = 0; a < 2; ++a) V[a][k] /= piv;
        V[2][k] = cplx(1.0, 0.0);
    }
    for (int a = 0; a < 3; ++a) V[a][2] = std::conj(V[a][1]);
    // W = V^-1 (adjugate)
    cplx detV = V[0][0] * (V[1][1] * V[2][2] - V[1][2] * V[2][1]) - V[0][1] * (V[1][0] * V[2][2] - V[1][2] * V[2][0]) +
                V[0][2] * (V[1][0] * V[2][1] - V[1][1] * V[2][0]);
    cplx W[3][3];
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) {
            const int r0 = (b + 1) % 3, r1 = (b + 2) % 3, c0 = (a + 1) % 3, c1i = (a + 2) % 3;
            W[a][b] = (V[r0][c0] * V[r1][c1i] - V[r0][c1i] * V[r1][c0]) / detV;
        }
    // self-check: V Lambda W = A and V W = I
    double res = 0;
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) {
            cplx s = 0, id = 0;
            for (int k = 0; k < 3; ++k) {
                s += V[a][k] * lam[k] * W[k][b];
                id += V[a][k] * W[k][b];
            }
            res = std::max(res, std::abs(s - A[a][b]));
            res = std::max(res, std::abs(id - (a == b ? 1.0 : 0.0)));
        }
    if (res > 1e-13) {
        char buf[96];
        snprintf(buf, sizeof buf, "modal: eigen-decomposition residual %.3e", res);
        err = buf;
        return false;
    }
    mc.lam0 = lam0;
    mc.mu = mu;
    mc.nu = nu;
    for (int a = 0; a < 3; ++a) {
        mc.W0[a] = W[0][a].real();
        mc.W1re[a] = W[1][a].real();
        mc.W1im[a] = W[1][a].imag();
        mc.V0[a] = V[a][0].real();
        mc.V1re[a] = V[a][1].real();
        mc.V1im[a] = V[a][1].imag();
    }
    for (int a = 0; a < 3; ++a) {
        mc.V1re2[a] = 2.0 * mc.V1re[a];
        mc.V1im2n[a] = -2.0 * mc.V1im[a];
    }
    // 9x9 real maps; modal reals m = [u00, u01r, u01i, u10r, u10i, u11r, u11i, u12r, u12i]
    const int pairs[5][2] = {{0, 0}, {0, 1}, {1, 0}, {1, 1}, {1, 2}};
    for (int k = 0; k < 9; ++k) {
        const int a = k % 3, b = k / 3;
        for (int pi = 0; pi < 5; ++pi) {
            const int al = pairs[pi][0], be = pairs[pi][1];
            const cplx f = W[al][a] * W[be][b];
            const cplx g = V[a][al] * V[b][be];
            if (pi == 0) {
                mc.fwd[0][k] = f.real();
                mc.bck[k][0] = g.real();
            } else {
                mc.fwd[2 * pi - 1][k] = f.real();
                mc.fwd[2 * pi][k] = f.imag();
                mc.bck[k][2 * pi - 1] = 2.0 * g.real();
                mc.bck[k][2 * pi] = -2.0 * g.imag();
            }
        }
    }
    double r2 = 0;
    for (int i = 0; i < 9; ++i)
        for (int j = 0; j < 9; ++j) {
            double s = 0;
            for (int k = 0; k < 9; ++k) s += mc.bck[i][k] * mc.fwd[k][j];
            r2 = std::max(r2, std::fabs(s - (i == j ? 1.0 : 0.0)));
        }
    if (r2 > 1e-13) {
        err = "modal: bck*fwd != I";
        return false;
    }
    return true;
}

static int ilog2_ceil(int v) {
    int l = 0;
    while ((1 << l) < v) ++l;
    return l;
}

// ---------------------------------------------------------------- ABI
extern "C" int sweep_nccl_unique_id(void* out128) {
    if (!out128) return SWEEP_E_ARG;
    std::string e;
    if (!g_nccl.load(e)) return fail(nullptr, SWEEP_E_NCCL, e);
    ncclUniqueId_t id;
    int r = g_nccl.getUniqueId(&id);
    if (r != 0) return fail(nullptr, SWEEP_E_NCCL, "ncclGetUniqueId failed");
    memcpy(out128, &id, 128);
    return SWEEP_OK;
}

extern "C" int sweep_setup(const sweep_desc* desc, sweep_handle** out) {
    NvtxRange nv("sweep_setup");
    if (out) *out = nullptr;
    if (!desc || !out || !desc->omega || !desc->w) return fail(nullptr, SWEEP_E_ARG, "null pointer");
    const sweep_desc& D = *desc;
    if (D.dim != 1 && D.dim != 2) return fail(nullptr, SWEEP_E_ARG, "dim must be 1 or 2");
    if (D.p != 1 && D.p != 2) return fail(nullptr, SWEEP_E_ARG, "p must be 1 or 2");
    if (D.nx <= 0 || (D.dim == 2 && D.ny <= 0) || D.n_dir <= 0 || D.n_group_local <= 0)
        return fail(nullptr, SWEEP_E_ARG, "sizes must be positive");
    if (!(D.lx > 0) || (D.dim == 2 && !(D.ly > 0))) return fail(nullptr, SWEEP_E_ARG, "lx, ly must be > 0");
    if (D.nranks < 1 || D.rank < 0 || D.rank >= D.nranks) return fail(nullptr, SWEEP_E_ARG, "bad nranks/rank");
    if (D.nranks > 1 && !D.nccl_id) return fail(nullptr, SWEEP_E_ARG, "nranks > 1 needs nccl_id");
    if ((long long)D.nx * (D.dim == 2 ? D.ny : 1) > (1LL << 30)) return fail(nullptr, SWEEP_E_ARG, "mesh too large");

    // quadrature validation
    double sw = 0;
    for (int d = 0; d < D.n_dir; ++d) {
        const double wd = D.w[d];
        if (!(wd > 0) || !std::isfinite(wd)) return fail(nullptr, SWEEP_E_QUAD, "weights must be positive");
        sw += wd;
        const double* o = D.omega + 3 * d;
        if (!std::isfinite(o[0]) || !std::isfinite(o[1]) || !std::isfinite(o[2]))
            return fail(nullptr, SWEEP_E_QUAD, "non-finite direction");
        if (D.dim == 2) {
            if (std::fabs(std::sqrt(o[0] * o[0] + o[1] * o[1] + o[2] * o[2]) - 1.0) > 1e-13)
                return fail(nullptr, SWEEP_E_QUAD, "directions must be unit vectors");
        } else if (std::fabs(o[0]) > 1.0) {
            return fail(nullptr, SWEEP_E_QUAD, "|mu| must be <= 1");
        }
    }
    if (std::fabs(sw - 1.0) > 1e-13) return fail(nullptr, SWEEP_E_QUAD, "weights must sum to 1");

    sweep_handle* h = new (std::nothrow) sweep_handle();
    if (!h) return fail(nullptr, SWEEP_E_ARG, "out of host memory");
    h->dim = D.dim;
    h->nx = D.nx;
    h->ny = (D.dim == 2) ? D.ny : 1;
    h->p = D.p;
    h->np1 = D.p + 1;
    h->n = (D.dim == 2) ? h->np1 * h->np1 : h->np1;
    h->nbnode = (D.dim == 1) ? 2 : 2 * (D.nx + D.ny) * h->np1;
    h->G = D.n_group_local;
    h->device = D.device;
    h->nranks = D.nranks;
    h->rank = D.rank;
    h->lx = D.lx;
    h->ly = (D.dim == 2) ? D.ly : 1.0;
    h->hx = h->lx / h->nx;
    h->hy = h->ly / h->ny;
    h->flags = D.flags;
    h->nodes = (size_t)h->nx * h->ny * h->n;
    const int nT = (D.dim == 1) ? 1 : 3;
    h->off[0] = 0;
    h->off[1] = h->nodes;
    h->off[2] = h->nodes * (1 + D.dim);
    h->off[3] = h->nodes * (1 + D.dim + nT);
    h->off[4] = h->off[3] + h->nbnode;
    h->out_size = h->off[4] + h->nbnode;
    h->opt = ((D.flags & SWEEP_SIGMA_MOMENTS) ? sweepk::OPT_SIGMA : 0) | ((D.flags & SWEEP_FIXUP) ? sweepk::OPT_FIXUP : 0);
    if (h->opt & sweepk::OPT_SIGMA) {
        h->off[5] = h->out_size;                 // sigma phi
        h->off[6] = h->off[5] + h->nodes;        // sigma J
        h->out_size = h->off[6] + h->nodes * D.dim;
    } else {
        h->off[5] = h->off[6] = h->out_size;
    }
    h->sum_size = h->out_size;
    h->off[7] = h->out_size;  // half-range rows (SWEEP_HALF_RANGE): 10 (dim 2) or 2 (dim 1) per node
    if (D.flags & SWEEP_HALF_RANGE) h->out_size += h->nodes * (D.dim == 2 ? 10 : 2);
    h->n_dir_in = D.n_dir;

    // alpha per outward normal (eq:alpha): sum w |Omega.n| / sum w
    double ax = 0, ay = 0;
    for (int d = 0; d < D.n_dir; ++d) {
        ax += D.w[d] * std::fabs(D.omega[3 * d]);
        ay += D.w[d] * ((D.dim == 2) ? std::fabs(D.omega[3 * d + 1]) : 0.0);
    }
    const double alpha[4] = {ax / sw, ax / sw, ay / sw, ay / sw};

    // fold directions with identical (Omega_x, Omega_y) (reading R20)
    struct Dir {
        double ox, oy, w;
    };
    std::vector<Dir> dirs;
    if (D.dim == 2 && (D.flags & SWEEP_FOLD_Z)) {
        std::map<std::pair<double, double>, size_t> seen;
        for (int d = 0; d < D.n_dir; ++d) {
            const double ox = D.omega[3 * d], oy = D.omega[3 * d + 1];
            auto key = std::make_pair(ox, oy);
            auto it = seen.find(key);
            if (it == seen.end()) {
                seen[key] = dirs.size();
                dirs.push_back({ox, oy, D.w[d]});
            } else {
                dirs[it->second].w += D.w[d];
            }
        }
    } else {
        for (int d = 0; d < D.n_dir; ++d) dirs.push_back({D.omega[3 * d], D.dim == 2 ? D.omega[3 * d + 1] : 0.0, D.w[d]});
    }
    h->n_dir_eff = (int)dirs.size();

    // per-direction constants, sorted by quadrant
    const int nquad = (D.dim == 2) ? 4 : 2;
    std::vector<std::vector<DirConst>> byq(nquad);
    for (const Dir& d : dirs) {
        DirConst c;
        memset(&c, 0, sizeof c);
        const int q = (d.ox < 0 ? 1 : 0) + ((D.dim == 2 && d.oy < 0) ? 2 : 0);
        c.cx = std::fabs(d.ox) / h->hx;
        c.cy = (D.dim == 2) ? std::fabs(d.oy) / h->hy : 0.0;
        if (D.dim == 2) {
            c.mom[0] = d.w;
            c.mom[1] = d.w * d.ox;
            c.mom[2] = d.w * d.oy;
            c.mom[3] = d.w * (d.ox * d.ox - 1.0 / 3.0);
            c.mom[4] = d.w * (d.ox * d.oy);
            c.mom[5] = d.w * (d.oy * d.oy - 1.0 / 3.0);
        } else {
            c.mom[0] = d.w;
            c.mom[1] = d.w * d.ox;
            c.mom[2] = d.w * (d.ox * d.ox - 1.0 / 3.0);
        }
        const double on[4] = {-d.ox, d.ox, -d.oy, d.oy};
        for (int f = 0; f < 4; ++f) {
            c.bw[f] = d.w * (std::fabs(on[f]) - alpha[f]);
            c.jw[f] = d.w * std::max(on[f], 0.0);
        }
        c.pw[0] = d.w * (d.ox * d.ox);
        c.pw[1] = d.w * (d.oy * d.oy);
        byq[q].push_back(c);
    }
    std::vector<DirConst> table;
    std::vector<int> qstart(nquad + 1, 0);
    for (int q = 0; q < nquad; ++q) {
        qstart[q] = (int)table.size();
        table.insert(table.end(), byq[q].begin(), byq[q].end());
    }
    qstart[nquad] = (int)table.size();

    // lane layout: GB lanes per direction (consecutive groups), 32/GB directions per
    // warp; in 2-D each lane carries kpl groups, so a stream covers GB*kpl groups
    const int gbw = std::min(32, 1 << ilog2_ceil(h->G));
    // 2-D p=2 with many groups: 4 groups per lane over 16 lanes (one CTA holds a
    // whole quadrant's directions); otherwise 1 group per lane over up to 32 lanes
    // (measured per-rank workloads of the group-sharded C5: 64 groups 4x16,
    // 32 groups 2x16, 16 groups 2x8; fewer: one group per lane.  With options only the
    // 4x16 and one-group layouts are instantiated.)
    const bool opt_layouts_only = h->opt != 0;
    if (D.dim == 2 && D.p == 2 && h->G >= 64) {
        h->kpl = 4;
        h->gb = 16;
        h->log2gb = 4;
    } else if (D.dim == 2 && D.p == 2 && h->G >= 16 && !opt_layouts_only) {
        h->kpl = 2;
        h->gb = (h->G >= 32) ? 16 : 8;
        h->log2gb = (h->G >= 32) ? 4 : 3;
    } else {
        h->kpl = 1;
        h->gb = gbw;
        h->log2gb = ilog2_ceil(gbw);
    }
#ifdef SWEEP_EXPERIMENTS
    // experiment builds only (scripts/build_variants.py): SWEEP_CFG="K,LG" with K in {1,2,4},
    // LG a power of two <= 32 overrides the 2-D lane layout
    if (D.dim == 2) {
        if (const char* ev = getenv("SWEEP_CFG")) {
            int k = 0, lg = 0;
            if (sscanf(ev, "%d,%d", &k, &lg) == 2 && (k == 1 || k == 2 || k == 4) && lg >= 1 && lg <= 32 &&
                (lg & (lg - 1)) == 0) {
                h->kpl = k;
                h->gb = lg;
                h->log2gb = ilog2_ceil(lg);
            }
        }
    }
#endif
    const int gbk = h->gb * h->kpl;
    const int n_gblocks = (h->G + gbk - 1) / gbk;
    const int dirs_per_warp = 32 / h->gb;
    int maxq = 1;
    for (int q = 0; q < nquad; ++q) maxq = std::max(maxq, (int)byq[q].size());
    std::vector<StreamDesc> streams;
    if (D.dim == 2) {
        int max_warps = 8;
#ifdef SWEEP_EXPERIMENTS
        if (const char* ev = getenv("SWEEP_MAXWARPS")) max_warps = std::max(1, std::min(8, atoi(ev)));
#endif
        const int nw = std::min(max_warps, std::max(1, (maxq + dirs_per_warp - 1) / dirs_per_warp));
        h->block = 32 * nw;
        h->dset = nw * dirs_per_warp;
    } else {
        h->dset = dirs_per_warp;
    }
    for (int q = 0; q < nquad; ++q) {
        const int nq = (int)byq[q].size();
        for (int gbi = 0; gbi < n_gblocks; ++gbi)
            for (int d0 = 0; d0 < nq; d0 += h->dset) {
                StreamDesc s;
                s.quadrant = q;
                s.g0 = gbi * gbk;
                s.ng = std::min(gbk, h->G - s.g0);
                s.d0 = qstart[q] + d0;
                s.nd = std::min(h->dset, nq - d0);
                streams.push_back(s);
            }
    }
    h->n_streams = (int)streams.size();

    DeviceGuard guard(h->device);
    if (!guard.ok) {
        std::string m = "cannot select CUDA device";
        delete h;
        return fail(nullptr, SWEEP_E_CUDA, m);
    }
    auto bail = [&](int code) {
        (void)cudaGetLastError();  // a failed setup leaves no pending error for later launch checks
        g_setup_error = h->err;
        sweep_destroy(h);
        return code;
    };

    // modal constants (used by p = 2)
    {
        ModalConsts mc;
        memset(&mc, 0, sizeof mc);
        std::string e;
        if (!build_modal(mc, e)) {
            h->err = e;
            return bail(SWEEP_E_INTERNAL);
        }
        int ce = sweepk::upload_modal(mc);
        if (ce) {
            cuda_fail(h, (cudaError_t)ce, "upload_modal");
            return bail(SWEEP_E_CUDA);
        }
    }

    // schedule + workspace
    cudaError_t ce;
    if ((ce = cudaDeviceGetAttribute(&h->n_sm, cudaDevAttrMultiProcessorCount, h->device)) || h->n_sm < 1) {
        if (!ce) ce = cudaErrorInvalidDevice;
        cuda_fail(h, ce, "SM count");
        return bail(SWEEP_E_CUDA);
    }
    if (int re = sweepk::reduce_caps(h->n_sm, &h->caps)) {
        cuda_fail(h, (cudaError_t)re, "occupancy of the reduction kernels");
        return bail(SWEEP_E_CUDA);
    }
    if (D.dim == 2) {
        const int T = sweepk::sweep2d_rows_per_strip(h->p, h->kpl), C = sweepk::sweep2d_cols_per_chunk(h->p, h->kpl, h->opt);
        h->n_strips = (h->ny + T - 1) / T;
        h->n_chunks = (h->nx + C - 1) / C;
        h->n_tasks = h->n_strips * h->n_streams;
        h->smem = (size_t)sweepk::sweep2d_smem_bytes(h->p, h->kpl, gbk, h->dset, h->opt);
        int bps = 0;
        int oe = sweepk::sweep2d_occupancy(h->p, h->log2gb, h->kpl, h->opt, h->block, h->smem, &bps);
        if (oe || bps < 1) {
            if (oe) cuda_fail(h, (cudaError_t)oe, "occupancy");
            else h->err = "sweep2d kernel cannot be resident (registers/shared memory)";
            return bail(SWEEP_E_CUDA);
        }
        h->grid = std::min(h->n_tasks, bps * h->n_sm);
        const int NT = h->np1;
        h->progress_ints = (size_t)h->n_streams * h->n_strips;
        (void)NT;
        // ring record per lane and column: K*NT reals as pairs, or as tagged LL lines
        const int RL = sweepk::sweep2d_ring_record(h->p, h->kpl, h->log2gb, h->opt);
        h->ring_len = (size_t)h->n_streams * 2 * (h->n_chunks * C) * RL * h->block;
        if ((ce = cudaMalloc(&h->d_ytr, sizeof(double) * h->ring_len)))
            return cuda_fail(h, ce, "cudaMalloc ytr"), bail(SWEEP_E_CUDA);
        // LL lines carry the tag of the run that wrote them: no stale memory may match a tag
        if ((ce = cudaMemset(h->d_ytr, 0, sizeof(double) * h->ring_len)))
            return cuda_fail(h, ce, "memset ytr"), bail(SWEEP_E_CUDA);
        if (sweepk::debug_build()) {
            const size_t ntag = (size_t)h->n_streams * 2 * (h->n_chunks * C);
            if ((ce = cudaMalloc(&h->d_ytag, sizeof(int) * ntag)))
                return cuda_fail(h, ce, "cudaMalloc ytag"), bail(SWEEP_E_CUDA);
            if ((ce = cudaMemset(h->d_ytag, 0xff, sizeof(int) * ntag)))
                return cuda_fail(h, ce, "memset ytag"), bail(SWEEP_E_CUDA);
        }
    } else if (!(h->opt & sweepk::OPT_FIXUP)) {
        // warp-scan kernel: one warp per chain (direction, group), one lane per segment;
        // a CTA = up to 8 chains of one half-range (its own slab)
        h->scan1d = true;
        int maxc = 1;
        for (int q = 0; q < 2; ++q) maxc = std::max(maxc, (int)byq[q].size() * h->G);
        const int W = std::min(8, maxc);
        streams.clear();
        for (int q = 0; q < 2; ++q) {
            const int chains = (int)byq[q].size() * h->G;
            for (int c0 = 0; c0 < chains; c0 += W) {
                StreamDesc sdc;
                sdc.quadrant = q;
                sdc.d0 = qstart[q];
                sdc.nd = (int)byq[q].size();
                sdc.g0 = c0;
                sdc.ng = std::min(W, chains - c0);
                streams.push_back(sdc);
            }
        }
        h->n_streams = (int)streams.size();
        h->seglen = (h->nx + 31) / 32;
        h->nseg = 32;
        h->block = 32 * W;
        const int opt1 = h->opt | ((h->flags & SWEEP_HALF_RANGE) ? sweepk::OPT_HALF : 0);
        h->smem = (size_t)sweepk::scan1d_smem_bytes(h->p, opt1, W, 0);
        h->grid = h->n_streams;
        h->n_tasks = h->n_streams;
        h->progress_ints = 0;
        h->fused1d = (size_t)h->n_streams * h->sum_size <= 16384;
        // tiny problems: every chain of both half-ranges in ONE CTA (<= 8 warps), the gray
        // fields accumulated in shared memory: one launch, no slab, no cross-CTA sum
        const int c0 = (int)byq[0].size() * h->G, c1 = (int)byq[1].size() * h->G;
        if (!(h->flags & SWEEP_HALF_RANGE) && c0 + c1 <= 8 && h->nodes * 5 <= 8192) {
            h->single1d = true;
            h->single_nw0 = c0;
            streams.clear();
            for (int q = 0; q < 2; ++q) {
                StreamDesc sdc;
                sdc.quadrant = q;
                sdc.d0 = qstart[q];
                sdc.nd = (int)byq[q].size();
                sdc.g0 = 0;
                sdc.ng = (int)byq[q].size() * h->G;
                streams.push_back(sdc);
            }
            h->n_streams = 2;
            h->block = 32 * (c0 + c1);
            h->smem = (size_t)sweepk::scan1d_smem_bytes(h->p, opt1, c0 + c1, h->nodes);
            h->grid = 1;
            h->n_tasks = 1;
            h->fused1d = true;
        }
    } else {
        // segmented affine scan of the chain; the fixup is not affine: one segment
        h->nseg = (h->opt & sweepk::OPT_FIXUP) ? 1 : std::min(32, std::max(1, (h->nx + 15) / 16));
        h->seglen = (h->nx + h->nseg - 1) / h->nseg;
        h->block = 32 * h->nseg;
        h->smem = sizeof(double) * (size_t)h->nseg * 96;
        h->grid = h->n_streams;
        h->n_tasks = h->n_streams;
        h->progress_ints = 0;
    }
    if ((ce = cudaMalloc(&h->d_dirs, sizeof(DirConst) * std::max<size_t>(1, table.size()))))
        return cuda_fail(h, ce, "cudaMalloc dirs"), bail(SWEEP_E_CUDA);
    if ((ce = cudaMemcpy(h->d_dirs, table.data(), sizeof(DirConst) * table.size(), cudaMemcpyHostToDevice)))
        return cuda_fail(h, ce, "copy dirs"), bail(SWEEP_E_CUDA);
    if ((ce = cudaMalloc(&h->d_streams, sizeof(StreamDesc) * streams.size())))
        return cuda_fail(h, ce, "cudaMalloc streams"), bail(SWEEP_E_CUDA);
    if ((ce = cudaMemcpy(h->d_streams, streams.data(), sizeof(StreamDesc) * streams.size(), cudaMemcpyHostToDevice)))
        return cuda_fail(h, ce, "copy streams"), bail(SWEEP_E_CUDA);
    // progress flags | task counter | error flag, contiguous so one memset resets them
    // progress flags | task counter | error flag | launch epoch (LL ring tags)
    if ((ce = cudaMalloc(&h->d_progress, sizeof(int) * (h->progress_ints + 3))))
        return cuda_fail(h, ce, "cudaMalloc flags"), bail(SWEEP_E_CUDA);
    h->d_counter = h->d_progress + h->progress_ints;
    h->d_err = h->d_counter + 1;
    if ((ce = cudaMemset(h->d_progress, 0, sizeof(int) * (h->progress_ints + 3))))
        return cuda_fail(h, ce, "memset flags"), bail(SWEEP_E_CUDA);
    if ((ce = cudaMalloc(&h->d_slabs, sizeof(double) * h->out_size * (size_t)h->n_streams)))
        return cuda_fail(h, ce, "cudaMalloc slabs"), bail(SWEEP_E_CUDA);
    if ((ce = cudaMalloc(&h->d_out, sizeof(double) * h->out_size)))
        return cuda_fail(h, ce, "cudaMalloc out"), bail(SWEEP_E_CUDA);

    // NCCL for nranks > 1; SWEEP_FORCE_COMM also builds a 1-rank communicator when an id is
    // given, so the NCCL plumbing can run on a single-GPU box
    if (h->nranks > 1 || ((D.flags & SWEEP_FORCE_COMM) && D.nccl_id)) {
        std::string e;
        if (!g_nccl.load(e)) {
            h->err = e;
            return bail(SWEEP_E_NCCL);
        }
        ncclUniqueId_t id;
        memcpy(&id, D.nccl_id, 128);
        int r = g_nccl.commInitRank(&h->comm, h->nranks, id, h->rank);
        if (r != 0) {
            h->comm = nullptr;
            h->err = std::string("ncclCommInitRank: ") + (g_nccl.getErrorString ? g_nccl.getErrorString(r) : "error");
            return bail(SWEEP_E_NCCL);
        }
    }
    *out = h;
    return SWEEP_OK;
}

extern "C" int sweep_layout(const sweep_handle* h, size_t off[8], size_t* total) {
    if (!h || !off || !total) return SWEEP_E_ARG;
    for (int i = 0; i < 8; ++i) off[i] = h->off[i];
    *total = h->out_size;
    return SWEEP_OK;
}

// InputBands: the 2-D kernel's per-band input-ready flags (sweep_run_host's overlapped copy);
// ready == nullptr: the inputs are resident when the kernel starts
struct InputBands {
    const int* ready = nullptr;
    int gen = 0, band_rows = 1;
};

static int run_impl(sweep_handle* h, const double* d_sigma, double inv_c_dt, const double* d_q,
                    const double* d_inflow, void* stream, InputBands bands);

extern "C" int sweep_run(sweep_handle* h, const double* d_sigma, double inv_c_dt, const double* d_q,
                         const double* d_inflow, void* stream) {
    return run_impl(h, d_sigma, inv_c_dt, d_q, d_inflow, stream, InputBands{});
}

static int run_impl(sweep_handle* h, const double* d_sigma, double inv_c_dt, const double* d_q,
                    const double* d_inflow, void* stream, InputBands bands) {
    NvtxRange nv("sweep_run");
    if (!h) return SWEEP_E_ARG;
    if (!d_sigma || !d_q || !d_inflow) return fail(h, SWEEP_E_ARG, "null input pointer");
    if (!std::isfinite(inv_c_dt) || !(inv_c_dt > 0)) return fail(h, SWEEP_E_ARG, "inv_c_dt must be finite and > 0");
    DeviceGuard guard(h->device);
    if (!guard.ok) return fail(h, SWEEP_E_CUDA, "cannot select device");
    cudaStream_t st = (cudaStream_t)stream;
    cudaError_t ce;
    // reset progress flags and the task counter (the error flag is sticky until closures_get);
    // the 1-D scan kernel has no flags and resets its own completion counter
    if (!h->scan1d && (ce = cudaMemsetAsync(h->d_progress, 0, sizeof(int) * (h->progress_ints + 1), st)))
        return cuda_fail(h, ce, "memset flags");
    if (h->d_ytag &&  // debug builds: tags of this run only
        (ce = cudaMemsetAsync(h->d_ytag, 0xff, sizeof(int) * (size_t)h->n_streams * 2 *
                                                   (h->n_chunks * sweepk::sweep2d_cols_per_chunk(h->p, h->kpl, h->opt)),
                              st)))
        return cuda_fail(h, ce, "memset ytag");
    int e;
    h->launches = 0;
    cudaEvent_t* evs = nullptr;
    if (h->timing) {
        evs = &h->ev[(size_t)(h->runs_recorded % sweep_handle::kRing) * 4];
        cudaEventRecord(evs[0], st);
    }
    if (h->dim == 2) {
        sweepk::Sweep2DParams prm;
        prm.nx = h->nx;
        prm.ny = h->ny;
        prm.G = h->G;
        prm.nx_pad = h->n_chunks * sweepk::sweep2d_cols_per_chunk(h->p, h->kpl, h->opt);
        // 1-D bulk copies (cp.async.bulk) of the q / sigma group rows need 16-byte aligned
        // rows: G even (the group offsets of the streams are even then) and aligned bases
        prm.bulk_ok = (h->G % 2 == 0 && (reinterpret_cast<uintptr_t>(d_q) & 15u) == 0 &&
                       (reinterpret_cast<uintptr_t>(d_sigma) & 15u) == 0)
                          ? 1
                          : 0;
        prm.n_streams = h->n_streams;
        prm.n_strips = h->n_strips;
        prm.n_chunks = h->n_chunks;
        prm.n_tasks = h->n_tasks;
        prm.gb = h->gb;
        prm.kpl = h->kpl;
        prm.dset = h->dset;
        prm.nbnode = h->nbnode;
        prm.half = (h->flags & SWEEP_HALF_RANGE) ? 1 : 0;
        prm.hr_off = h->off[7];
        prm.inv_c_dt = inv_c_dt;
        prm.sigma = d_sigma;
        prm.q = d_q;
        prm.inflow = d_inflow;
        prm.dirs = h->d_dirs;
        prm.streams = h->d_streams;
        prm.progress = h->d_progress;
        prm.epoch = h->d_err + 1;
        prm.task_counter = h->d_counter;
        prm.ytr = h->d_ytr;
        prm.ring_len = h->ring_len;
        prm.ytag = h->d_ytag;
        prm.slabs = h->d_slabs;
        prm.out_size = h->out_size;
        prm.nodes = h->nodes;
        prm.err = h->d_err;
        prm.in_ready = bands.ready;
        prm.in_gen = bands.gen;
        prm.in_band_rows = bands.band_rows;
        e = sweepk::launch_sweep2d(h->p, h->log2gb, h->kpl, h->opt, prm, h->grid, h->block, h->smem, stream);
    } else if (h->scan1d) {
        sweepk::Sweep1DScanParams prm;
        prm.nx = h->nx;
        prm.G = h->G;
        prm.seglen = h->seglen;
        prm.nodes = h->nodes;
        prm.out_size = h->out_size;
        prm.sum_size = h->sum_size;
        prm.hr_off = h->off[7];
        prm.inv_c_dt = inv_c_dt;
        prm.sigma = d_sigma;
        prm.q = d_q;
        prm.inflow = d_inflow;
        prm.dirs = h->d_dirs;
        prm.streams = h->d_streams;
        prm.slabs = h->d_slabs;
        prm.err = h->d_err;
        prm.done_counter = h->d_counter;
        prm.fused_out = h->fused1d ? h->d_out : nullptr;
        prm.single = h->single1d ? 1 : 0;
        prm.nw0 = h->single_nw0;
        const int opt1 = h->opt | ((h->flags & SWEEP_HALF_RANGE) ? sweepk::OPT_HALF : 0);
        e = sweepk::launch_sweep1d_scan(h->p, opt1, prm, h->grid, h->block, h->smem, stream);
    } else {
        sweepk::Sweep1DParams prm;
        prm.nx = h->nx;
        prm.G = h->G;
        prm.n_streams = h->n_streams;
        prm.gb = h->gb;
        prm.nseg = h->nseg;
        prm.seglen = h->seglen;
        prm.hr_off = h->off[7];
        prm.inv_c_dt = inv_c_dt;
        prm.sigma = d_sigma;
        prm.q = d_q;
        prm.inflow = d_inflow;
        prm.dirs = h->d_dirs;
        prm.streams = h->d_streams;
        prm.slabs = h->d_slabs;
        prm.out_size = h->out_size;
        prm.nodes = h->nodes;
        prm.err = h->d_err;
        const int opt1 = h->opt | ((h->flags & SWEEP_HALF_RANGE) ? sweepk::OPT_HALF : 0);
        e = sweepk::launch_sweep1d(h->p, h->log2gb, opt1, prm, h->grid, h->block, h->smem, stream);
    }
    if (e) return cuda_fail(h, (cudaError_t)e, "launch sweep");
    ++h->launches;
    if (evs) cudaEventRecord(evs[1], st);
    const bool modal = (h->dim == 2 && h->p == 2);  // the p = 2 sweep leaves modal node fields in the slabs
    if (h->fused1d) {
        // summed by the sweep kernel's last CTA
    } else if (!modal) {
        e = sweepk::launch_finalize(h->d_slabs, h->n_streams, h->out_size, h->sum_size, h->d_out, h->d_err,
                                    h->caps.finalize, stream);
        if (e) return cuda_fail(h, (cudaError_t)e, "launch finalize");
        ++h->launches;
    } else {
        const size_t nel = h->nodes / 9;
        // phi, J, T rows | beta, J+ (plain sum) | sigma phi, sigma J rows (SWEEP_SIGMA_MOMENTS)
        e = sweepk::launch_finalize_modal(h->d_slabs, h->n_streams, h->out_size, h->d_streams, 0, 6, nel, h->d_out,
                                          h->d_err, h->caps.finalize_modal, stream);
        if (!e)
            e = sweepk::launch_finalize(h->d_slabs + h->off[3], h->n_streams, h->out_size, 2 * (size_t)h->nbnode,
                                        h->d_out + h->off[3], h->d_err, h->caps.finalize, stream);
        if (!e && h->off[7] > h->off[5])
            e = sweepk::launch_finalize_modal(h->d_slabs, h->n_streams, h->out_size, h->d_streams, h->off[5], 3, nel,
                                              h->d_out, h->d_err, h->caps.finalize_modal, stream);
        if (e) return cuda_fail(h, (cudaError_t)e, "launch finalize");
        h->launches += (h->off[7] > h->off[5]) ? 3 : 2;
    }
    if (h->out_size > h->sum_size) {
        e = sweepk::launch_halfrange(h->d_slabs, h->n_streams, h->out_size, h->d_streams, h->nodes, h->off[7], h->dim,
                                     modal ? 1 : 0, h->d_out + h->sum_size, h->caps.halfrange, stream);
        if (e) return cuda_fail(h, (cudaError_t)e, "launch halfrange");
        ++h->launches;
    }
    if (evs) cudaEventRecord(evs[2], st);
    if (h->comm) {
        NvtxRange nva("sweep_allreduce");
        int r = g_nccl.allReduce(h->d_out, h->d_out, h->out_size, kNcclFloat64, kNcclSum, h->comm, st);
        if (r != 0)
            return fail(h, SWEEP_E_NCCL, std::string("ncclAllReduce: ") + (g_nccl.getErrorString ? g_nccl.getErrorString(r) : "error"));
    }
    if (evs) {
        if (h->comm) cudaEventRecord(evs[3], st);  // without a collective: no all-reduce interval
        ++h->runs_recorded;
    }
    return SWEEP_OK;
}

extern "C" int sweep_timing(sweep_handle* h, int enable) {
    if (!h) return SWEEP_E_ARG;
    DeviceGuard guard(h->device);
    if (enable && h->ev.empty()) {
        h->ev.resize((size_t)sweep_handle::kRing * 4);
        for (auto& e : h->ev) {
            cudaError_t ce = cudaEventCreate(&e);
            if (ce) return cuda_fail(h, ce, "cudaEventCreate");
        }
    }
    h->timing = enable != 0;
    if (enable) h->runs_recorded = 0;
    return SWEEP_OK;
}

extern "C" int sweep_kernel_times(sweep_handle* h, double* ms, int max_runs, int* n_runs) {
    if (!h || !ms || !n_runs) return SWEEP_E_ARG;
    DeviceGuard guard(h->device);
    const long long have = std::min<long long>(h->runs_recorded, sweep_handle::kRing);
    const int n = (int)std::min<long long>(have, max_runs);
    const long long first = h->runs_recorded - n;
    for (int r = 0; r < n; ++r) {
        cudaEvent_t* e = &h->ev[(size_t)((first + r) % sweep_handle::kRing) * 4];
        const int last = h->comm ? 3 : 2;
        cudaError_t ce = cudaEventSynchronize(e[last]);
        if (ce) return cuda_fail(h, ce, "cudaEventSynchronize");
        ms[3 * r + 2] = 0.0;
        for (int k = 0; k < last; ++k) {
            float t = 0;
            ce = cudaEventElapsedTime(&t, e[k], e[k + 1]);
            if (ce) return cuda_fail(h, ce, "cudaEventElapsedTime");
            ms[3 * r + k] = t;
        }
    }
    *n_runs = n;
    return SWEEP_OK;
}

extern "C" int sweep_fp64_probe(int device, double* tflops) {
    if (!tflops) return SWEEP_E_ARG;
    int prev = -1;
    cudaGetDevice(&prev);
    int e = sweepk::fp64_probe(device, tflops);
    if (prev >= 0) cudaSetDevice(prev);
    if (e) return fail(nullptr, SWEEP_E_CUDA, std::string("fp64 probe: ") + sweepk::cuda_err_string(e));
    return SWEEP_OK;
}

extern "C" int closures_get(sweep_handle* h, double* out, size_t n, void* stream) {
    NvtxRange nv("closures_get");
    if (!h || !out) return SWEEP_E_ARG;
    if (n != h->out_size) return fail(h, SWEEP_E_ARG, "n_doubles must equal the layout total");
    DeviceGuard guard(h->device);
    cudaStream_t st = (cudaStream_t)stream;
    cudaError_t ce;
    int flag = 0;
    if ((ce = cudaMemcpyAsync(out, h->d_out, sizeof(double) * n, cudaMemcpyDefault, st))) return cuda_fail(h, ce, "copy out");
    if ((ce = cudaMemcpyAsync(&flag, h->d_err, sizeof(int), cudaMemcpyDeviceToHost, st))) return cuda_fail(h, ce, "copy flag");
    if ((ce = cudaStreamSynchronize(st))) return cuda_fail(h, ce, "sync");
    if (flag) {
        cudaMemset(h->d_err, 0, sizeof(int));
        return fail(h, SWEEP_E_SIGMA,
                    (flag & 32)  ? "debug check failed: out-of-bounds index or trace-ring inconsistency"
                    : (flag & 4) ? "internal: wavefront dependency timeout"
                    : (flag & 1) ? "sigma_t + 1/(c dt) <= 0 or non-finite sigma"
                                 : "non-finite result (non-finite q or inflow)");
    }
    return SWEEP_OK;
}

// cuStreamWriteValue32 from the driver the runtime loaded (no link-time libcuda dependency);
// nullptr if unavailable (sweep_run_host then copies before the sweep)
using WriteValue32Fn = int (*)(void* stream, unsigned long long addr, unsigned value, unsigned flags);
static WriteValue32Fn write_value32() {
    static WriteValue32Fn fn = []() -> WriteValue32Fn {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &f, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess) {
            cudaGetLastError();
            return nullptr;
        }
        return reinterpret_cast<WriteValue32Fn>(f);
    }();
    return fn;
}

extern "C" int sweep_run_host(sweep_handle* h, const double* h_sigma, double inv_c_dt, const double* h_q,
                              const double* h_inflow, double* h_out, size_t n, void* stream) {
    if (!h || !h_sigma || !h_q || !h_inflow || !h_out) return SWEEP_E_ARG;
    DeviceGuard guard(h->device);
    const size_t ns = (size_t)h->nx * h->ny * h->G, nq = ns * h->n, nf = (size_t)h->nbnode * h->G;
    cudaError_t ce;
    if (!h->d_in_sigma) {
        if ((ce = cudaMalloc(&h->d_in_sigma, sizeof(double) * ns))) return cuda_fail(h, ce, "cudaMalloc staging");
        if ((ce = cudaMalloc(&h->d_in_q, sizeof(double) * nq))) return cuda_fail(h, ce, "cudaMalloc staging");
        if ((ce = cudaMalloc(&h->d_in_inflow, sizeof(double) * nf))) return cuda_fail(h, ce, "cudaMalloc staging");
    }
    cudaStream_t st = (cudaStream_t)stream;
    if (h->dim == 2 && write_value32()) {
        // 2-D: the copy overlaps the sweep.  Bands of kBandRows physical rows are copied on a
        // copy stream from both ends of the mesh inwards (the order in which the +y and -y
        // quadrant streams reach them); after each band a stream memory operation (no SM
        // needed, preceded by a system-scope fence) writes the band's flag = this run's
        // generation, and every strip of the kernel waits for the flags of its rows.
        constexpr int kBandRows = 8;
        const int nb = (h->ny + kBandRows - 1) / kBandRows;
        if (!h->cp_stream) {
            if ((ce = cudaStreamCreateWithFlags(&h->cp_stream, cudaStreamNonBlocking))) return cuda_fail(h, ce, "copy stream");
            if ((ce = cudaEventCreateWithFlags(&h->cp_ev[0], cudaEventDisableTiming))) return cuda_fail(h, ce, "copy event");
            if ((ce = cudaEventCreateWithFlags(&h->cp_ev[1], cudaEventDisableTiming))) return cuda_fail(h, ce, "copy event");
            if ((ce = cudaMalloc(&h->d_in_ready, sizeof(int) * nb))) return cuda_fail(h, ce, "cudaMalloc band flags");
            if ((ce = cudaMemset(h->d_in_ready, 0, sizeof(int) * nb))) return cuda_fail(h, ce, "memset band flags");
        }
        if (++h->in_gen <= 0) {  // generation wrap (2^31 runs): restart from 1 with cleared flags
            h->in_gen = 1;
            if ((ce = cudaMemsetAsync(h->d_in_ready, 0, sizeof(int) * nb, st))) return cuda_fail(h, ce, "memset band flags");
        }
        cudaStream_t cp = h->cp_stream;
        // the staging buffers are free once the work queued on st so far is done
        if ((ce = cudaEventRecord(h->cp_ev[0], st)) || (ce = cudaStreamWaitEvent(cp, h->cp_ev[0], 0)))
            return cuda_fail(h, ce, "copy stream order");
        if ((ce = cudaMemcpyAsync(h->d_in_inflow, h_inflow, sizeof(double) * nf, cudaMemcpyHostToDevice, cp))) return cuda_fail(h, ce, "H2D");
        const size_t row_s = (size_t)h->nx * h->G, row_q = row_s * h->n;
        for (int k = 0; k < nb; ++k) {
            const int b = (k & 1) ? nb - 1 - k / 2 : k / 2;
            const size_t j0 = (size_t)b * kBandRows, nr = std::min<size_t>(kBandRows, h->ny - j0);
            if ((ce = cudaMemcpyAsync(h->d_in_q + j0 * row_q, h_q + j0 * row_q, sizeof(double) * nr * row_q,
                                      cudaMemcpyHostToDevice, cp)) ||
                (ce = cudaMemcpyAsync(h->d_in_sigma + j0 * row_s, h_sigma + j0 * row_s, sizeof(double) * nr * row_s,
                                      cudaMemcpyHostToDevice, cp)))
                return cuda_fail(h, ce, "H2D");
            const int rv = write_value32()(cp, reinterpret_cast<unsigned long long>(h->d_in_ready + b), (unsigned)h->in_gen, 0);
            if (rv) return fail(h, SWEEP_E_CUDA, "cuStreamWriteValue32 failed: " + std::to_string(rv));
        }
        if ((ce = cudaEventRecord(h->cp_ev[1], cp))) return cuda_fail(h, ce, "copy event");
        InputBands bands;
        bands.ready = h->d_in_ready;
        bands.gen = h->in_gen;
        bands.band_rows = kBandRows;
        int r = run_impl(h, h->d_in_sigma, inv_c_dt, h->d_in_q, h->d_in_inflow, stream, bands);
        // join: later work on st (and the next run's copies) is ordered after the copies
        if ((ce = cudaStreamWaitEvent(st, h->cp_ev[1], 0))) return cuda_fail(h, ce, "copy join");
        if (r) return r;
        return closures_get(h, h_out, n, stream);
    }
    if ((ce = cudaMemcpyAsync(h->d_in_sigma, h_sigma, sizeof(double) * ns, cudaMemcpyHostToDevice, st))) return cuda_fail(h, ce, "H2D");
    if ((ce = cudaMemcpyAsync(h->d_in_q, h_q, sizeof(double) * nq, cudaMemcpyHostToDevice, st))) return cuda_fail(h, ce, "H2D");
    if ((ce = cudaMemcpyAsync(h->d_in_inflow, h_inflow, sizeof(double) * nf, cudaMemcpyHostToDevice, st))) return cuda_fail(h, ce, "H2D");
    int r = sweep_run(h, h->d_in_sigma, inv_c_dt, h->d_in_q, h->d_in_inflow, stream);
    if (r) return r;
    return closures_get(h, h_out, n, stream);
}

extern "C" int trt_step(sweep_handle* h, const double* d_sigma, const double* d_inflow, const double* d_Tk,
                        const double* d_Iprev, const trt_params* prm, double* d_T, int* iterations, void* stream) {
    if (!h || !d_sigma || !d_inflow || !d_Tk || !d_Iprev || !prm || !prm->nu || !d_T || !iterations)
        return SWEEP_E_ARG;
    if (!(h->opt & sweepk::OPT_SIGMA)) return fail(h, SWEEP_E_ARG, "trt_step needs a handle with SWEEP_SIGMA_MOMENTS");
    if (h->nranks != 1) return fail(h, SWEEP_E_ARG, "trt_step runs on one rank (the elimination needs every group)");
    if (!(prm->cv > 0) || !(prm->dt > 0) || prm->max_iter < 1 || !std::isfinite(prm->cv) || !std::isfinite(prm->dt))
        return fail(h, SWEEP_E_ARG, "trt_step: cv, dt > 0 and max_iter >= 1 required");
    for (int g = 0; g <= h->G; ++g)
        if (!(prm->nu[g] >= 0) || (g > 0 && !(prm->nu[g] > prm->nu[g - 1])))
            return fail(h, SWEEP_E_ARG, "trt_step: nu must be increasing and >= 0");
    DeviceGuard guard(h->device);
    cudaStream_t st = (cudaStream_t)stream;
    cudaError_t ce;
    const size_t nq = h->nodes * (size_t)h->G;
    if (!h->d_trt_q) {
        if ((ce = cudaMalloc(&h->d_trt_q, sizeof(double) * nq))) return cuda_fail(h, ce, "cudaMalloc trt q");
        if ((ce = cudaMalloc(&h->d_trt_nu, sizeof(double) * (h->G + 1)))) return cuda_fail(h, ce, "cudaMalloc trt nu");
        if ((ce = cudaMalloc(&h->d_trt_part, sizeof(double) * 2 * sweepk::trt_blocks(h->n_sm))))
            return cuda_fail(h, ce, "cudaMalloc trt partials");
        if ((ce = cudaMalloc(&h->d_trt_norm, sizeof(double) * 2))) return cuda_fail(h, ce, "cudaMalloc trt norms");
        if ((ce = cudaMalloc(&h->d_trt_E, sizeof(double) * h->nodes))) return cuda_fail(h, ce, "cudaMalloc trt E");
    }
    if ((ce = cudaMemcpyAsync(h->d_trt_nu, prm->nu, sizeof(double) * (h->G + 1), cudaMemcpyHostToDevice, st)))
        return cuda_fail(h, ce, "copy nu");
    if ((ce = cudaMemcpyAsync(d_T, d_Tk, sizeof(double) * h->nodes, cudaMemcpyDeviceToDevice, st)))
        return cuda_fail(h, ce, "copy Tk");
    // u^0 = [T^k, E^k], E^k = sum_g I^k_g
    if (int e0 = sweepk::launch_trt_e0(d_Iprev, h->G, h->nodes, h->d_trt_E, h->n_sm, stream))
        return cuda_fail(h, (cudaError_t)e0, "launch trt E0");
    const double inv_dt = 1.0 / prm->dt, cv_dt = prm->cv / prm->dt;
    // outer stopping rule (eq:relative_tol): stop after the first
    // iteration l >= 2 with ||u^l - u^{l-1}||_2 < eps ||u^1 - u^0||_2, u = [T, E = phi];
    // after iteration 1 if u^1 = u^0 exactly
    double first = 0.0;
    int it = 0;
    for (it = 1; it <= prm->max_iter; ++it) {
        NvtxRange nvi("trt_outer_iteration");
        int e = sweepk::launch_trt_emission(d_T, d_sigma, d_Iprev, h->d_trt_nu, h->G, h->n, h->nodes, inv_dt, h->d_trt_q,
                                            h->n_sm, stream);
        if (e) return cuda_fail(h, (cudaError_t)e, "launch trt emission");
        int rc = sweep_run(h, d_sigma, inv_dt, h->d_trt_q, d_inflow, stream);
        if (rc) return rc;
        e = sweepk::launch_trt_update(d_Tk, d_T, h->d_out + h->off[5], h->d_out + h->off[0], h->d_trt_E, d_sigma,
                                      h->d_trt_nu, h->G, h->n, h->nodes, cv_dt, h->d_trt_part, h->d_trt_norm, h->d_err,
                                      h->n_sm, stream);
        if (e) return cuda_fail(h, (cudaError_t)e, "launch trt update");
        double norms[2] = {0.0, 0.0};
        if ((ce = cudaMemcpyAsync(norms, h->d_trt_norm, sizeof norms, cudaMemcpyDeviceToHost, st)))
            return cuda_fail(h, ce, "copy norms");
        if ((ce = cudaStreamSynchronize(st))) return cuda_fail(h, ce, "sync");
        const double dn = std::sqrt(norms[0] + norms[1]);
        if (it == 1) first = dn;
        if (prm->ratios) prm->ratios[it - 1] = (first > 0.0) ? dn / first : 0.0;
        if (prm->eps > 0 && (first == 0.0 || (it >= 2 && dn < prm->eps * first))) break;
    }
    *iterations = std::min(it, prm->max_iter);
    int flag = 0;
    if ((ce = cudaMemcpy(&flag, h->d_err, sizeof(int), cudaMemcpyDeviceToHost))) return cuda_fail(h, ce, "copy flag");
    if (flag) {
        cudaMemset(h->d_err, 0, sizeof(int));
        return fail(h, SWEEP_E_SIGMA, (flag & 16) ? "trt_step: temperature elimination failed (non-positive or no root)"
                                                  : "trt_step: device error flag set in the sweep");
    }
    return SWEEP_OK;
}

extern "C" int sweep_stats(const sweep_handle* h, long long out[8]) {
    if (!h || !out) return SWEEP_E_ARG;
    out[0] = h->launches;
    out[1] = h->n_dir_eff;
    out[2] = h->n_streams;
    out[3] = h->grid;
    out[4] = h->block;
    out[5] = (h->dim == 2) ? h->kpl : 1;
    out[6] = h->gb;
    out[7] = h->n_sm;
    return SWEEP_OK;
}

extern "C" int sweep_selfcheck_solves(int device, int p, int n, unsigned long long seed, double* max_rel_err) {
    if (!max_rel_err || (p != 1 && p != 2) || n < 1) return SWEEP_E_ARG;
    int prev = -1;
    cudaGetDevice(&prev);
    // the p = 2 check needs the modal constants of the library's own setup
    ModalConsts mc;
    memset(&mc, 0, sizeof mc);
    std::string err;
    int e = 0;
    if (!build_modal(mc, err)) {
        if (prev >= 0) cudaSetDevice(prev);
        return fail(nullptr, SWEEP_E_INTERNAL, err);
    }
    if (!(e = cudaSetDevice(device))) e = sweepk::upload_modal(mc);
    if (!e) e = sweepk::selfcheck_solves(device, p, n, seed, max_rel_err);
    if (prev >= 0) cudaSetDevice(prev);
    if (e) return fail(nullptr, SWEEP_E_CUDA, std::string("selfcheck: ") + sweepk::cuda_err_string(e));
    return SWEEP_OK;
}

extern "C" int sweep_launch_floor(int device, int reps, double* us_per_launch) {
    if (!us_per_launch || reps < 1) return SWEEP_E_ARG;
    int prev = -1;
    cudaGetDevice(&prev);
    int e = sweepk::launch_floor(device, reps, us_per_launch);
    if (prev >= 0) cudaSetDevice(prev);
    if (e) return fail(nullptr, SWEEP_E_CUDA, std::string("launch floor: ") + sweepk::cuda_err_string(e));
    return SWEEP_OK;
}

extern "C" void sweep_destroy(sweep_handle* h) {
    if (!h) return;
    DeviceGuard guard(h->device);
    if (h->comm && g_nccl.commDestroy) g_nccl.commDestroy(h->comm);
    for (auto& e : h->ev) cudaEventDestroy(e);
    cudaFree(h->d_dirs);
    cudaFree(h->d_streams);
    cudaFree(h->d_trt_q);
    cudaFree(h->d_trt_nu);
    cudaFree(h->d_trt_part);
    cudaFree(h->d_trt_norm);
    cudaFree(h->d_trt_E);
    cudaFree(h->d_progress);
    cudaFree(h->d_ytr);
    cudaFree(h->d_ytag);
    cudaFree(h->d_slabs);
    cudaFree(h->d_out);
    if (h->cp_stream) {  // copies still in flight write the staging buffers freed below
        cudaStreamSynchronize(h->cp_stream);
        cudaStreamDestroy(h->cp_stream);
    }
    cudaFree(h->d_in_sigma);
    cudaFree(h->d_in_q);
    cudaFree(h->d_in_inflow);
    cudaFree(h->d_in_ready);
    for (auto& e : h->cp_ev)
        if (e) cudaEventDestroy(e);
    delete h;
}

extern "C" const char* sweep_last_error(const sweep_handle* h) {
    if (!h) return g_setup_error.c_str();
    return h->err.c_str();
}
