/*
 * sweep.h — C ABI of libsweep.so: the B200 (sm_100a) DG S_N transport sweep
 * fused with the gray Second-Moment closures of arXiv 2504.21784.
 *
 * What one sweep_run computes (PAPER.md = /root/reference/PAPER.md):
 *   For every direction d of the quadrature set and every local group g,
 *   psi_{d,g} in Y_p (discontinuous, tensor GLL nodal basis of order p) is the
 *   solution of the lumped upwind-DG weak form (eq:dgsn_transport,
 *   PAPER.md:332-336, upwind flux PAPER.md:299-327, GLL lumping PAPER.md:654)
 *   of the backward-Euler transport equation (eq:smm_be_transport)
 *       Omega_d . grad psi + (sigma_t,g + 1/(c dt)) psi = q_g
 *   with a GIVEN isotropic nodal source q (each high-order solve "inverts the
 *   left hand side ... only") and the prescribed isotropic inflow
 *   on inflow faces.  psi is never stored; the library
 *   returns only the gray sums over all directions and groups
 *       phi  = sum_g sum_d w_d psi                     (c E,   PAPER.md:156-158)
 *       J    = sum_g sum_d w_d Omega_d psi             (F,     PAPER.md:160-161)
 *       T    = sum_g sum_d w_d (Omega_d Omega_d - I/3) psi
 *       beta = sum_g sum_d w_d (|Omega_d . n| - alpha_n) psi
 *       J+   = sum_g sum_{Omega_d.n > 0} w_d (Omega_d . n) psi
 *   with alpha_n = sum_d w_d |Omega_d . n| / sum_d w_d  (eq:alpha),
 *   beta and J+ on every boundary face node, using the element's own nodal
 *   trace for every direction (reading R5).
 *
 * Mesh: uniform Cartesian, dim 1 (slab [0,lx], nx elements) or 2 ([0,lx]x[0,ly],
 * nx*ny quads).  Element e = i + nx*j.  Node k = a + (p+1)*b (a: x index,
 * b: y index) at the GLL points of the element; n = (p+1)^dim.
 * Boundary face nodes, in this order: face x- (j = 0..ny-1, b = 0..p),
 * x+ (j, b), y- (i = 0..nx-1, a = 0..p), y+ (i, a); a corner node appears once
 * per face (reading R18).  dim 1: [x = 0, x = lx].  N_bnode = 2 (dim 1) or
 * 2 (nx + ny)(p + 1).
 *
 * Output packing (doubles), all gray = summed over every group of every rank:
 *   phi[N_el][n] | J[dim][N_el][n] | T[nT][N_el][n] | beta[N_bnode] | Jplus[N_bnode]
 *   [ | sphi[N_el][n] | sJ[dim][N_el][n]    with SWEEP_SIGMA_MOMENTS ]
 *   [ | HR[10 or 2][N_el][n]                 with SWEEP_HALF_RANGE ]
 *   nT = 1 (dim 1: T_xx) or 3 (dim 2: T_xx, T_xy, T_yy; T_zz = -T_xx - T_yy).
 *   sphi = sum_g sigma_t,g phi_g and sJ = sum_g sigma_t,g J_g are the sigma-weighted
 *   gray moments the gray low-order system takes from the sweep: the numerator of
 *   sigma_E (eq:sigmaE) and the high-order part of the additive
 *   multigroup correction sum_g (sigma_F - sigma_g) F_g (eq:additive_mg_correction,
 *   PAPER.md:197-203, :247).  sigma_t excludes 1/(c dt).
 *   HR are the half-range moments of the consistent low-order method
 *   (PAPER.md:424-428), at every node (= each element's own trace at its face nodes):
 *     dim 2: F+_{+x}[x,y], P+_{+x}[xx,xy,yy], F+_{+y}[x,y], P+_{+y}[xx,xy,yy]
 *     dim 1: F+ , P+            (F+_n = sum_g sum_{Omega.n>0} w Omega psi,
 *                                P+_n = sum_g sum_{Omega.n>0} w Omega Omega psi;
 *   Omega.n = 0 counts as + (reading R23); the minus halves are J - F+ and
 *   (T + phi I/3) - P+, and sum w |Omega.n| psi = 2 F+_n . n - J.n gives beta on
 *   every interior face, so the jumps the consistent method needs follow).
 *
 * Every function returns an int status (SWEEP_OK = 0) and never aborts or
 * throws across the ABI; sweep_last_error gives the message of the last
 * failure on a handle.  A handle is not re-entrant; separate handles may be
 * used from separate threads/streams.  Each call sets the handle's device and
 * restores the caller's current device before returning.
 */
#ifndef PAPER_2504_21784_B200_SWEEP_H
#define PAPER_2504_21784_B200_SWEEP_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    SWEEP_OK = 0,
    SWEEP_E_ARG = 1,      /* null pointer, dim not in {1,2}, p not in {1,2}, sizes <= 0, lx/ly <= 0 */
    SWEEP_E_QUAD = 2,     /* |sum w - 1| > 1e-13, w_d <= 0, |Omega_d| != 1 (dim 2) or |mu| > 1 (dim 1) */
    SWEEP_E_SIGMA = 3,    /* sigma_t + 1/(c dt) <= 0 or non-finite sigma, or a non-finite result
                             (non-finite q / inflow); detected on the device, reported by closures_get */
    SWEEP_E_CUDA = 4,     /* CUDA error (message via sweep_last_error) */
    SWEEP_E_NCCL = 5,     /* NCCL missing or failed */
    SWEEP_E_INTERNAL = 6  /* setup self-check failed (e.g. eigen-decomposition residual) */
};

/* flags */
#define SWEEP_FOLD_Z 1u          /* dim 2: sweep each pair of directions with identical (Omega_x, Omega_y)
                                    (e.g. +-Omega_z) once with the summed weight; exact (reading R20) */
#define SWEEP_DETERMINISTIC 2u   /* accepted for API compatibility: every reduction already runs in a
                                    fixed order, so results are bitwise repeatable in all modes */
#define SWEEP_SIGMA_MOMENTS 4u   /* also return sphi, sJ (see the output packing above) */
#define SWEEP_HALF_RANGE 16u     /* also return the half-range moments HR (see the output packing) */
#define SWEEP_FIXUP 8u           /* zero-and-scale negative flux fixup inside the sweep (PAPER.md:987,
                                    :1321): after every element solve, negative nodal values are set
                                    to 0 and the others scaled to keep the element integral
                                    sum_k W_k psi_k (W_k the lumped GLL mass); a non-positive integral
                                    zeroes the element.  The downwind elements see the fixed values.
                                    Nonlinear: no longer the solution of one linear system. */
#define SWEEP_FORCE_COMM 32u     /* with nranks = 1 and a nccl_id: still build a 1-rank NCCL communicator
                                    and end every sweep_run with the (trivial) all-reduce, so the
                                    collective's plumbing can be exercised on a single GPU */

typedef struct sweep_handle sweep_handle;   /* opaque, owned by the library */

typedef struct {
    int dim;                 /* 1 or 2 */
    int nx, ny;              /* elements per axis; ny ignored (treated as 1) for dim 1 */
    double lx, ly;           /* domain lengths (> 0); ly ignored for dim 1 */
    int p;                   /* DG order: 1 (paper) or 2 (reading R1) */
    int n_dir;               /* number of directions */
    const double *omega;     /* HOST [n_dir][3] unit vectors (dim 1: omega[d][0] = mu_d); copied at setup */
    const double *w;         /* HOST [n_dir] weights, sum = 1 (+-1e-13), each > 0; copied at setup */
    int n_group_local;       /* groups held by this rank (G_loc >= 1) */
    int group_offset;        /* first global group index of this rank (informational) */
    int n_group_total;       /* total groups over all ranks (informational) */
    int device;              /* CUDA device ordinal */
    int nranks, rank;        /* nranks = 1: no collective; > 1: NCCL all-reduce of the gray output */
    const void *nccl_id;     /* 128-byte ncclUniqueId created by rank 0 and broadcast (nranks > 1), else NULL */
    unsigned flags;          /* SWEEP_FOLD_Z | SWEEP_DETERMINISTIC | SWEEP_SIGMA_MOMENTS | SWEEP_FIXUP | SWEEP_HALF_RANGE
                                | SWEEP_FORCE_COMM */
} sweep_desc;

/* Validate the description, fold/sort directions into sweep quadrants,
 * precompute per-direction tables (a1) and the wavefront schedule (a2),
 * allocate device workspace and, for nranks > 1, initialise the NCCL
 * communicator (ncclCommInitRank; collective over all ranks).
 * *out receives the handle, or NULL on failure. */
int sweep_setup(const sweep_desc *desc, sweep_handle **out);

/* Offsets (in doubles) of phi, J, T, beta, Jplus, sphi, sJ, HR inside the packed
 * output, and its total length (an option's offsets equal the next field's offset
 * when the option is off). */
int sweep_layout(const sweep_handle *h, size_t off[8], size_t *total_doubles);

/* One sweep + fused closures, enqueued asynchronously on cuda_stream
 * (a cudaStream_t; NULL = legacy default stream).  Device pointers, borrowed,
 * must stay valid and unmodified until the stream work completes:
 *   d_sigma  [N_el][G_loc]       sigma_t,g per element (piecewise constant)
 *   d_q      [N_el][n][G_loc]    nodal isotropic source q_g (reading R2: no 1/(4 pi))
 *   d_inflow [N_bnode][G_loc]    isotropic inflow per boundary face node (0 = vacuum)
 * inv_c_dt = 1/(c dt) > 0 is added to sigma_t.  Group is the
 * fastest index.  Ends with the in-place NCCL all-reduce when nranks > 1.
 * May be captured into a CUDA graph and replayed (also with new contents of the
 * input buffers): the strip hand-off tags come from a device-side launch counter,
 * not from the host.  Runs of one handle must be stream-ordered (not concurrent). */
int sweep_run(sweep_handle *h, const double *d_sigma, double inv_c_dt, const double *d_q,
              const double *d_inflow, void *cuda_stream);

/* Synchronise cuda_stream, report the device error flag (SWEEP_E_SIGMA), and
 * copy the packed gray output (n_doubles must equal the layout total) to
 * out, which may be device or host memory (cudaMemcpyDefault). */
int closures_get(sweep_handle *h, double *out, size_t n_doubles, void *cuda_stream);

/* End-to-end convenience call with HOST buffers (pinned recommended): copies
 * the inputs host->device into library-owned buffers, runs the sweep, copies
 * the packed output device->host and synchronises.  Same shapes as sweep_run.
 * 2-D: the copy overlaps the sweep -- bands of 8 mesh rows are copied on a
 * library-owned stream from both ends of the mesh inwards, each followed by a
 * stream write of the band's ready flag (cuStreamWriteValue32), and every strip
 * of the sweep kernel waits for the flags of its rows (pinned buffers give the
 * overlap; pageable ones are copied before the launch).  Calls on one handle
 * must be stream-ordered (the staging buffers are reused).  Not capturable into a
 * CUDA graph (it synchronises cuda_stream; the flag generation is a host counter). */
int sweep_run_host(sweep_handle *h, const double *h_sigma, double inv_c_dt, const double *h_q,
                   const double *h_inflow, double *h_out, size_t n_doubles, void *cuda_stream);

/* One backward-Euler step of the UNACCELERATED TRT scheme (
 * SURVEY NEXT-4), the baseline the SM acceleration is measured against:
 *   repeat {  q_g = sigma_g B_g(T) + I^k_g / dt            (emission, eq:smm_be_transport, c = 1)
 *             sweep_run(sigma, 1/dt, q, inflow)           (this handle)
 *             T <- root of C_v (T - T^k)/dt + sum_g sigma_g B_g(T) = sum_g sigma_g phi_g
 *                  at every node (pointwise nonlinear elimination, PAPER.md:588-596;
 *                  bracketed Newton to 1e-15 relative)
 *   } until the paper's relative stopping criterion (eq:relative_tol)
 *       ||u^l - u^{l-1}||_2 < eps ||u^1 - u^0||_2,   u = [T, E]   (paper: eps = 1e-4 for this
 *   scheme), checked after every iteration l >= 2 (after l = 1 only when
 *   u^1 = u^0 exactly), or max_iter iterations.  u^0 is the initial guess on entry:
 *   T^0 = T^k and E^0 = sum_g I^k_g (c = 1, sum_d w_d = 1: the energy density of the
 *   isotropic I^k); E^l = phi of the l-th sweep (c E = phi); the norm
 *   is the 2-norm of the nodal coefficient vectors of T and E together (reading R24).
 * B_g(T) = T^4 [P(nu_{g+1}/T) - P(nu_g/T)], P the normalised Planck integral (a = c = 1).
 * Requires a handle set up with SWEEP_SIGMA_MOMENTS and nranks = 1.
 *   d_sigma [N_el][G], d_inflow [N_bnode][G]  as for sweep_run (sigma at T^k: explicit)
 *   d_Tk    [N_el][n]     nodal temperature at t_k (> 0)
 *   d_Iprev [N_el][n][G]  isotropic intensity at t_k (the time-edge source, reading R17)
 *   d_T     [N_el][n]     output: T^{k+1} (may alias nothing else)
 * *iterations receives the number of outer iterations (sweeps) run.  The gray outputs
 * of the last sweep stay available through closures_get.  Errors: SWEEP_E_ARG (flags,
 * ranks, parameters), SWEEP_E_SIGMA (device flags, incl. a failed elimination). */
typedef struct {
    const double *nu;   /* HOST [G_loc + 1] group bounds, increasing, >= 0 (temperature units) */
    double cv;          /* volumetric heat capacity C_v > 0 */
    double dt;          /* time step > 0 */
    double eps;         /* relative tolerance of the outer iteration; <= 0: run max_iter */
    int max_iter;       /* >= 1 */
    double *ratios;     /* HOST [max_iter] or NULL: receives ||u^l - u^{l-1}||_2 / ||u^1 - u^0||_2
                           for l = 1 .. *iterations (0 when u^1 = u^0) */
} trt_params;

int trt_step(sweep_handle *h, const double *d_sigma, const double *d_inflow, const double *d_Tk,
             const double *d_Iprev, const trt_params *prm, double *d_T, int *iterations, void *cuda_stream);

/* Statistics of the handle and its last sweep_run: out[0] kernels launched by the last
 * sweep_run, out[1] distinct directions swept (after folding), out[2] work streams,
 * out[3] CTAs of the sweep kernel, out[4] threads per CTA, out[5] groups per lane,
 * out[6] lanes per direction, out[7] SMs of the device. */
int sweep_stats(const sweep_handle *h, long long out[8]);

/* Device cross-check of the element solves (a plain register LU kept as a
 * reference variant inside the GPU build): n random element systems in sweep coordinates
 * (sigma~ I + cx A (x) I + cy I (x) A) psi = q + lifts (the lumped weak form of
 * eq:dgsn_transport, in the scaled form of DESIGN.md §4), sigma~ in
 * [0.1, 1e4], cx, cy = |Omega|/h with h = 1/512, each solved on the device both by dense
 * Gaussian elimination of the assembled (p+1)^2 system and by the structured solve of the
 * sweep (p = 1 closed form, p = 2 modal).  *max_rel_err = the largest max-norm relative
 * difference of the nodal solutions.  seed selects the systems (counter-based generator). */
int sweep_selfcheck_solves(int device, int p, int n, unsigned long long seed, double *max_rel_err);

/* Launch-latency floor of the device: back-to-back launches of an empty kernel on one
 * stream, device time per launch in microseconds (the floor the latency-bound configs
 * C1-C3 are reported against). */
int sweep_launch_floor(int device, int reps, double *us_per_launch);

/* Per-run kernel timing (CUDA events recorded on the run's stream around the
 * sweep kernel, the finalize kernel and the all-reduce).  enable != 0 clears
 * and starts recording (ring of the last 1024 runs); 0 stops. */
int sweep_timing(sweep_handle *h, int enable);

/* Durations (ms) of the recorded runs, oldest first: ms[3*r + 0] sweep kernel,
 * [3*r + 1] finalize kernel, [3*r + 2] all-reduce (0 when nranks = 1).
 * Synchronises on the recorded events; *n_runs receives the count (<= max_runs). */
int sweep_kernel_times(sweep_handle *h, double *ms, int max_runs, int *n_runs);

/* Measure the device's FP64 FMA throughput (TFLOP/s) with a dependent-chain-free
 * DFMA kernel on every SM (roofline denominator). */
int sweep_fp64_probe(int device, double *tflops);

/* Fill out128 with a fresh 128-byte ncclUniqueId (rank 0 calls this, then
 * broadcasts it to the other ranks, e.g. with torch.distributed). */
int sweep_nccl_unique_id(void *out128);

/* Free every device and host resource of the handle (and the NCCL comm). */
void sweep_destroy(sweep_handle *h);

/* Message of the last failure on h ("" if none); h may be NULL for setup failures. */
const char *sweep_last_error(const sweep_handle *h);

#ifdef __cplusplus
}
#endif
#endif
