/*
 * sweep_oracle.c — CPU ORACLE for the DG S_N sweep + gray SM closures.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or constant with the CUDA path
 * (paper_2504_21784_b200/csrc), and the CUDA path never calls it.
 *
 * What it computes (PAPER.md, arXiv 2504.21784):
 *   For every direction d and group g, psi_{d,g} in Y_p solving the lumped
 *   upwind-DG weak form of
 *       Omega_d . grad psi + sigma~_g psi = q_g,   sigma~ = sigma_t + 1/(c dt)
 *   (eq:smm_be_transport PAPER.md:219, sigma~ PAPER.md:239; weak form
 *   eq:dgsn_transport PAPER.md:332-336 with the upwind flux PAPER.md:299-327;
 *   every integral evaluated with the tensor Gauss-Lobatto rule).
 *   Each high-order solve "inverts the left hand side only":
 *   q is a given nodal source.  Then the gray sums over d and g
 *       phi = sum w psi              (c E,  PAPER.md:156-158)
 *       J   = sum w Omega psi        (F,    PAPER.md:160-161)
 *       T   = sum w (Omega Omega - I/3) psi
 *       beta = sum w (|Omega.n| - alpha) psi  on boundary face nodes
 *       alpha = sum w |Omega.n| / sum w       (eq:alpha PAPER.md:173-175)
 *       J+  = sum_{Omega.n>0} w (Omega.n) psi on boundary face nodes
 *   Options (opts bit 0): the sigma-weighted gray moments the
 *   gray low-order system takes from the sweep,
 *       sphi = sum_g sigma_g phi_g    (numerator of sigma_E, eq:sigmaE PAPER.md:183-185)
 *       sJ   = sum_g sigma_g J_g      (additive correction sum_g (sigma_F - sigma_g) F_g,
 *                                      eq:additive_mg_correction PAPER.md:197-203, :247)
 *   with sigma_g the opacity WITHOUT the 1/(c dt) pseudo-absorption.
 *   (opts bit 1): the zero-and-scale negative flux fixup inside the
 *   sweep: after each element solve, if a nodal value is
 *   negative, negatives are set to 0 and the rest scaled so the element integral
 *   sum_k W_k psi_k is preserved; a non-positive integral zeroes the element.  The
 *   fixed-up values are what the downwind elements see.
 *   (opts bit 2): the half-range moments of the consistent
 *   low-order method at every node,
 *       F+_n = sum_g sum_{Omega.n > 0} w Omega psi,  P+_n = sum_g sum_{Omega.n > 0} w Omega Omega psi
 *   for n = +x, +y (dim 1: n = +x), with Omega.n = 0 counted as + (reading R23).
 *
 * oracle_trt_step: one backward-Euler step of the UNACCELERATED
 * scheme: repeat { emission source q_g = sigma_g B_g(T) + I^k_g/dt
 * from the current temperature (eq:smm_be_transport; c = 1); sweep;
 * pointwise nonlinear elimination of T from the energy balance
 *     C_v (T - T^k)/dt = sum_g sigma_g (phi_g - B_g(T))   (eq:smm_be_meb)
 * } until the paper's relative stopping criterion (eq:relative_tol,
 * PAPER.md:657-660; eps = 1e-4 for the unaccelerated scheme)
 *     ||u^{l+1} - u^l||_2 < eps ||u^1 - u^0||_2,   u = [T, E]
 * with u^0 the initial guess on entry (T^0 = T^k, E^0 = E^k = sum_g I^k_g: c = 1 and
 * sum_d w_d = 1, so the energy density of the isotropic I^k is its group sum) and
 * E^l = phi^l = sum_g sum_d w_d psi (c E = phi) of the l-th sweep;
 * the 2-norm is over the nodal coefficient vectors of T and E (reading R24).
 * B_g(T) = T^4 [P(nu_{g+1}/T) - P(nu_g/T)], P(x) = (15/pi^4) int_0^x t^3/(e^t-1) dt
 * (eq:planck PAPER.md:106-125, a = c = 1) evaluated here by composite Gauss-Legendre
 * quadrature of the integrand (no series), and T found by bisection (no Newton).
 *
 * How (deliberately plain): for each (d,g), elements are visited in upwind
 * nested-loop order; the element matrix is assembled UNSCALED straight from
 * the weak form and solved with partial-pivot LU; contributions are summed
 * with Neumaier compensation.  No closed forms, no Kronecker structure.
 *
 * Readings of the paper: R1 GLL nodal basis of order p with the
 * collocated (p+1)-point GLL rule for p = 2; R2 nodal source; R3 sum w = 1, no
 * 1/(4 pi); R4 T components xx (1-D) or xx,xy,yy (2-D); R5 beta/J+ from the
 * element's own nodal trace for every direction; R6 alpha per normal;
 * R15 Omega.n = 0 gives no face term.
 *
 * Parity pins: tests/test_oracle_pins.py (dense global assembly in the
 * jump/average form, closed-form 1-D transmission, constant-solution
 * exactness, particle balance, convergence order, symmetries).
 */
#define _GNU_SOURCE
#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define MAXN 9   /* (p+1)^dim <= 9 */

/* ---- reference element: GLL nodes/weights on [0,1] and D_ab = l_b'(xi_a) ---- */
typedef struct {
    int p, np1;
    double xi[3], wh[3];
    double D[3][3];
} refel;

static int make_refel(int p, refel *R) {
    if (p == 1) {
        R->xi[0] = 0.0; R->xi[1] = 1.0;
        R->wh[0] = 0.5; R->wh[1] = 0.5;
    } else if (p == 2) {
        R->xi[0] = 0.0; R->xi[1] = 0.5; R->xi[2] = 1.0;
        R->wh[0] = 1.0 / 6.0; R->wh[1] = 2.0 / 3.0; R->wh[2] = 1.0 / 6.0;
    } else {
        return -1;
    }
    R->p = p; R->np1 = p + 1;
    /* derivative of the Lagrange basis l_b at node xi_a, from its definition */
    for (int a = 0; a <= p; ++a)
        for (int b = 0; b <= p; ++b) {
            double s = 0.0;
            for (int m = 0; m <= p; ++m) {
                if (m == b) continue;
                double term = 1.0 / (R->xi[b] - R->xi[m]);
                for (int l = 0; l <= p; ++l) {
                    if (l == b || l == m) continue;
                    term *= (R->xi[a] - R->xi[l]) / (R->xi[b] - R->xi[l]);
                }
                s += term;
            }
            R->D[a][b] = s;
        }
    return 0;
}

/* ---- problem ---- */
typedef struct {
    int dim, nx, ny, p, n, np1, ndir, G, nbnode;
    double hx, hy;
    const double *omega, *w, *sigma, *q, *inflow;
    double inv_c_dt;
    refel R;
} prob;

static int bnode(const prob *P, int face, int idx, int node) {
    /* face 0:x- 1:x+ 2:y- 3:y+ ; idx = j (x faces) or i (y faces); node = b or a */
    if (P->dim == 1) return face;  /* [x=0, x=1] */
    int np1 = P->np1;
    switch (face) {
        case 0: return idx * np1 + node;
        case 1: return P->ny * np1 + idx * np1 + node;
        case 2: return 2 * P->ny * np1 + idx * np1 + node;
        default: return 2 * P->ny * np1 + P->nx * np1 + idx * np1 + node;
    }
}

/* Solve A x = r (n x n, row-major, destroyed) by LU with partial pivoting. */
static int lu_solve(int n, double *A, double *r, double *x) {
    int piv[MAXN];
    for (int k = 0; k < n; ++k) piv[k] = k;
    for (int k = 0; k < n; ++k) {
        int pr = k;
        double best = fabs(A[k * n + k]);
        for (int i = k + 1; i < n; ++i)
            if (fabs(A[i * n + k]) > best) { best = fabs(A[i * n + k]); pr = i; }
        if (best == 0.0) return -1;
        if (pr != k) {
            for (int j = 0; j < n; ++j) { double t = A[k * n + j]; A[k * n + j] = A[pr * n + j]; A[pr * n + j] = t; }
            double t = r[k]; r[k] = r[pr]; r[pr] = t;
        }
        for (int i = k + 1; i < n; ++i) {
            double f = A[i * n + k] / A[k * n + k];
            A[i * n + k] = 0.0;
            for (int j = k + 1; j < n; ++j) A[i * n + j] -= f * A[k * n + j];
            r[i] -= f * r[k];
        }
    }
    for (int i = n - 1; i >= 0; --i) {
        double s = r[i];
        for (int j = i + 1; j < n; ++j) s -= A[i * n + j] * x[j];
        x[i] = s / A[i * n + i];
    }
    return 0;
}

/*
 * Zero-and-scale fixup of one element's nodal values x[n] with lumped-mass
 * weights W[n] ("zero and scale negative flux fixup ... preserving
 * particle balance"; reading F1 in DESIGN.md: the preserved quantity is the
 * element integral sum_k W_k x_k).  Returns 1 if x was changed.
 */
int oracle_fixup(int n, const double *W, double *x) {
    int neg = 0;
    for (int k = 0; k < n; ++k)
        if (x[k] < 0.0) neg = 1;
    if (!neg) return 0;
    double total = 0.0, pos = 0.0;
    for (int k = 0; k < n; ++k) {
        total += W[k] * x[k];
        if (x[k] > 0.0) pos += W[k] * x[k];
    }
    if (total <= 0.0) {
        for (int k = 0; k < n; ++k) x[k] = 0.0;
        return 1;
    }
    const double scale = total / pos;
    for (int k = 0; k < n; ++k) x[k] = (x[k] > 0.0) ? x[k] * scale : 0.0;
    return 1;
}

/*
 * One (d,g) sweep.  psi [N_el][n].  Returns 0, or -1 on a singular block.
 * Weak form per element K, test function l_k (eq:dgsn_transport with the
 * upwind flux):
 *   - int_K Omega.grad(l_k) psi + sum_faces int_f (Omega.n) l_k psi^ + int_K sigma~ l_k psi = int_K l_k q
 * psi^ = own trace on outflow faces (Omega.n > 0), the upwind neighbour's
 * coincident trace or the prescribed inflow on inflow faces (Omega.n < 0).
 * GLL lumping: int_K f = sum_l W_l f(x_l), W_l = hx hy wh_a wh_b;
 * int_f f = sum over face nodes of (face weight) f; grad l_k at node l =
 * (D_{a_l a_k}/hx delta_{b_k b_l}, D_{b_l b_k}/hy delta_{a_k a_l}).
 */
static int sweep_dg(const prob *P, int d, int g, double *psi, int fixup) {
    const int nx = P->nx, ny = P->ny, np1 = P->np1, n = P->n, G = P->G;
    const double ox = P->omega[3 * d + 0], oy = (P->dim == 2) ? P->omega[3 * d + 1] : 0.0;
    const double hx = P->hx, hy = P->hy;
    const refel *R = &P->R;
    const int i0 = (ox >= 0.0) ? 0 : nx - 1, di = (ox >= 0.0) ? 1 : -1;
    const int j0 = (oy >= 0.0) ? 0 : ny - 1, dj = (oy >= 0.0) ? 1 : -1;
    double A[MAXN * MAXN], r[MAXN], x[MAXN];
    double W[MAXN];
    int ak[MAXN], bk[MAXN];
    for (int k = 0; k < n; ++k) {
        ak[k] = k % np1;
        bk[k] = (P->dim == 2) ? k / np1 : 0;
        W[k] = (P->dim == 2) ? hx * hy * R->wh[ak[k]] * R->wh[bk[k]] : hx * R->wh[ak[k]];
    }
    for (int jj = 0; jj < ny; ++jj) {
        const int j = j0 + dj * jj;
        for (int ii = 0; ii < nx; ++ii) {
            const int i = i0 + di * ii;
            const int e = i + nx * j;
            const double sig_t = P->sigma[(size_t)e * G + g] + P->inv_c_dt;
            memset(A, 0, sizeof(A));
            for (int k = 0; k < n; ++k) {
                /* mass: int sigma~ l_k psi ;  source: int l_k q */
                A[k * n + k] += sig_t * W[k];
                r[k] = W[k] * P->q[((size_t)e * n + k) * G + g];
                /* streaming: - int Omega.grad(l_k) psi = - sum_l W_l Omega.grad l_k(x_l) psi_l */
                for (int l = 0; l < n; ++l) {
                    double gx = (bk[k] == bk[l]) ? R->D[ak[l]][ak[k]] / hx : 0.0;
                    double gy = (P->dim == 2 && ak[k] == ak[l]) ? R->D[bk[l]][bk[k]] / hy : 0.0;
                    A[k * n + l] -= W[l] * (ox * gx + oy * gy);
                }
            }
            /* faces: (normal component, node-on-face test, face weight, upwind value) */
            const int nfaces = (P->dim == 2) ? 4 : 2;
            for (int f = 0; f < nfaces; ++f) {
                double on;  /* Omega . n_f */
                switch (f) {
                    case 0: on = -ox; break;
                    case 1: on = ox; break;
                    case 2: on = -oy; break;
                    default: on = oy; break;
                }
                if (on == 0.0) continue;  /* R15: no face term */
                for (int k = 0; k < n; ++k) {
                    int onface;
                    double wf;
                    switch (f) {
                        case 0: onface = (ak[k] == 0); wf = (P->dim == 2) ? hy * R->wh[bk[k]] : 1.0; break;
                        case 1: onface = (ak[k] == np1 - 1); wf = (P->dim == 2) ? hy * R->wh[bk[k]] : 1.0; break;
                        case 2: onface = (bk[k] == 0); wf = hx * R->wh[ak[k]]; break;
                        default: onface = (bk[k] == np1 - 1); wf = hx * R->wh[ak[k]]; break;
                    }
                    if (!onface) continue;
                    if (on > 0.0) {
                        A[k * n + k] += on * wf;  /* outflow: own trace */
                    } else {
                        double up;
                        int ni = i, nj = j, nk;
                        switch (f) {
                            case 0: ni = i - 1; nk = (np1 - 1) + np1 * bk[k]; break;
                            case 1: ni = i + 1; nk = 0 + np1 * bk[k]; break;
                            case 2: nj = j - 1; nk = ak[k] + np1 * (np1 - 1); break;
                            default: nj = j + 1; nk = ak[k]; break;
                        }
                        if (ni < 0 || ni >= nx || nj < 0 || nj >= ny) {
                            int idx = (f < 2) ? j : i;
                            int node = (f < 2) ? bk[k] : ak[k];
                            up = P->inflow[(size_t)bnode(P, f, idx, node) * G + g];
                        } else {
                            if (P->dim == 1) nk = (f == 0) ? np1 - 1 : 0;
                            up = psi[(size_t)(ni + nx * nj) * n + nk];
                        }
                        r[k] += (-on) * wf * up;  /* inflow: upwind trace */
                    }
                }
            }
            if (lu_solve(n, A, r, x) != 0) return -1;
            if (fixup) oracle_fixup(n, W, x);
            for (int k = 0; k < n; ++k) psi[(size_t)e * n + k] = x[k];
        }
    }
    return 0;
}

/* ---- Neumaier-compensated accumulator ---- */
static inline void nadd(double *s, double *c, double v) {
    double t = *s + v;
    if (fabs(*s) >= fabs(v)) *c += (*s - t) + v;
    else *c += (v - t) + *s;
    *s = t;
}

static int setup(prob *P, int dim, int nx, int ny, double lx, double ly, int p, int ndir,
                 const double *omega, const double *w, int G, const double *sigma, double inv_c_dt,
                 const double *q, const double *inflow) {
    if (dim != 1 && dim != 2) return -2;
    if (make_refel(p, &P->R) != 0) return -2;
    if (nx <= 0 || (dim == 2 && ny <= 0) || ndir <= 0 || G <= 0 || lx <= 0.0) return -2;
    P->dim = dim; P->nx = nx; P->ny = (dim == 2) ? ny : 1; P->p = p; P->np1 = p + 1;
    P->n = (dim == 2) ? (p + 1) * (p + 1) : p + 1;
    P->ndir = ndir; P->G = G;
    P->nbnode = (dim == 1) ? 2 : 2 * (nx + ny) * (p + 1);
    P->hx = lx / nx; P->hy = (dim == 2) ? ly / ny : 1.0;
    P->omega = omega; P->w = w; P->sigma = sigma; P->q = q; P->inflow = inflow;
    P->inv_c_dt = inv_c_dt;
    return 0;
}

/* number of output doubles: phi, J(dim), T(1 or 3) per node; beta, J+ per boundary
 * node; with opts bit 0 also sphi, sJ(dim) per node */
static size_t out_size(const prob *P, size_t *nodes, int *nT, int opts) {
    *nodes = (size_t)P->nx * P->ny * P->n;
    *nT = (P->dim == 1) ? 1 : 3;
    return (*nodes) * (1 + P->dim + *nT) + 2 * (size_t)P->nbnode + ((opts & 1) ? (*nodes) * (1 + P->dim) : 0) +
           ((opts & 4) ? (*nodes) * (P->dim == 2 ? 10 : 2) : 0);
}

int oracle_out_size2(int dim, int nx, int ny, int p, int opts) {
    int n = (dim == 2) ? (p + 1) * (p + 1) : p + 1;
    int nel = (dim == 2) ? nx * ny : nx;
    int nT = (dim == 1) ? 1 : 3;
    int nb = (dim == 1) ? 2 : 2 * (nx + ny) * (p + 1);
    return nel * n * (1 + dim + nT) + 2 * nb + ((opts & 1) ? nel * n * (1 + dim) : 0) +
           ((opts & 4) ? nel * n * (dim == 2 ? 10 : 2) : 0);
}

int oracle_out_size(int dim, int nx, int ny, int p) { return oracle_out_size2(dim, nx, ny, p, 0); }

/* alpha_n = sum_d w_d |Omega_d . n| / sum_d w_d for n in {x-, x+, y-, y+} (eq:alpha) */
void oracle_alpha(int dim, int ndir, const double *omega, const double *w, double *alpha4) {
    double sw = 0.0, sx = 0.0, sy = 0.0;
    for (int d = 0; d < ndir; ++d) {
        sw += w[d];
        sx += w[d] * fabs(omega[3 * d]);
        sy += w[d] * ((dim == 2) ? fabs(omega[3 * d + 1]) : 0.0);
    }
    alpha4[0] = alpha4[1] = sx / sw;
    alpha4[2] = alpha4[3] = sy / sw;
}

/* psi for a single (d,g): psi_out [N_el][n].  0 = ok. */
int oracle_sweep_psi(int dim, int nx, int ny, double lx, double ly, int p, int ndir,
                     const double *omega, const double *w, int G, const double *sigma,
                     double inv_c_dt, const double *q, const double *inflow, int d, int g,
                     double *psi_out, int opts) {
    prob P;
    int rc = setup(&P, dim, nx, ny, lx, ly, p, ndir, omega, w, G, sigma, inv_c_dt, q, inflow);
    if (rc) return rc;
    if (d < 0 || d >= ndir || g < 0 || g >= G) return -2;
    return sweep_dg(&P, d, g, psi_out, (opts >> 1) & 1);
}

/*
 * Full sweep + gray moments.  out layout (packed, as the C-ABI's closures_get):
 *   phi[N_el][n] | J[dim][N_el][n] | T[nT][N_el][n] | beta[N_bnode] | Jplus[N_bnode]
 *   [ | sphi[N_el][n] | sJ[dim][N_el][n]   when opts bit 0 ]
 * opts bit 1: zero-and-scale fixup inside the sweep.
 * nthreads <= 0: OpenMP default.  Returns 0, -1 singular block, -2 bad args, -3 OOM.
 */
int oracle_sweep2(int dim, int nx, int ny, double lx, double ly, int p, int ndir,
                  const double *omega, const double *w, int G, const double *sigma,
                  double inv_c_dt, const double *q, const double *inflow, double *out,
                  int nthreads, int opts) {
    prob P;
    int rc = setup(&P, dim, nx, ny, lx, ly, p, ndir, omega, w, G, sigma, inv_c_dt, q, inflow);
    if (rc) return rc;
    size_t nodes;
    int nT;
    const size_t nout = out_size(&P, &nodes, &nT, opts);
    const int ncomp = 1 + dim + nT;
    const int sig_mom = opts & 1, fixup = (opts >> 1) & 1;
    const size_t off_sig = (size_t)ncomp * nodes + 2 * (size_t)P.nbnode;  /* sphi, then sJ */
    const int half = (opts >> 2) & 1;
    const size_t off_hr = off_sig + (sig_mom ? (size_t)(1 + dim) * nodes : 0);

    /* per-direction closure coefficients, precomputed as w (Omega Omega - I/3) (R16) */
    double *coef = (double *)malloc(sizeof(double) * (size_t)ndir * 6);
    if (!coef) return -3;
    for (int d = 0; d < ndir; ++d) {
        const double wd = w[d], ox = omega[3 * d], oy = (dim == 2) ? omega[3 * d + 1] : 0.0;
        double *c = coef + 6 * d;
        c[0] = wd;
        if (dim == 1) {
            c[1] = wd * ox;
            c[2] = wd * (ox * ox - 1.0 / 3.0);
        } else {
            c[1] = wd * ox;
            c[2] = wd * oy;
            c[3] = wd * (ox * ox - 1.0 / 3.0);
            c[4] = wd * (ox * oy);
            c[5] = wd * (oy * oy - 1.0 / 3.0);
        }
    }
    double alpha4[4];
    oracle_alpha(dim, ndir, omega, w, alpha4);

    /* boundary face nodes: element, node, face */
    const int nb = P.nbnode;
    int *b_el = (int *)malloc(sizeof(int) * nb), *b_k = (int *)malloc(sizeof(int) * nb), *b_f = (int *)malloc(sizeof(int) * nb);
    if (!b_el || !b_k || !b_f) { free(coef); free(b_el); free(b_k); free(b_f); return -3; }
    if (dim == 1) {
        b_el[0] = 0; b_k[0] = 0; b_f[0] = 0;
        b_el[1] = nx - 1; b_k[1] = P.np1 - 1; b_f[1] = 1;
    } else {
        const int np1 = P.np1;
        for (int j = 0; j < P.ny; ++j)
            for (int b = 0; b < np1; ++b) {
                int t = bnode(&P, 0, j, b); b_el[t] = 0 + nx * j; b_k[t] = 0 + np1 * b; b_f[t] = 0;
                t = bnode(&P, 1, j, b); b_el[t] = (nx - 1) + nx * j; b_k[t] = (np1 - 1) + np1 * b; b_f[t] = 1;
            }
        for (int i = 0; i < nx; ++i)
            for (int a = 0; a < np1; ++a) {
                int t = bnode(&P, 2, i, a); b_el[t] = i; b_k[t] = a; b_f[t] = 2;
                t = bnode(&P, 3, i, a); b_el[t] = i + nx * (P.ny - 1); b_k[t] = a + np1 * (np1 - 1); b_f[t] = 3;
            }
    }

    int nth = 1;
#ifdef _OPENMP
    nth = (nthreads > 0) ? nthreads : omp_get_max_threads();
#endif
    const long npairs = (long)ndir * G;
    if (nth > npairs) nth = (int)npairs;
    if (nth < 1) nth = 1;
    double *acc = (double *)calloc((size_t)nth * nout * 2, sizeof(double));
    if (!acc) { free(coef); free(b_el); free(b_k); free(b_f); return -3; }
    int fail = 0;

#pragma omp parallel num_threads(nth)
    {
        int tid = 0;
#ifdef _OPENMP
        tid = omp_get_thread_num();
#endif
        double *S = acc + (size_t)tid * nout * 2;  /* sums */
        double *C = S + nout;                      /* compensations */
        double *psi = (double *)malloc(sizeof(double) * nodes);
        if (!psi) {
#pragma omp atomic write
            fail = -3;
        }
#pragma omp for schedule(static)
        for (long pr = 0; pr < npairs; ++pr) {
            if (!psi) continue;
            const int d = (int)(pr / G), g = (int)(pr % G);
            if (sweep_dg(&P, d, g, psi, fixup) != 0) {
#pragma omp atomic write
                fail = -1;
                continue;
            }
            const double *c = coef + 6 * d;
            for (size_t v = 0; v < nodes; ++v) {
                const double ps = psi[v];
                for (int m = 0; m < ncomp; ++m) nadd(&S[m * nodes + v], &C[m * nodes + v], c[m] * ps);
            }
            if (half) {
                /* half-range moments: directions with Omega_x >= 0 (rows 0-4), Omega_y >= 0 (rows 5-9);
                 * dim 1: mu >= 0 (rows 0-1) */
                const double ox = omega[3 * d], oy = (dim == 2) ? omega[3 * d + 1] : 0.0, wd = w[d];
                double row[10];
                int nrow;
                if (dim == 2) {
                    const double vx[5] = {wd * ox, wd * oy, wd * ox * ox, wd * ox * oy, wd * oy * oy};
                    for (int m = 0; m < 5; ++m) {
                        row[m] = (ox >= 0.0) ? vx[m] : 0.0;
                        row[5 + m] = (oy >= 0.0) ? vx[m] : 0.0;
                    }
                    nrow = 10;
                } else {
                    row[0] = (ox >= 0.0) ? wd * ox : 0.0;
                    row[1] = (ox >= 0.0) ? wd * ox * ox : 0.0;
                    nrow = 2;
                }
                for (size_t v = 0; v < nodes; ++v) {
                    const double ps = psi[v];
                    for (int m = 0; m < nrow; ++m) {
                        if (row[m] == 0.0) continue;
                        const size_t o = off_hr + m * nodes + v;
                        nadd(&S[o], &C[o], row[m] * ps);
                    }
                }
            }
            if (sig_mom) {
                /* sum_g sigma_g (w, w Omega) psi: sigma_g of the node's element, no 1/(c dt) */
                for (size_t v = 0; v < nodes; ++v) {
                    const double sg = P.sigma[(v / P.n) * G + g];
                    const double ps = psi[v];
                    for (int m = 0; m <= dim; ++m) {
                        const size_t o = off_sig + m * nodes + v;
                        nadd(&S[o], &C[o], sg * (c[m] * ps));
                    }
                }
            }
            const double ox = omega[3 * d], oy = (dim == 2) ? omega[3 * d + 1] : 0.0;
            for (int t = 0; t < nb; ++t) {
                double on;
                switch (b_f[t]) {
                    case 0: on = -ox; break;
                    case 1: on = ox; break;
                    case 2: on = -oy; break;
                    default: on = oy; break;
                }
                const double ps = psi[(size_t)b_el[t] * P.n + b_k[t]];
                const size_t ib = (size_t)ncomp * nodes + t, ij = ib + nb;
                nadd(&S[ib], &C[ib], w[d] * (fabs(on) - alpha4[b_f[t]]) * ps);
                if (on > 0.0) nadd(&S[ij], &C[ij], w[d] * on * ps);
            }
        }
        free(psi);
    }
    if (!fail) {
        for (size_t v = 0; v < nout; ++v) {
            double s = 0.0, c = 0.0;
            for (int t = 0; t < nth; ++t) {
                const double *S = acc + (size_t)t * nout * 2;
                nadd(&s, &c, S[v]);
                nadd(&s, &c, S[nout + v]);
            }
            out[v] = s + c;
        }
    }
    free(acc); free(coef); free(b_el); free(b_k); free(b_f);
    return fail;
}

int oracle_sweep(int dim, int nx, int ny, double lx, double ly, int p, int ndir,
                 const double *omega, const double *w, int G, const double *sigma,
                 double inv_c_dt, const double *q, const double *inflow, double *out,
                 int nthreads) {
    return oracle_sweep2(dim, nx, ny, lx, ly, p, ndir, omega, w, G, sigma, inv_c_dt, q, inflow, out, nthreads, 0);
}

/* ---------------------------------------------------------------- NEXT-4 */
/* 20-point Gauss-Legendre rule on [-1,1], nodes found by Newton on P_20 */
static double gl_x[20], gl_w[20];
static int gl_ready = 0;
static void gl_init(void) {
    if (gl_ready) return;
    const int n = 20;
    for (int i = 0; i < n; ++i) {
        double x = cos(M_PI * (i + 0.75) / (n + 0.5));
        for (int it = 0; it < 100; ++it) {
            double p0 = 1.0, p1 = x;
            for (int k = 2; k <= n; ++k) {
                double p2 = ((2.0 * k - 1.0) * x * p1 - (k - 1.0) * p0) / k;
                p0 = p1;
                p1 = p2;
            }
            double dp = n * (x * p1 - p0) / (x * x - 1.0);
            double dx = p1 / dp;
            x -= dx;
            if (fabs(dx) < 1e-16) {
                p0 = 1.0; p1 = x;
                for (int k = 2; k <= n; ++k) {
                    double p2 = ((2.0 * k - 1.0) * x * p1 - (k - 1.0) * p0) / k;
                    p0 = p1;
                    p1 = p2;
                }
                dp = n * (x * p1 - p0) / (x * x - 1.0);
                break;
            }
        }
        gl_x[i] = x;
        double p0 = 1.0, p1 = x;
        for (int k = 2; k <= n; ++k) {
            double p2 = ((2.0 * k - 1.0) * x * p1 - (k - 1.0) * p0) / k;
            p0 = p1;
            p1 = p2;
        }
        double dp = n * (x * p1 - p0) / (x * x - 1.0);
        gl_w[i] = 2.0 / ((1.0 - x * x) * dp * dp);
    }
    gl_ready = 1;
}

static double planck_integrand(double t) { return (t < 1e-300) ? 0.0 : t * t * t / expm1(t); }

/* P(x) = (15/pi^4) int_0^x t^3/(e^t-1) dt, composite 20-point Gauss-Legendre on unit
 * panels up to min(x, 60) (the tail beyond 60 is < 1e-20 of the total). */
double oracle_planck_P(double x) {
    if (!(x > 0.0)) return 0.0;
    gl_init();
    const double X = (x < 60.0) ? x : 60.0;
    const int np = (int)ceil(X);
    double s = 0.0;
    for (int k = 0; k < np; ++k) {
        const double a = X * k / np, b = X * (k + 1) / np, m = 0.5 * (a + b), hw = 0.5 * (b - a);
        double ps = 0.0;
        for (int i = 0; i < 20; ++i) ps += gl_w[i] * planck_integrand(m + hw * gl_x[i]);
        s += hw * ps;
    }
    return s * 15.0 / (M_PI * M_PI * M_PI * M_PI);
}

/* B_g(T) for g = 0..G-1 from the bounds nu[0..G] */
static void planck_groups_T(double T, int G, const double *nu, double *Bg) {
    const double T4 = T * T * T * T;
    double Pl = oracle_planck_P(nu[0] / T);
    for (int g = 0; g < G; ++g) {
        const double Pr = oracle_planck_P(nu[g + 1] / T);
        Bg[g] = T4 * (Pr - Pl);
        Pl = Pr;
    }
}

void oracle_planck_groups(double T, int G, const double *nu, double *Bg) { planck_groups_T(T, G, nu, Bg); }

/* nonlinear elimination at one node: f(T) = cv/dt (T - Tk) + sum_g sig_g B_g(T) - sphi = 0,
 * f increasing in T >= 0; bisection to relative width 1e-15 */
double oracle_t_eliminate(double Tk, double sphi, int G, const double *sig, const double *nu, double cv_dt) {
    double Bg[512];
    if (G > 512) return -1.0;
    #define F_OF(T, out) do { planck_groups_T((T), G, nu, Bg); double e_ = 0.0; \
        for (int g_ = 0; g_ < G; ++g_) e_ += sig[g_] * Bg[g_]; (out) = cv_dt * ((T) - Tk) + e_ - sphi; } while (0)
    double lo = 0.0, hi = (Tk > 1.0) ? Tk : 1.0, fh;
    F_OF(hi, fh);
    while (fh < 0.0) { lo = hi; hi *= 2.0; F_OF(hi, fh); }
    while (hi - lo > 1e-15 * hi) {
        const double mid = 0.5 * (lo + hi);
        double fm;
        F_OF(mid, fm);
        if (fm < 0.0) lo = mid; else hi = mid;
        if (mid == lo && mid == hi) break;
    }
    #undef F_OF
    return 0.5 * (lo + hi);
}

/* One unaccelerated backward-Euler step.  Tk, T [N_el][n] nodal; Iprev [N_el][n][G]
 * isotropic previous intensity; sigma [N_el][G]; inflow [N_bnode][G]; nu [G+1].
 * c = 1: 1/(c dt) = 1/dt.  Iteration l = 1, 2, ...: u^l = [T^l, E^l]; stops after the
 * first iteration l >= 2 with ||u^l - u^{l-1}||_2 < eps ||u^1 - u^0||_2 (eq:relative_tol,
 * PAPER.md:657-660), or after iteration 1 when ||u^1 - u^0||_2 = 0 (u^0 is already the
 * fixed point), or after max_iter iterations; eps <= 0 runs max_iter.  ratio (may be
 * NULL) receives ||u^l - u^{l-1}||_2 / ||u^1 - u^0||_2 for l = 1..iterations.
 * Returns the iteration count, or < 0 on failure. */
int oracle_trt_step(int dim, int nx, int ny, double lx, double ly, int p, int ndir, const double *omega,
                    const double *w, int G, const double *sigma, const double *inflow, const double *Tk,
                    const double *Iprev, const double *nu, double cv, double dt, double eps, int max_iter,
                    double *T, double *ratio, int nthreads) {
    prob P;
    int rc = setup(&P, dim, nx, ny, lx, ly, p, ndir, omega, w, G, sigma, 1.0 / dt, Iprev, inflow);
    if (rc) return rc;
    size_t nodes;
    int nT;
    const size_t nout = out_size(&P, &nodes, &nT, 1);
    const size_t off_sig = (size_t)(1 + dim + nT) * nodes + 2 * (size_t)P.nbnode;
    double *q = (double *)malloc(sizeof(double) * nodes * G);
    double *out = (double *)malloc(sizeof(double) * nout);
    double *Tn = (double *)malloc(sizeof(double) * nodes);
    double *E = (double *)malloc(sizeof(double) * nodes);
    double *Bg = (double *)malloc(sizeof(double) * G);
    if (!q || !out || !Tn || !E || !Bg) { free(q); free(out); free(Tn); free(E); free(Bg); return -3; }
    for (size_t v = 0; v < nodes; ++v) {
        T[v] = Tk[v];
        double e = 0.0;                 /* E^0 = sum_g I^k_g (isotropic, sum_d w_d = 1) */
        for (int g = 0; g < G; ++g) e += Iprev[v * G + g];
        E[v] = e;
    }
    double first = 0.0;                 /* ||u^1 - u^0||_2 */
    int it = 0;
    for (it = 1; it <= max_iter; ++it) {
        for (size_t v = 0; v < nodes; ++v) {
            const size_t e = v / P.n;
            planck_groups_T(T[v], G, nu, Bg);
            for (int g = 0; g < G; ++g) q[v * G + g] = sigma[e * G + g] * Bg[g] + Iprev[v * G + g] / dt;
        }
        rc = oracle_sweep2(dim, nx, ny, lx, ly, p, ndir, omega, w, G, sigma, 1.0 / dt, q, inflow, out, nthreads, 1);
        if (rc) break;
        double du = 0.0;                /* ||u^it - u^(it-1)||_2^2 over T and E = phi */
        for (size_t v = 0; v < nodes; ++v) {
            const size_t e = v / P.n;
            Tn[v] = oracle_t_eliminate(Tk[v], out[off_sig + v], G, sigma + e * G, nu, cv / dt);
            du += (Tn[v] - T[v]) * (Tn[v] - T[v]);
            du += (out[v] - E[v]) * (out[v] - E[v]);
        }
        for (size_t v = 0; v < nodes; ++v) {
            T[v] = Tn[v];
            E[v] = out[v];
        }
        const double dn = sqrt(du);
        if (it == 1) first = dn;
        if (ratio) ratio[it - 1] = (first > 0.0) ? dn / first : 0.0;
        if (eps > 0.0 && (first == 0.0 || (it >= 2 && dn < eps * first))) break;
    }
    if (it > max_iter) it = max_iter;
    free(q); free(out); free(Tn); free(E); free(Bg);
    return rc ? rc : it;
}
