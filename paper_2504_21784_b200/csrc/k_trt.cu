// k_trt.cu — the UNACCELERATED TRT iteration around the sweep (
// PAPER.md:667-672): emission source from the current temperature, and the pointwise
// nonlinear elimination of the temperature from the energy balance
//     C_v (T - T^k)/dt + sum_g sigma_g B_g(T) = sum_g sigma_g phi_g   (eq:smm_be_meb, c = 1)
// with sum_g sigma_g phi_g the sweep's sigma-weighted moment (SWEEP_SIGMA_MOMENTS).
// B_g(T) = T^4 [P(nu_{g+1}/T) - P(nu_g/T)], P(x) = (15/pi^4) int_0^x t^3/(e^t-1) dt
// (eq:planck PAPER.md:106-125, a = c = 1), evaluated with the two classical series of
// the Planck integral ("polylogarithmic and Taylor series expansions").
#include <cuda_runtime.h>

#include "sweep_internal.h"

namespace sweepk {


constexpr double K15_PI4 = 0.15398973382026503;  // 15 / pi^4

// int_0^x t^3/(e^t-1) dt * 15/pi^4, its derivative (15/pi^4) x^3/(e^x-1) and 1/(e^x-1)
__device__ __forceinline__ void planck_P(double x, double& P, double& dP, double& rem1) {
    if (!(x > 0.0)) {
        P = 0.0;
        dP = 0.0;
        rem1 = 0.0;
        return;
    }
    const double x2 = x * x, x3 = x2 * x;
    rem1 = 1.0 / expm1(x);
    dP = K15_PI4 * x3 * rem1;
    if (x < 3.0) {
        // Bernoulli series sum_k B_k x^(k+3) / (k! (k+3)) (|x| < 2 pi): x^3/3 - x^4/8 +
        // sum_j c_j x^(2j+3), c_j = B_2j / ((2j)! (2j+3)), j = 1..25 (Horner in x^2; the
        // j = 25 term is below 1e-16 of the sum at x = 3).  Exact Bernoulli numbers,
        // rounded once to double (hex literals).  The switch at x = 3 (not 1.5) cuts the
        // tail loop below from 27 to 14 terms; a warp's lanes straddle the switch, so
        // both branches are paid.
        constexpr double c[26] = {1.0 / 3.0,
                                  0x1.1111111111111p-6,  -0x1.a01a01a01a01ap-13, 0x1.ed284dc73b445p-19,
                                  -0x1.42cb40df7f3abp-24, 0x1.b96d79892884cp-30, -0x1.35de417c02910p-35,
                                  0x1.bb28a22b53d89p-41,  -0x1.41626d7230484p-46, 0x1.d762338fbb4bfp-52,
                                  -0x1.5cdcee4b98370p-57, 0x1.0427c1f1c4c70p-62, -0x1.8681da5029235p-68,
                                  0x1.26b40ee19058bp-73,  -0x1.beeea26d5ca6ap-79, 0x1.5450579047e7ap-84,
                                  -0x1.0415d3bd22f20p-89, 0x1.8ed7e280fa8fbp-95, -0x1.32b61253f8daap-100,
                                  0x1.d8f77f88e815cp-106, -0x1.6d8a89aff8a6ap-111, 0x1.1b20b5bdfa81ap-116,
                                  -0x1.b7753eeb0a071p-122, 0x1.55ac07fbb064ep-127, -0x1.0a1690e38bf07p-132,
                                  0x1.9f1680b3fee0ep-138};
        double s = c[25];
#pragma unroll
        for (int j = 24; j >= 1; --j) s = fma(s, x2, c[j]);
        // sum = x^3 [1/3 - x/8 + x^2 (c1 + x^2 (c2 + ...))]
        P = K15_PI4 * x3 * (c[0] - x * 0.125 + s * x2);
    } else {
        // 1 - (15/pi^4) sum_n e^{-n x} (x^3/n + 3x^2/n^2 + 6x/n^3 + 6/n^4); terms until
        // e^{-n x} < e^{-38} (x >= 3: at most 14), 1/n from an unrolled table
        double tail = 0.0;
        const double e1 = exp(-x);
        double en = 1.0;
        const int nmax = (int)(38.0 / x) + 2;
        const double x6 = 6.0 * x, x23 = 3.0 * x2;
#pragma unroll
        for (int n = 1; n <= 14; ++n) {
            if (n > nmax) break;
            const double rn = 1.0 / (double)n;  // folded to a constant (unrolled)
            en *= e1;
            tail = fma(en * rn, fma(rn, fma(rn, fma(6.0, rn, x6), x23), x3), tail);
        }
        P = 1.0 - K15_PI4 * tail;
    }
}

// q[v][g] = sigma[e][g] B_g(T[v]) + Iprev[v][g] * inv_dt   (v = e*n + k).  The (node,
// bound) pairs are laid out flat, G + 1 slots per node; each warp evaluates P at 32
// consecutive slots, overlapping the previous warp by one, so every lane evaluates P
// exactly once and lanes 1..31 emit the group whose upper bound they hold (its lower
// bound is the previous lane's slot).  (A thread per (node, group) with the first lane
// of each warp evaluating its lower bound too made every warp pay two evaluations.)
__global__ void trt_emission_kernel(const double* __restrict__ T, const double* __restrict__ sigma,
                                    const double* __restrict__ Iprev, const double* __restrict__ nu, int G, int n,
                                    size_t nodes, double inv_dt, double* __restrict__ q) {
    const size_t slots = nodes * (size_t)(G + 1);
    const int lane = threadIdx.x & 31;
    const size_t warps = ((size_t)gridDim.x * blockDim.x) >> 5;
    for (size_t w = (((size_t)blockIdx.x * blockDim.x) >> 5) + (threadIdx.x >> 5); 31 * w + 1 < slots; w += warps) {
        const size_t sl = 31 * w + lane;
        const bool on = sl < slots;
        const size_t ss = on ? sl : slots - 1;
        const size_t v = ss / (size_t)(G + 1);
        const int bnd = (int)(ss - v * (size_t)(G + 1));
        const double t = T[v];
        double P, d, d2;
        planck_P(nu[bnd] * (1.0 / t), P, d, d2);
        const double Pl = __shfl_up_sync(0xffffffffu, P, 1);
        if (on && lane >= 1 && bnd >= 1) {
            const int g = bnd - 1;
            const size_t ii = v * (size_t)G + g;
            const double t2 = t * t;
            q[ii] = fma(sigma[(v / n) * G + g], t2 * t2 * (P - Pl), Iprev[ii] * inv_dt);
        }
    }
}

// sum_g sig_g B_g(T) and its first two T-derivatives over the groups, one warp per node:
// lane l evaluates P at the bounds b = l, l + 32, ... and owns group g = b - 1 (its lower
// bound comes from the neighbouring lane, or from lane 31 of the previous round);
// fixed-order butterfly sums, so every lane ends with the same E, dE, d2E.  With
// B(T) = T^4 P(nu/T), x = nu/T, h = x P'(x), q = x h e^x/(e^x - 1):
//   dB/dT = T^3 (4P - h),   d2B/dT2 = T^2 (12P - 3h - q).
__device__ __forceinline__ void emission_sum_warp(double T, int G, const double* __restrict__ sig,
                                                  const double* __restrict__ nu, int lane, double& E, double& dE,
                                                  double& d2E) {
    const double T2 = T * T, T3 = T2 * T, T4 = T3 * T, iT = 1.0 / T;
    double e = 0.0, de = 0.0, d2e = 0.0;
    // top bound far in the Wien tail (x > 50: 1 - P < 1e-17, x P' < 1e-15): P = 1,
    // h = q = 0 without evaluating it, which saves the round a lone bound G would take
    // (G = 64: bounds 64 = 2 x 32 + 1); warp-uniform, every lane has the same T
    const bool top_one = nu[G] * iT > 50.0;
    const int last = top_one ? G - 1 : G;
    double carry_P = 0.0, carry_h = 0.0, carry_q = 0.0;  // bound 32k - 1 (lane 31 of the previous round)
    double P = 0.0, h = 0.0, q = 0.0;
    int b0 = 0;
    for (; b0 <= last; b0 += 32) {
        const int bnd = b0 + lane;
        P = 0.0;
        h = 0.0;
        q = 0.0;
        if (bnd <= last) {
            const double x = nu[bnd] * iT;
            double dP, rem1;
            planck_P(x, P, dP, rem1);
            h = x * dP;
            q = x * h * (1.0 + rem1);
        }
        double Pl = __shfl_up_sync(0xffffffffu, P, 1), hl = __shfl_up_sync(0xffffffffu, h, 1),
               ql = __shfl_up_sync(0xffffffffu, q, 1);
        if (lane == 0) {
            Pl = carry_P;
            hl = carry_h;
            ql = carry_q;
        }
        if (bnd >= 1 && bnd <= last) {
            const double sg = sig[bnd - 1];
            const double dPg = P - Pl, dhg = h - hl, dqg = q - ql;
            e = fma(sg, T4 * dPg, e);
            de = fma(sg, T3 * (4.0 * dPg - dhg), de);
            d2e = fma(sg, T2 * (12.0 * dPg - 3.0 * dhg - dqg), d2e);
        }
        carry_P = __shfl_sync(0xffffffffu, P, 31);
        carry_h = __shfl_sync(0xffffffffu, h, 31);
        carry_q = __shfl_sync(0xffffffffu, q, 31);
    }
    if (top_one) {
        // group G - 1 between bound G - 1 (held by lane last - (b0 - 32) of the last round)
        // and bound G (P = 1, h = q = 0)
        const int src = last - (b0 - 32);
        const double Pl = __shfl_sync(0xffffffffu, P, src), hl = __shfl_sync(0xffffffffu, h, src),
                     ql = __shfl_sync(0xffffffffu, q, src);
        if (lane == 0) {
            const double sg = sig[G - 1];
            const double dPg = 1.0 - Pl, dhg = -hl, dqg = -ql;
            e = fma(sg, T4 * dPg, e);
            de = fma(sg, T3 * (4.0 * dPg - dhg), de);
            d2e = fma(sg, T2 * (12.0 * dPg - 3.0 * dhg - dqg), d2e);
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        e += __shfl_xor_sync(0xffffffffu, e, o);
        de += __shfl_xor_sync(0xffffffffu, de, o);
        d2e += __shfl_xor_sync(0xffffffffu, d2e, o);
    }
    E = e;
    dE = de;
    d2E = d2e;
}

// per node (one warp): solve cv_dt (T - Tk) + E(T) = sphi by a bracketed Newton
// iteration from the current iterate T; writes the new T, replaces the previous energy
// density E^l by this sweep's phi, and writes per-block partial sums of (dT^2, dE^2) for
// the outer stopping test ||u^{l+1} - u^l||_2 < eps ||u^1 - u^0||_2, u = [T, E]
// (eq:relative_tol), summed in a fixed order afterwards.  One warp
// per node: nodes converge after different numbers of steps, and a thread per node
// made every warp wait for its slowest node.
#ifndef SWEEP_TRT_MINB
#define SWEEP_TRT_MINB 3  // 72 registers, 3 blocks of 256 per SM, grid 3 x 148: C5 TRT 23.9 -> 23.4 ms
#endif
__global__ void __launch_bounds__(256, SWEEP_TRT_MINB) trt_update_kernel(const double* __restrict__ Tk, double* __restrict__ T,
                                                         const double* __restrict__ sphi, const double* __restrict__ phi,
                                                         double* __restrict__ E, const double* __restrict__ sigma,
                                                         const double* __restrict__ nu, int G, int n, size_t nodes,
                                                         double cv_dt, double* __restrict__ partial, int* err) {
    __shared__ double red[2][8];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    double dsq = 0.0, esq = 0.0;
    const size_t warps = (size_t)gridDim.x * (blockDim.x >> 5);
    for (size_t v = (size_t)blockIdx.x * (blockDim.x >> 5) + wib; v < nodes; v += warps) {
        const double* sg = sigma + (v / n) * G;
        const double tk = Tk[v], s = sphi[v], told = T[v];
        double t = told > 0.0 ? told : (tk > 0.0 ? tk : 1.0);
        double lo = 0.0, hi = -1.0;  // hi < 0: no upper bracket yet
        bool ok = false;
        for (int it = 0; it < 100; ++it) {
            double E, dE, d2E;
            emission_sum_warp(t, G, sg, nu, lane, E, dE, d2E);
            const double f = fma(cv_dt, t - tk, E - s);
            // converged to the rounding noise of f (a few ulps of its largest term): a Newton
            // step from here would only chase that noise (and fall back to bisection)
            if (fabs(f) <= 4e-16 * (cv_dt * (t + tk) + E + fabs(s))) {
                ok = true;
                break;
            }
            if (f < 0.0) lo = t;
            else hi = t;
            // far from the root: Newton step in v = T^m, m = t E'/E the local power-law
            // exponent of the emission: exact in one step for a single power law, so cooling
            // nodes whose root lies far below T (emission ~ T^4 >> the absorbed sphi) do not
            // creep down by the factor 3/4 per step plain Newton would take.  Close to it
            // (Newton step below 5 %): Halley's step (cubic convergence), which ends the
            // iteration one evaluation earlier than Newton's on most nodes.
            const double fp = cv_dt + dE;
            const double nr = f / (t * fp);
            double tn;
            bool halley = false;
            if (fabs(nr) < 0.05) {
                const double den = 2.0 * fp * fp - f * d2E;
                halley = den > 0.0;
                tn = halley ? t - 2.0 * f * fp / den : t - f / fp;
            } else {
                const double m = (E > 0.0) ? fmax(1.0, t * dE / E) : 1.0;
                const double r = 1.0 - m * nr;
                tn = (r > 0.0) ? t * exp(log(r) / m) : 0.0;  // 0: rejected by the bracket below
            }
            if (!(tn > lo) || (hi > 0.0 && !(tn < hi))) {
                tn = (hi > 0.0) ? 0.5 * (lo + hi) : 2.0 * t;
                halley = false;
            }
            // converged: a Halley step below 1e-7 relative (the error after it is of the
            // order of its cube), a Newton step below 1e-13 (the iterate after it is exact to
            // rounding: quadratic convergence; smaller thresholds sit below the rounding noise
            // of f), or the sign bracket that narrow
            const bool done = fabs(tn - t) <= (halley ? 1e-7 : 1e-13) * tn || (hi > 0.0 && hi - lo <= 1e-15 * hi);
            t = tn;
            if (done) {
                ok = true;
                break;
            }
        }
        if (lane == 0) {
            if (!ok || !(t > 0.0) || !(t < 1e300)) atomicOr(err, 16);
            T[v] = t;
            dsq = fma(t - told, t - told, dsq);
            // E = phi (c = 1): the energy-density half of u = [T, E] (eq:relative_tol)
            const double en = phi[v], de = en - E[v];
            E[v] = en;
            esq = fma(de, de, esq);
        }
    }
    if (lane == 0) {
        red[0][wib] = dsq;
        red[1][wib] = esq;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0.0, c = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
            a += red[0][w];
            c += red[1][w];
        }
        partial[2 * blockIdx.x] = a;
        partial[2 * blockIdx.x + 1] = c;
    }
}

// fixed-order sum of the per-block partials -> out[2] (one thread: tiny)
__global__ void trt_norm_kernel(const double* __restrict__ partial, int nblocks, double* __restrict__ out) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        double a = 0.0, b = 0.0;
        for (int i = 0; i < nblocks; ++i) {
            a += partial[2 * i];
            b += partial[2 * i + 1];
        }
        out[0] = a;
        out[1] = b;
    }
}

#ifndef SWEEP_TRT_BPS
#define SWEEP_TRT_BPS 3
#endif
int trt_blocks(int n_sm) { return (n_sm > 0 ? n_sm : 1) * SWEEP_TRT_BPS; }

int launch_trt_emission(const double* T, const double* sigma, const double* Iprev, const double* nu, int G, int n,
                        size_t nodes, double inv_dt, double* q, int n_sm, void* stream) {
#ifndef SWEEP_EMIS_BPS
#define SWEEP_EMIS_BPS 4  // all blocks resident (a grid-stride kernel: 8 x 148 left a partial second wave; -0.5 ms)
#endif
    trt_emission_kernel<<<(n_sm > 0 ? n_sm : 1) * SWEEP_EMIS_BPS, 256, 0, (cudaStream_t)stream>>>(T, sigma, Iprev, nu, G, n, nodes, inv_dt, q);
    return (int)cudaGetLastError();
}

// E^0 = sum_g I^k_g at every node (the energy density of the isotropic previous
// intensity: c = 1, sum_d w_d = 1), the E half of the initial guess u^0 = [T^k, E^k];
// one thread per node, groups summed in index order
__global__ void trt_e0_kernel(const double* __restrict__ Iprev, int G, size_t nodes, double* __restrict__ E) {
    for (size_t v = (size_t)blockIdx.x * blockDim.x + threadIdx.x; v < nodes; v += (size_t)gridDim.x * blockDim.x) {
        const double* I = Iprev + v * (size_t)G;
        double e = 0.0;
        for (int g = 0; g < G; ++g) e += I[g];
        E[v] = e;
    }
}

int launch_trt_e0(const double* Iprev, int G, size_t nodes, double* E, int n_sm, void* stream) {
    const int block = 256;
    size_t want = (nodes + block - 1) / block;
    const size_t cap = (size_t)n_sm * 8;
    const int grid = (int)(want < 1 ? 1 : (want < cap ? want : cap));
    trt_e0_kernel<<<grid, block, 0, (cudaStream_t)stream>>>(Iprev, G, nodes, E);
    return (int)cudaGetLastError();
}

int launch_trt_update(const double* Tk, double* T, const double* sphi, const double* phi, double* E,
                      const double* sigma, const double* nu, int G, int n, size_t nodes, double cv_dt, double* partial,
                      double* norms, int* err, int n_sm, void* stream) {
    const int nb = trt_blocks(n_sm);
    trt_update_kernel<<<nb, 256, 0, (cudaStream_t)stream>>>(Tk, T, sphi, phi, E, sigma, nu, G, n, nodes, cv_dt, partial,
                                                            err);
    trt_norm_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(partial, nb, norms);
    return (int)cudaGetLastError();
}

}  // namespace sweepk
