// k_1d.cu — the 1-D (slab) sweep as a warp-level affine scan (C1, C2).
//
// PAPER.md: the lumped upwind-DG element system (eq:dgsn_transport :332-336, GLL lumping
// :654) in 1-D, swept in upwind order (:299-327), with the gray moments phi, J, T_xx,
// beta, J+ (:156-176).  With a given source the outflow of element e is affine in its
// inflow, psi_out = t_e psi_in + s_e, 0 < t_e < 1 (p = 2: the modal solve of
// solve1d), so a chain of elements is a composition of affine maps: a scan.
//
// Layout ("1-D"): one WARP per chain (direction d, group g), one LANE per
// segment of L = ceil(nx / 32) consecutive elements (sweep order).  Phase 1: each lane
// composes its segment's maps (inputs prefetched D elements ahead in registers: the chain
// step is latency bound).  Phase 2: an exclusive warp scan of the maps (5 shuffle steps)
// gives every segment its inflow.  Phase 3: each lane re-sweeps its segment; at step t all
// warps of the CTA (W chains of one half-range) are at the same elements s L + t, so the
// sum over the CTA's chains of the moment contributions is one shared-memory reduction per
// step, in a fixed warp order (deterministic), written to the CTA's slab.  Slabs are summed
// in a fixed order by the last CTA to finish when they are small (one launch per sweep),
// else by the finalize kernel.  The zero-and-scale fixup is not affine: it keeps the
// sequential kernel (sweep1d_kernel).
#include "sweep_device.cuh"

namespace sweepk {

template <int P, int OPT>
__global__ void __launch_bounds__(256) sweep1d_scan_kernel(const Sweep1DScanParams prm) {
    constexpr bool SIG = (OPT & OPT_SIGMA) != 0;
    constexpr bool HALF = (OPT & OPT_HALF) != 0;
    constexpr int NP1 = P + 1;
    constexpr int NM = SIG ? 5 : 3;                  // phi, J, Txx (+ sigma phi, sigma J)
    constexpr int NV = (NM + (HALF ? 1 : 0)) * NP1;  // (+ P_xx)
    constexpr int D = 8;                             // prefetch distance (elements): ~HBM latency / step
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int W = blockDim.x >> 5;
    const int nx = prm.nx, G = prm.G, L = prm.seglen;
    const size_t nodes = prm.nodes;
    extern __shared__ __align__(16) double red[];    // [2][W][32][NV] + [W][4] (+ single: [NM][nodes])
    double* bred = red + 2 * (size_t)W * 32 * NV;
    double* acc1 = bred + 4 * (size_t)W;             // single: the gray fields of the whole mesh

    // this warp's chain.  Slab mode: the CTA's chains are one half-range's [g0, g0 + ng).
    // Single mode (one CTA, tiny problems): warps [0, nw0) are the mu >= 0 chains, the rest the
    // mu < 0 chains, and the gray fields are accumulated in shared memory (no slab, no finalize).
    const bool single = prm.single != 0;
    const StreamDesc sd = prm.streams[single ? (w >= prm.nw0 ? 1 : 0) : blockIdx.x];
    const bool fx = (sd.quadrant & 1) != 0;
    const int wl = single ? (w >= prm.nw0 ? w - prm.nw0 : w) : w;
    const int j = sd.g0 + wl;
    const bool on = wl < sd.ng;
    const int d = sd.d0 + (on ? j / G : 0), g = on ? j % G : 0;
    if (single)
        for (size_t k = tid; k < (size_t)NM * nodes; k += blockDim.x) acc1[k] = 0.0;
    double c = 0.0, cm[NM + 1], bw0 = 0.0, bw1 = 0.0, jw0 = 0.0, jw1 = 0.0;
#pragma unroll
    for (int m = 0; m <= NM; ++m) cm[m] = 0.0;
    if (on) {
        const DirConst& Dc = prm.dirs[d];
        c = Dc.cx;
        cm[0] = Dc.mom[0];
        cm[1] = Dc.mom[1];
        cm[2] = Dc.mom[2];
        cm[NM] = Dc.pw[0];
        bw0 = Dc.bw[0];
        bw1 = Dc.bw[1];
        jw0 = Dc.jw[0];
        jw1 = Dc.jw[1];
    }
    const int e0 = min(nx, lane * L), e1 = min(nx, e0 + L);  // this lane's segment (sweep order)

    // inputs of sweep-order element ip: sigma~, sigma, nodal q in sweep node order
    struct In {
        double st, sg, q[NP1];
    };
    auto load = [&](int ip, In& x) {
        const int i = fx ? nx - 1 - ip : ip;
        x.sg = __ldg(prm.sigma + (size_t)i * G + g);
#pragma unroll
        for (int aq = 0; aq < NP1; ++aq) x.q[aq] = __ldg(prm.q + ((size_t)i * NP1 + (fx ? P - aq : aq)) * G + g);
    };
    // software pipeline over the segment: element ip's inputs were requested D steps earlier.
    // A segment of at most D elements (C1) is loaded once: phase 3 reuses phase 1's buffer.
    In buf[D];
    auto sweep_segment = [&](bool preload, auto&& body) {
#pragma unroll
        for (int u = 0; u < D; ++u)
            if (preload && on && e0 + u < e1) load(e0 + u, buf[u]);
        for (int t0 = 0; t0 < L; t0 += D) {
#pragma unroll
            for (int u = 0; u < D; ++u) {
                if (t0 + u >= L) break;  // uniform over the CTA (every lane has L steps)
                const int ip = e0 + t0 + u;
                In cur = buf[u];
                if (on && ip + D < e1) load(ip + D, buf[u]);
                cur.st = cur.sg + prm.inv_c_dt;
                body(ip, cur);
            }
        }
    };

    // ---- phase 1: compose this segment's affine maps
    double Tm = 1.0, Sm = 0.0;
    sweep_segment(true, [&](int ip, const In& x) {
        if (!(on && ip < e1)) return;
        if (bad_sigma(x.st)) atomicOr(prm.err, 1);
        double psi[NP1], ta, sa;
        solve1d<P>(c, x.st, x.q, 0.0, psi, ta, sa);
        Sm = fma(ta, Sm, sa);
        Tm = ta * Tm;
    });
    // ---- phase 2: exclusive warp scan of the maps (lane s gets lanes 0..s-1 composed)
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const double Tp = __shfl_up_sync(FULLMASK, Tm, off), Sp = __shfl_up_sync(FULLMASK, Sm, off);
        if (lane >= off) {
            Sm = fma(Tm, Sp, Sm);  // (ours) o (earlier): x -> Tm (Tp x + Sp) + Sm
            Tm = Tm * Tp;
        }
    }
    const double psi_bc = on ? prm.inflow[(size_t)(fx ? 1 : 0) * G + g] : 0.0;
    double Tl = __shfl_up_sync(FULLMASK, Tm, 1), Sl = __shfl_up_sync(FULLMASK, Sm, 1);
    double up = (lane == 0) ? psi_bc : fma(Tl, psi_bc, Sl);

    // ---- phase 3: final sweep; per step, the CTA's chains summed in shared memory
    double bv[4] = {0.0, 0.0, 0.0, 0.0};  // beta x=0, beta x=lx, J+ x=0, J+ x=lx of this chain
    double* slab = prm.slabs + (size_t)blockIdx.x * prm.out_size;
    const size_t sig_off = 3 * nodes + 4;  // after phi, J, Txx, beta[2], J+[2]
    int t = 0;
    sweep_segment(L > D, [&](int ip, const In& x) {
        double v[NV];
        const bool live = on && ip < e1;
        if (live) {
            double psi[NP1], ta, sa;
            solve1d<P>(c, x.st, x.q, up, psi, ta, sa);
            up = psi[P];
#pragma unroll
            for (int aq = 0; aq < NP1; ++aq) {
                v[0 * NP1 + aq] = cm[0] * psi[aq];
                v[1 * NP1 + aq] = cm[1] * psi[aq];
                v[2 * NP1 + aq] = cm[2] * psi[aq];
                if constexpr (SIG) {
                    v[3 * NP1 + aq] = x.sg * v[0 * NP1 + aq];
                    v[4 * NP1 + aq] = x.sg * v[1 * NP1 + aq];
                }
                if constexpr (HALF) v[NM * NP1 + aq] = cm[NM] * psi[aq];
            }
            // boundary closures at x = 0 (node a = 0) and x = lx (node a = P), the element's
            // own trace for every direction (reading R5)
            const int i = fx ? nx - 1 - ip : ip;
            if (i == 0) {
                const double p0 = psi[fx ? P : 0];
                bv[0] = bw0 * p0;
                bv[2] = jw0 * p0;
            }
            if (i == nx - 1) {
                const double p1 = psi[fx ? 0 : P];
                bv[1] = bw1 * p1;
                bv[3] = jw1 * p1;
            }
        } else {
#pragma unroll
            for (int k = 0; k < NV; ++k) v[k] = 0.0;
        }
        double* rb = red + ((size_t)(t & 1) * W + w) * 32 * NV + lane * NV;
#pragma unroll
        for (int k = 0; k < NV; ++k) rb[k] = v[k];
        __syncthreads();
        // sum over the CTA's chains (warp order) for the 32 elements of this step
        const double* rs = red + (size_t)(t & 1) * W * 32 * NV;
        if (single) {
            // per half-range (its own physical element at this step), added to the mesh fields;
            // one thread per (segment, value) handles both halves: no two threads share an entry
            for (int o = tid; o < 32 * NV; o += blockDim.x) {
                const int s = o / NV, r = o - s * NV;
                const int ips = s * L + t;
                if (ips >= min(nx, (s + 1) * L)) continue;
                const int m = r / NP1, aq = r - m * NP1;
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int w0 = h ? prm.nw0 : 0, w1 = h ? W : prm.nw0;
                    if (w0 >= w1) continue;
                    double acc = 0.0;
                    for (int ww = w0; ww < w1; ++ww) acc += rs[((size_t)ww * 32 + s) * NV + r];
                    const int i = h ? nx - 1 - ips : ips;
                    const int a = h ? P - aq : aq;
                    acc1[(size_t)m * nodes + (size_t)i * NP1 + a] += acc;
                }
            }
            ++t;
            return;
        }
        for (int o = tid; o < 32 * NV; o += blockDim.x) {
            const int s = o / NV, r = o - s * NV;
            const int ips = s * L + t;
            if (ips >= min(nx, (s + 1) * L)) continue;
            double acc = 0.0;
            for (int ww = 0; ww < W; ++ww) acc += rs[((size_t)ww * 32 + s) * NV + r];
            const int m = r / NP1, aq = r - m * NP1;
            const int i = fx ? nx - 1 - ips : ips;
            const int a = fx ? P - aq : aq;
            const size_t rowb = (m < 3) ? (size_t)m * nodes : (m < NM) ? sig_off + (size_t)(m - 3) * nodes : prm.hr_off;
            slab[rowb + (size_t)i * NP1 + a] = acc;
        }
        ++t;
    });
    // boundary closures: warp sums (fixed butterfly), then over warps in order
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) bv[k] += __shfl_xor_sync(FULLMASK, bv[k], o);
    if (lane == 0)
#pragma unroll
        for (int k = 0; k < 4; ++k) bred[w * 4 + k] = bv[k];
    __syncthreads();
    if (tid < 4) {
        double acc = 0.0;
        for (int ww = 0; ww < W; ++ww) acc += bred[ww * 4 + tid];
        // beta[x=0], beta[x=lx], J+[x=0], J+[x=lx]
        (single ? prm.fused_out : slab)[3 * nodes + tid] = acc;
    }
    if (single) {
        // the mesh fields straight to the packed output (rows phi, J, Txx [, sigma phi, sigma J])
        bool bad = false;
        for (size_t k = tid; k < (size_t)NM * nodes; k += blockDim.x) {
            const size_t m = k / nodes, rest = k - m * nodes;
            const double v = acc1[k];
            prm.fused_out[(m < 3 ? m * nodes : sig_off + (m - 3) * nodes) + rest] = v;
            bad |= !(fabs(v) < 1.0e300);
        }
        if (bad) atomicOr(prm.err, 2);
        return;
    }

    // ---- fused final sum: the last CTA to finish sums the slabs in order (small outputs)
    if (prm.fused_out) {
        __threadfence();
        __syncthreads();
        __shared__ int s_last;
        if (tid == 0) s_last = (atomicAdd(prm.done_counter, 1) == (int)gridDim.x - 1);
        __syncthreads();
        if (s_last) {
            __threadfence();
            bool bad = false;
            for (size_t k = tid; k < prm.sum_size; k += blockDim.x) {
                double acc = 0.0;
                for (int b = 0; b < (int)gridDim.x; ++b) acc += __ldcg(prm.slabs + (size_t)b * prm.out_size + k);
                prm.fused_out[k] = acc;
                bad |= !(fabs(acc) < 1.0e300);
            }
            if (bad) atomicOr(prm.err, 2);
            if (tid == 0) *prm.done_counter = 0;  // ready for the next run
        }
    }
}

template <int P>
static const void* pick_scan(int opt) {
    switch (opt & (OPT_SIGMA | OPT_HALF)) {
        case 0: return (const void*)sweep1d_scan_kernel<P, 0>;
        case OPT_SIGMA: return (const void*)sweep1d_scan_kernel<P, OPT_SIGMA>;
        case OPT_HALF: return (const void*)sweep1d_scan_kernel<P, OPT_HALF>;
        default: return (const void*)sweep1d_scan_kernel<P, OPT_SIGMA | OPT_HALF>;
    }
}

int scan1d_smem_bytes(int p, int opt, int warps, size_t single_nodes) {
    const int nm = (opt & OPT_SIGMA) ? 5 : 3;
    const int nv = (nm + ((opt & OPT_HALF) ? 1 : 0)) * (p + 1);
    return (int)(sizeof(double) * (2 * (size_t)warps * 32 * nv + warps * 4 + (size_t)nm * single_nodes));
}

int launch_sweep1d_scan(int p, int opt, const Sweep1DScanParams& prm, int grid, int block, size_t smem, void* stream) {
    const void* f = (p == 2) ? pick_scan<2>(opt) : pick_scan<1>(opt);
    if (smem > 48 * 1024) {
        const int e = raise_smem_cap(f);
        if (e) return e;
    }
    void* args[] = {(void*)&prm};
    return (int)cudaLaunchKernel(f, dim3(grid), dim3(block), args, smem, (cudaStream_t)stream);
}

int upload_modal_1d(const ModalConsts& mc) { return (int)cudaMemcpyToSymbol(cM, &mc, sizeof(ModalConsts)); }

}  // namespace sweepk
