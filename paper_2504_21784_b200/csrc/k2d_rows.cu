// k2d_rows.cu — 2-D p = 1 sweep for FEW chains per quadrant (gray / few-group problems such as
// C3): a diagonal wavefront inside each warp instead of the strip pipeline.
//
// PAPER.md: the lumped upwind-DG element system (eq:dgsn_transport :332-336, GLL lumping
// :654), swept in upwind order (:299-327), with the gray moments phi, J, T and the boundary
// closures beta, J+ (:156-176) accumulated on the fly.
//
// Layout ("few chains"): a chain is one (direction, group) of a quadrant.  A
// WARP sweeps 32 consecutive element rows (sweep coordinates) of one chain, one LANE per row;
// at step t lane r solves the element in column t - (32 b + r) of its row, so the lanes form
// an anti-diagonal.  The y-trace a lane needs was produced one step earlier by the lane below
// (same column): one shuffle per step.  The x-trace stays in the lane's registers.  The
// warps of the next row blocks of the same chain lag by 32 steps each and take their bottom
// lane's y-trace from the block below through shared memory.  A CTA holds W chains x all row
// blocks of one quadrant, so every element the CTA touches at step t is touched by all its
// chains at that step: the chain sum with the moment / boundary weights is one
// shared-memory reduction per step (fixed chain order: deterministic), written to the CTA's
// slab; the slabs are summed in a fixed order by the finalize kernel.  The critical path is
// the wavefront itself, nx + ny - 1 steps, with no inter-CTA hand-off.
#include "sweep_device.cuh"

namespace sweepk {

__global__ void __launch_bounds__(256) sweep2d_rows_kernel(const Sweep2DRowsParams prm) {
    constexpr int P = 1, NP1 = 2, NN = 4, D = 4;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int W = prm.W, nrb = prm.nrb;
    const int c = wid % W, b = wid / W;  // chain within the CTA, row block
    const StreamDesc sd = prm.streams[blockIdx.x];
    const bool fx = (sd.quadrant & 1) != 0, fy = (sd.quadrant & 2) != 0;
    const int nx = prm.nx, ny = prm.ny, G = prm.G;
    const size_t nodes = prm.nodes;
    const int nsteps = nx + 32 * nrb - 1;

    extern __shared__ __align__(16) double sh[];
    double* psi = sh;                                  // [2][W * nrb][32][NN]  this step's solutions
    double* hand = psi + 2 * (size_t)W * nrb * 32 * NN;  // [2][W][nrb][NP1]     y-trace between row blocks
    double* coef = hand + 2 * (size_t)W * nrb * NP1;     // [W][16] moment, beta, J+ weights

    const int jc = sd.g0 + c;
    const bool con = c < sd.ng;
    const int dd = sd.d0 + (con ? jc / G : 0), g = con ? jc % G : 0;
    for (int it = tid; it < W * 16; it += blockDim.x) {
        const int cc = it / 16, f = it - cc * 16;
        double v = 0.0;
        if (cc < sd.ng) {
            const DirConst& Dc = prm.dirs[sd.d0 + (sd.g0 + cc) / G];
            v = (f < 6) ? Dc.mom[f] : (f < 10) ? Dc.bw[f - 6] : (f < 14) ? Dc.jw[f - 10] : 0.0;
        }
        coef[it] = v;
    }
    double cx = 0.0, cy = 0.0;
    if (con) {
        cx = prm.dirs[dd].cx;
        cy = prm.dirs[dd].cy;
    }
    const LaneP1 L = make_lane_p1(cx, cy);
    const int jp = 32 * b + lane;  // this lane's row (sweep order)
    const bool rowok = con && jp < ny;
    const int j = fy ? ny - 1 - jp : jp;

    // x-inflow of the row (physical face x- or x+)
    double tx[NP1] = {0.0, 0.0};
    if (rowok) {
#pragma unroll
        for (int bq = 0; bq < NP1; ++bq) {
            const int bb = fy ? P - bq : bq;
            tx[bq] = prm.inflow[(size_t)bnode2d(fx ? 1 : 0, j, bb, nx, ny, NP1) * G + g];
        }
    }
    // inputs of sweep column ip of this row: sigma~ and q in sweep node order
    struct In {
        double st, q[NN], yin[NP1];  // yin: the physical y-inflow (bottom lane of block 0 only)
    };
    auto load = [&](int ip, In& x) {
        const int i = fx ? nx - 1 - ip : ip;
        const size_t e = (size_t)i + (size_t)nx * j;
        x.st = __ldg(prm.sigma + e * G + g) + prm.inv_c_dt;
#pragma unroll
        for (int kk = 0; kk < NN; ++kk) {
            const int aq = kk % NP1, bq = kk / NP1;
            const int a = fx ? P - aq : aq, bb = fy ? P - bq : bq;
            x.q[kk] = __ldg(prm.q + (e * NN + a + NP1 * bb) * G + g);
        }
        if (lane == 0 && b == 0) {
#pragma unroll
            for (int aq = 0; aq < NP1; ++aq) {
                const int a = fx ? P - aq : aq;
                x.yin[aq] = __ldg(prm.inflow + (size_t)bnode2d(fy ? 3 : 2, i, a, nx, ny, NP1) * G + g);
            }
        }
    };
    // the element needed at step t is requested at step t - D into slot t % D
    In buf[D];
#pragma unroll
    for (int u = 0; u < D; ++u) {
        const int ip = u - jp;
        if (rowok && ip >= 0 && ip < nx) load(ip, buf[u]);
    }
    double ty_in[NP1] = {0.0, 0.0};  // y-trace from the lane below, produced last step
    bool bad = false;

    for (int t0 = 0; t0 < nsteps; t0 += D) {
#pragma unroll
        for (int u = 0; u < D; ++u) {
            const int t = t0 + u;
            const int ip = t - jp;
            const bool act = rowok && ip >= 0 && ip < nx && t < nsteps;
            In cur = buf[u];
            {
                const int ipn = ip + D;
                if (rowok && ipn >= 0 && ipn < nx) load(ipn, buf[u]);
            }
            // the y-trace of this lane's element: the physical y-inflow (row 0), the block
            // below's top lane (through shared memory, written last step), or the lane below
            double ty[NP1];
            if (lane == 0) {
                if (b == 0) {
#pragma unroll
                    for (int aq = 0; aq < NP1; ++aq) ty[aq] = act ? cur.yin[aq] : 0.0;
                } else {
#pragma unroll
                    for (int aq = 0; aq < NP1; ++aq) ty[aq] = hand[(((size_t)((t + 1) & 1) * W + c) * nrb + b) * NP1 + aq];
                }
            } else {
#pragma unroll
                for (int aq = 0; aq < NP1; ++aq) ty[aq] = ty_in[aq];
            }
            double uu[NN] = {0.0, 0.0, 0.0, 0.0}, txo[NP1], tyo[NP1] = {0.0, 0.0};
            if (act) {
                bad |= bad_sigma(cur.st);
                solve_p1(L, cur.st, cur.q, tx, ty, uu, txo, tyo);
#pragma unroll
                for (int k = 0; k < NP1; ++k) tx[k] = txo[k];
            }
#pragma unroll
            for (int k = 0; k < NP1; ++k) ty_in[k] = __shfl_up_sync(FULLMASK, tyo[k], 1);
            if (lane == 31 && b + 1 < nrb)
#pragma unroll
                for (int k = 0; k < NP1; ++k) hand[(((size_t)(t & 1) * W + c) * nrb + b + 1) * NP1 + k] = tyo[k];
            double* ps = psi + (((size_t)(t & 1) * W * nrb + wid) * 32 + lane) * NN;
#pragma unroll
            for (int k = 0; k < NN; ++k) ps[k] = uu[k];
            __syncthreads();
            // ---- the CTA's chains summed with the weights, per (row block, row, node)
            const double* pr = psi + (size_t)(t & 1) * W * nrb * 32 * NN;
            for (int o = tid; o < nrb * 32 * NN; o += blockDim.x) {
                const int kk = o % NN, rr = (o / NN) % 32, bb = o / (32 * NN);
                const int jpo = 32 * bb + rr, ipo = t - jpo;
                if (jpo >= ny || ipo < 0 || ipo >= nx) continue;
                double acc[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
                for (int cc = 0; cc < sd.ng; ++cc) {
                    const double v = pr[(((size_t)bb * W + cc) * 32 + rr) * NN + kk];
                    const double* cf = coef + cc * 16;
#pragma unroll
                    for (int f = 0; f < 6; ++f) acc[f] = fma(cf[f], v, acc[f]);
                }
                const int i = fx ? nx - 1 - ipo : ipo, jj = fy ? ny - 1 - jpo : jpo;
                const int aq = kk % NP1, bq = kk / NP1;
                const int a = fx ? P - aq : aq, bn = fy ? P - bq : bq;
                const size_t e = (size_t)i + (size_t)nx * jj;
                double* slab = prm.slabs + (size_t)blockIdx.x * prm.out_size;
#pragma unroll
                for (int f = 0; f < 6; ++f) slab[(size_t)f * nodes + e * NN + a + NP1 * bn] = acc[f];
                // boundary closures at this node, for every physical boundary face it lies on
                // (the element's own trace for every direction, reading R5)
                const bool onf[4] = {i == 0 && a == 0, i == nx - 1 && a == P, jj == 0 && bn == 0, jj == ny - 1 && bn == P};
#pragma unroll
                for (int face = 0; face < 4; ++face) {
                    if (!onf[face]) continue;
                    double vb = 0.0, vj = 0.0;
                    for (int cc = 0; cc < sd.ng; ++cc) {
                        const double v = pr[(((size_t)bb * W + cc) * 32 + rr) * NN + kk];
                        vb = fma(coef[cc * 16 + 6 + face], v, vb);
                        vj = fma(coef[cc * 16 + 10 + face], v, vj);
                    }
                    const int idx = (face < 2) ? jj : i, node = (face < 2) ? bn : a;
                    const int bnd = bnode2d(face, idx, node, nx, ny, NP1);
                    slab[6 * nodes + bnd] = vb;
                    slab[6 * nodes + prm.nbnode + bnd] = vj;
                }
            }
        }
    }
    if (bad) atomicOr(prm.err, 1);
}

int rows_smem_bytes(int W, int nrb) {
    return (int)sizeof(double) * (2 * W * nrb * 32 * 4 + 2 * W * nrb * 2 + W * 16);
}

int launch_sweep2d_rows(const Sweep2DRowsParams& prm, int grid, int block, size_t smem, void* stream) {
    const void* f = (const void*)sweep2d_rows_kernel;
    if (smem > 48 * 1024) {
        const int e = raise_smem_cap(f);
        if (e) return e;
    }
    void* args[] = {(void*)&prm};
    return (int)cudaLaunchKernel(f, dim3(grid), dim3(block), args, smem, (cudaStream_t)stream);
}

}  // namespace sweepk
