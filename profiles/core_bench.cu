// core_bench.cu — isolate the 2-D p=2 element loop (solve + group reduction)
// from the wavefront pipeline: every warp sweeps columns of a T-row strip on
// shared-memory data, nothing else.  Reports cycles per lane-solve.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2504_21784_b200/csrc \
//      -o profiles/core_bench profiles/core_bench.cu
#include <cstdio>
#include <cstring>
#include <type_traits>
#include "../paper_2504_21784_b200/csrc/sweep_device.cuh"

using namespace sweepk;

template <int K, int T, bool RED, int MINB, int LG = 32>
__global__ void __launch_bounds__(256, MINB) core_kernel(double* out, int ncols, double cx, double cy) {
    constexpr int NQ = 9, NT = 3, GBK = LG * K;
    extern __shared__ __align__(16) double sm[];
    double* qs = sm;                 // [T][NQ][GBK]
    double* ss = qs + T * NQ * GBK;  // [T][GBK]
    double* S = ss + T * GBK;        // [T][8][NQ]
    const int tid = threadIdx.x, lane = tid & 31, dl = tid >> 5, gl = tid & (LG - 1);
    for (int i = tid; i < T * NQ * GBK; i += blockDim.x) qs[i] = 0.001 * (i % 97);
    for (int i = tid; i < T * GBK; i += blockDim.x) ss[i] = 1.0 + 0.01 * (i % 13);
    __syncthreads();
    const LaneP2 L = make_lane_p2(cx * (1 + 0.01 * dl), cy);
    double tx[K][T][NT], ty[K][NT];
    for (int k = 0; k < K; ++k)
        for (int r = 0; r < T; ++r)
            for (int t = 0; t < NT; ++t) tx[k][r][t] = 0.1 * t + r;
    for (int k = 0; k < K; ++k)
        for (int t = 0; t < NT; ++t) ty[k][t] = 0.2 * t;
    double acc = 0;
#pragma unroll 1
    for (int col = 0; col < ncols; ++col) {
#pragma unroll
        for (int r = 0; r < T; ++r) {
            double us[NQ];
#pragma unroll
            for (int k = 0; k < K; ++k) {
                double qh[NQ], u[NQ], txo[NT], tyo[NT];
#pragma unroll
                for (int m = 0; m < NQ; ++m) qh[m] = qs[(r * NQ + m) * GBK + gl + k * LG];
                const double st = ss[r * GBK + gl + k * LG];
                solve_p2(L, st, qh, tx[k][r], ty[k], u, txo, tyo);
#pragma unroll
                for (int t = 0; t < NT; ++t) {
                    tx[k][r][t] = txo[t];
                    ty[k][t] = tyo[t];
                }
#pragma unroll
                for (int m = 0; m < NQ; ++m) us[m] = (k == 0) ? u[m] : us[m] + u[m];
            }
            if constexpr (RED) {
                double* Sd = S + ((size_t)r * 8 + (dl & 7)) * NQ;
                auto sink = [&](int idx, double val) { Sd[idx] = val; };
                ReduceScatter<NQ, LG / 2>::run(us, lane, 0, NQ, sink);
            } else {
                acc += us[0] + us[4] + us[8];
            }
        }
    }
    out[blockIdx.x * blockDim.x + tid] = acc + tx[0][0][0] + ty[0][0] + S[tid % 64];
}

template <int K, int T, bool RED, int MINB, int LG = 32>
void run(const char* name, int warps, int ctas_per_sm, double* d) {
    const int nsm = 148, ncols = 512;
    const size_t smem = (size_t)(T * 9 * LG * K + T * LG * K + T * 8 * 9) * 8;
    cudaFuncSetAttribute(core_kernel<K, T, RED, MINB, LG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int bps = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, core_kernel<K, T, RED, MINB, LG>, 32 * warps, smem);
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, core_kernel<K, T, RED, MINB, LG>);
    const int grid = nsm * ctas_per_sm;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    core_kernel<K, T, RED, MINB, LG><<<grid, 32 * warps, smem>>>(d, 8, 0.3, 0.2);
    cudaEventRecord(a);
    core_kernel<K, T, RED, MINB, LG><<<grid, 32 * warps, smem>>>(d, ncols, 300.0, 200.0);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double lane_solves = (double)grid * 32 * warps * ncols * T * K;
    const double cyc = ms * 1e-3 * 1.965e9;
    // cycles per lane-solve per SMSP-equivalent: SMSP-cycles / (lane-solves / 32)
    const double per_warp_solve = cyc * nsm * 4 / (lane_solves / 32);
    printf("%-26s warps/SM %2d regs %3d occ(b/SM) %d: %.3f ms, %.1f SMSP-cycles per warp-solve, %.2e lane-solves/s\n",
           name, warps * ctas_per_sm, fa.numRegs, bps, ms, per_warp_solve, lane_solves / (ms * 1e-3));
    if (cudaGetLastError()) printf("  launch error\n");
}

int main() {
    double* d;
    cudaMalloc(&d, 64 << 20);
    ModalConsts mc;
    memset(&mc, 0, sizeof mc);
    mc.lam0 = 2.6258;
    mc.mu = 1.6871;
    mc.nu = 2.5087;
    for (int a = 0; a < 3; ++a) {
        mc.W0[a] = 0.3 + a;
        mc.W1re[a] = 0.2 * a;
        mc.W1im[a] = 0.1;
        mc.V0[a] = 0.5;
        mc.V1re[a] = 0.25;
        mc.V1im[a] = 0.125 * a;
    }
    cudaMemcpyToSymbol(cM, &mc, sizeof(ModalConsts));  // this unit's copy of the constants
    run<2, 4, true, 1>("K2 T4 red LG32", 8, 1, d);
    run<4, 2, true, 1, 16>("K4 T2 red LG16", 8, 1, d);
    run<4, 4, true, 1, 16>("K4 T4 red LG16", 8, 1, d);
    run<4, 2, false, 1, 16>("K4 T2 nored LG16", 8, 1, d);
    run<4, 2, true, 1, 8>("K4 T2 red LG8", 8, 1, d);
    run<8, 2, true, 1, 8>("K8 T2 red LG8", 8, 1, d);
    run<3, 2, true, 1, 16>("K3 T2 red LG16", 8, 1, d);
    run<4, 3, true, 1, 16>("K4 T3 red LG16", 8, 1, d);
    return 0;
}
