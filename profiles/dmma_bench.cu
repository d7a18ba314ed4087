// dmma_bench.cu — does FP64 mma.sync (DMMA) issue outside the DFMA pipe on sm_100a?
// Throughput of DFMA alone, DMMA alone, and both interleaved in one instruction stream.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/dmma profiles/dmma_bench.cu && /tmp/dmma
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

// MODE 0: DFMA only (8 chains); 1: DMMA only (8 accumulators); 2: both (8 + 8)
template <int MODE>
__global__ void __launch_bounds__(256) kern(double* sink, int iters, double b, double c) {
    double f[8], m0[8], m1[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        f[k] = threadIdx.x * 1e-3 + k;
        m0[k] = m1[k] = 1e-3 * k;
    }
    const double a = 1.0 + threadIdx.x * 1e-9;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            if (MODE != 1) {
#pragma unroll
                for (int k = 0; k < 8; ++k) f[k] = fma(f[k], b, c);
            }
            if (MODE != 0) {
#pragma unroll
                for (int k = 0; k < 8; ++k) dmma(m0[k], m1[k], a, b);
            }
        }
    }
    double r = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) r += f[k] + m0[k] + m1[k];
    if (r == 1.2345) sink[threadIdx.x] = r;
}

template <int MODE>
double run(int nsm, int bps, int iters) {
    double* sink;
    cudaMalloc(&sink, 4096);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    kern<MODE><<<nsm * bps, 256>>>(sink, 16, 0.999999, 1e-7);
    float best = 1e30f;
    for (int r = 0; r < 3; ++r) {
        cudaEventRecord(a);
        kern<MODE><<<nsm * bps, 256>>>(sink, iters, 0.999999, 1e-7);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        best = ms < best ? ms : best;
    }
    const double threads = (double)nsm * bps * 256;
    const double fl_dfma = (MODE != 1) ? 2.0 * 8 * 8 * iters * threads : 0;
    const double fl_dmma = (MODE != 0) ? 512.0 * 8 * 8 * iters * (threads / 32) : 0;
    printf("mode %d bps %d: %.3f ms  DFMA %.2f TF  DMMA %.2f TF  total %.2f TF  (%s)\n", MODE, bps, best,
           fl_dfma / best / 1e9, fl_dmma / best / 1e9, (fl_dfma + fl_dmma) / best / 1e9,
           cudaGetErrorString(cudaGetLastError()));
    cudaFree(sink);
    return best;
}

int main() {
    int nsm;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    printf("SMs %d\n", nsm);
    for (int bps : {2, 4, 8}) {
        run<0>(nsm, bps, 512);
        run<1>(nsm, bps, 512);
        run<2>(nsm, bps, 512);
    }
    return 0;
}
