// microbench.cu — FP64 latency / throughput probes on B200 (sm_100a).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb profiles/microbench.cu && /tmp/mb
#include <cstdio>
#include <cuda_runtime.h>

__global__ void lat_dfma(double* out, long long* cyc, int n, double b, double c) {
    double a = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int k = 0; k < 32; ++k) a = fma(a, b, c);
    }
    long long t1 = clock64();
    out[threadIdx.x] = a;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void lat_dmul(double* out, long long* cyc, int n, double b) {
    double a = threadIdx.x + 1;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int k = 0; k < 32; ++k) a = a * b;
    }
    long long t1 = clock64();
    out[threadIdx.x] = a;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void lat_rcp(double* out, long long* cyc, int n) {
    double a = threadIdx.x + 1.5;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int k = 0; k < 32; ++k) {
            double y;
            asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(a));
            a = y + 1.0;
        }
    }
    long long t1 = clock64();
    out[threadIdx.x] = a;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void lat_lds(double* out, long long* cyc, int n) {
    __shared__ double buf[256];
    buf[threadIdx.x] = threadIdx.x % 7;
    __syncthreads();
    int idx = threadIdx.x & 7;
    long long t0 = clock64();
    for (int i = 0; i < n * 32; ++i) idx = (int)buf[idx];
    long long t1 = clock64();
    out[threadIdx.x] = idx;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
// throughput with ILP chains per thread
template <int ILP>
__global__ void thr_dfma(double* out, int n, double b, double c) {
    double a[ILP];
#pragma unroll
    for (int j = 0; j < ILP; ++j) a[j] = threadIdx.x + j;
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k)
#pragma unroll
            for (int j = 0; j < ILP; ++j) a[j] = fma(a[j], b, c);
    }
    double s = 0;
#pragma unroll
    for (int j = 0; j < ILP; ++j) s += a[j];
    if (s == 1.234) out[threadIdx.x] = s;
}

int main() {
    double* d;
    long long* c;
    cudaMalloc(&d, 1 << 20);
    cudaMalloc(&c, 64);
    long long h;
    const int n = 1000;
    lat_dfma<<<1, 32>>>(d, c, n, 0.999, 1e-3);
    lat_dfma<<<1, 32>>>(d, c, n, 0.999, 1e-3);
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("DFMA dependent latency: %.2f cycles\n", (double)h / (n * 32));
    lat_dmul<<<1, 32>>>(d, c, n, 0.9999);
    lat_dmul<<<1, 32>>>(d, c, n, 0.9999);
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("DMUL dependent latency: %.2f cycles\n", (double)h / (n * 32));
    lat_rcp<<<1, 32>>>(d, c, n);
    lat_rcp<<<1, 32>>>(d, c, n);
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("MUFU.RCP64H + DADD dependent latency: %.2f cycles\n", (double)h / (n * 32));
    lat_lds<<<1, 32>>>(d, c, n);
    lat_lds<<<1, 32>>>(d, c, n);
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("LDS.64 + F2I dependent latency: %.2f cycles\n", (double)h / (n * 32));
    int nsm;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int warps = 1; warps <= 16; warps *= 2) {
        for (int ilp = 1; ilp <= 8; ilp *= 2) {
            const int iters = 2000;
            auto launch = [&]() {
                if (ilp == 1) thr_dfma<1><<<nsm, 32 * warps>>>(d, iters, 0.999, 1e-3);
                if (ilp == 2) thr_dfma<2><<<nsm, 32 * warps>>>(d, iters, 0.999, 1e-3);
                if (ilp == 4) thr_dfma<4><<<nsm, 32 * warps>>>(d, iters, 0.999, 1e-3);
                if (ilp == 8) thr_dfma<8><<<nsm, 32 * warps>>>(d, iters, 0.999, 1e-3);
            };
            launch();
            cudaEventRecord(e0);
            launch();
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            double fl = 2.0 * iters * 8 * ilp * 32.0 * warps * nsm;
            printf("warps/SM %2d ILP %d: %.2f TFLOP/s\n", warps, ilp, fl / (ms * 1e-3) / 1e12);
        }
    }
    printf("SMs %d, clock %d kHz\n", nsm, clk);
    return 0;
}
