// handoff_bench.cu — latency of a strip-to-strip hand-off between two CTAs on sm_100a:
//  (a) global: producer stores a payload + st.release.gpu flag; consumer polls ld.relaxed.gpu,
//      ld.acquire, then loads the payload (the sweep's current trace ring protocol);
//  (b) DSMEM: producer stores the payload into the consumer's shared memory
//      (st.shared::cluster) + st.release.cluster flag in the consumer's smem; consumer polls its
//      own shared memory with ld.acquire.cluster.
// Ping-pong N rounds between the two CTAs (cluster of 2); one-way latency = time / (2N).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/hb profiles/handoff_bench.cu && /tmp/hb
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

constexpr int PAY = 256;  // doubles per hand-off (one trace column of 256 lanes)

__device__ __forceinline__ int ld_relaxed(const int* p) {
    int v;
    asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ int ld_acq(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_rel(int* p, int v) { asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory"); }

__global__ void __cluster_dims__(2, 1, 1) pingpong_global(int* flags, double* buf, int n, long long* cyc) {
    const int me = blockIdx.x & 1, other = me ^ 1;
    const int tid = threadIdx.x;
    long long t0 = clock64();
    double acc = 0;
    for (int r = 0; r < n; ++r) {
        const int turn = 2 * r + me;  // CTA 0 sends at even turns
        if (turn > 0) {
            if (tid == 0) {
                while (ld_relaxed(flags + me) < turn) {
                }
                (void)ld_acq(flags + me);
            }
            __syncthreads();
            acc += __ldcg(buf + (size_t)me * PAY + tid);  // payload written by the other CTA
        }
        __stcg(buf + (size_t)other * PAY + tid, acc + r);
        __syncthreads();
        if (tid == 0) st_rel(flags + other, turn + 1);
    }
    if (tid == 0) cyc[me] = clock64() - t0;
    if (acc == 1.2345) buf[0] = acc;
}

__global__ void __cluster_dims__(2, 1, 1) pingpong_dsmem(int n, long long* cyc, double* sink) {
    __shared__ double pay[PAY];
    __shared__ int flag;
    cg::cluster_group cl = cg::this_cluster();
    const int me = cl.block_rank(), other = me ^ 1;
    const int tid = threadIdx.x;
    if (tid == 0) flag = 0;
    cl.sync();
    double* rpay = cl.map_shared_rank(pay, other);
    int* rflag = cl.map_shared_rank(&flag, other);
    const unsigned lflag = (unsigned)__cvta_generic_to_shared(&flag);
    long long t0 = clock64();
    double acc = 0;
    for (int r = 0; r < n; ++r) {
        const int turn = 2 * r + me;
        if (turn > 0) {
            if (tid == 0) {
                int v = 0;
                do {
                    asm volatile("ld.acquire.cluster.shared::cta.s32 %0, [%1];" : "=r"(v) : "r"(lflag) : "memory");
                } while (v < turn);
            }
            __syncthreads();
            acc += pay[tid];
        }
        rpay[tid] = acc + r;  // remote store into the other CTA's shared memory
        __syncthreads();
        if (tid == 0) {
            asm volatile("fence.acq_rel.cluster;" ::: "memory");
            asm volatile("st.relaxed.cluster.shared::cluster.s32 [%0], %1;" ::"l"(rflag), "r"(turn + 1) : "memory");
        }
    }
    if (tid == 0) cyc[me] = clock64() - t0;
    cl.sync();
    if (acc == 1.2345) sink[0] = acc;
}

int main() {
    int *flags;
    double* buf;
    long long* cyc;
    cudaMalloc(&flags, 64);
    cudaMalloc(&buf, 2 * PAY * sizeof(double));
    cudaMalloc(&cyc, 16);
    const int n = 2000;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int rep = 0; rep < 2; ++rep) {
        cudaMemset(flags, 0, 64);
        cudaEventRecord(a);
        pingpong_global<<<2, PAY>>>(flags, buf, n, cyc);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("global ring + flags: %.3f us per one-way hand-off (%s)\n", ms * 1e3 / (2 * n),
               cudaGetErrorString(cudaGetLastError()));
        cudaEventRecord(a);
        pingpong_dsmem<<<2, PAY>>>(n, cyc, buf);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("DSMEM store + cluster flag: %.3f us per one-way hand-off (%s)\n", ms * 1e3 / (2 * n),
               cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
