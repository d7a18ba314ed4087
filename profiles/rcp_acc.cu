// accuracy of rcp.approx.ftz.f64 and of the refinements used by the kernels
#include <cstdio>
#include <cmath>
#include <cuda_runtime.h>
__global__ void k(const double* x, double* seed, double* cubic, double* both, int n) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double v = x[i], y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(v));
    seed[i] = y;
    double e = fma(-v, y, 1.0);
    double y1 = fma(y, fma(e, e, e), y);
    cubic[i] = y1;
    e = fma(-v, y1, 1.0);
    both[i] = fma(y1, e, y1);
}
int main() {
    const int n = 1 << 22;
    double* h = new double[n];
    unsigned long long s = 88172645463325252ull;
    for (int i = 0; i < n; ++i) {
        s ^= s << 13; s ^= s >> 7; s ^= s << 17;
        double u = (s >> 11) * (1.0 / 9007199254740992.0);
        h[i] = exp(-30.0 + 120.0 * u);  // 1e-13 .. 1e39
    }
    double *dx, *a, *b, *c;
    cudaMalloc(&dx, n * 8); cudaMalloc(&a, n * 8); cudaMalloc(&b, n * 8); cudaMalloc(&c, n * 8);
    cudaMemcpy(dx, h, n * 8, cudaMemcpyHostToDevice);
    k<<<n / 256, 256>>>(dx, a, b, c, n);
    double *ha = new double[n], *hb = new double[n], *hc = new double[n];
    cudaMemcpy(ha, a, n * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(hb, b, n * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(hc, c, n * 8, cudaMemcpyDeviceToHost);
    double ea = 0, eb = 0, ec = 0;
    for (int i = 0; i < n; ++i) {
        double r = 1.0 / h[i];
        ea = fmax(ea, fabs(ha[i] - r) / r);
        eb = fmax(eb, fabs(hb[i] - r) / r);
        ec = fmax(ec, fabs(hc[i] - r) / r);
    }
    printf("max rel err: seed %.3e (2^%.1f)  cubic %.3e  cubic+newton %.3e  (ulp %.3e)\n", ea, log2(ea), eb, ec,
           ldexp(1.0, -53));
    return 0;
}
