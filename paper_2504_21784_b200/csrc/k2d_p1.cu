// k2d_p1.cu — instantiates the 2-D p = 1 sweep kernels without options (compiled in parallel with the other k_*.cu units).
#define SWEEP_TRACE_OWNER sweep_debug_trace_p1
#include "sweep_device.cuh"

namespace sweepk {

template <int K, int OPT>
static const void* pick_lg(int log2lg) {
    switch (log2lg) {
        case 0: return (const void*)sweep2d_kernel<1, 0, K, OPT>;
        case 1: return (const void*)sweep2d_kernel<1, 1, K, OPT>;
        case 2: return (const void*)sweep2d_kernel<1, 2, K, OPT>;
        case 3: return (const void*)sweep2d_kernel<1, 3, K, OPT>;
        case 4: return (const void*)sweep2d_kernel<1, 4, K, OPT>;
        default: return (const void*)sweep2d_kernel<1, 5, K, OPT>;
    }
}

const void* pick2d_p1(int log2lg, int k) {
    // K = 2 and K = 4 are the many-group layouts (K = 2 only via the SWEEP_CFG experiment override)
    return (k == 4) ? pick_lg<4, 0>(log2lg) : (k == 2) ? pick_lg<2, 0>(log2lg) : pick_lg<1, 0>(log2lg);
}

int upload_modal_p1(const ModalConsts& mc) { return (int)cudaMemcpyToSymbol(cM, &mc, sizeof(ModalConsts)); }

}  // namespace sweepk
