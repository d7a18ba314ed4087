// k2d_p2.cu — instantiates the 2-D p = 2 sweep kernels without options (compiled in parallel with the other k_*.cu units).
#define SWEEP_TRACE_OWNER sweep_debug_trace
#include "sweep_device.cuh"

namespace sweepk {

template <int K, int OPT>
static const void* pick_lg(int log2lg) {
    switch (log2lg) {
        case 0: return (const void*)sweep2d_kernel<2, 0, K, OPT>;
        case 1: return (const void*)sweep2d_kernel<2, 1, K, OPT>;
        case 2: return (const void*)sweep2d_kernel<2, 2, K, OPT>;
        case 3: return (const void*)sweep2d_kernel<2, 3, K, OPT>;
        case 4: return (const void*)sweep2d_kernel<2, 4, K, OPT>;
        default: return (const void*)sweep2d_kernel<2, 5, K, OPT>;
    }
}

const void* pick2d_p2(int log2lg, int k) {
    // K = 2 and K = 4 are the many-group layouts (K = 2 only via the SWEEP_CFG experiment override)
    return (k == 4) ? pick_lg<4, 0>(log2lg) : (k == 2) ? pick_lg<2, 0>(log2lg) : pick_lg<1, 0>(log2lg);
}

int upload_modal_p2(const ModalConsts& mc) { return (int)cudaMemcpyToSymbol(cM, &mc, sizeof(ModalConsts)); }

}  // namespace sweepk
