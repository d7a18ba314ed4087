// k2d_opt_p1.cu — instantiates the 2-D p = 1 sweep kernels with options (sigma moments, fixup) (compiled in parallel with the other k_*.cu units).
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

const void* pick2d_opt_p1(int log2lg, int k, int opt) {
    // options are instantiated for the default layouts only: 1 group per lane (any lane
    // count) and the many-group layout (16 lanes x 4 groups)
    if (k == 4) {
        if (log2lg != 4) return nullptr;
        switch (opt) {
            case 1: return (const void*)sweep2d_kernel<1, 4, 4, 1>;
            case 2: return (const void*)sweep2d_kernel<1, 4, 4, 2>;
            case 3: return (const void*)sweep2d_kernel<1, 4, 4, 3>;
            default: return nullptr;
        }
    }
    if (k != 1) return nullptr;
    switch (opt) {
        case 1: return pick_lg<1, 1>(log2lg);
        case 2: return pick_lg<1, 2>(log2lg);
        case 3: return pick_lg<1, 3>(log2lg);
        default: return nullptr;
    }
}

int upload_modal_opt_p1(const ModalConsts& mc) { return (int)cudaMemcpyToSymbol(cM, &mc, sizeof(ModalConsts)); }

}  // namespace sweepk
