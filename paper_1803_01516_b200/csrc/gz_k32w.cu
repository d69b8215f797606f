// gz_k32w.cu -- v4 instances for chains of four or eight 32-lane segments (64 < m <= 256).
#include "gz_common.cuh"

namespace gz4 {

const void *kernels_lp32w(int R, bool win) {
    if (R == 4) return win ? (const void *)gz_tilesolve_kernel<32, 4, true, 1> : (const void *)gz_tilesolve_kernel<32, 4, false, 1>;
    if (R == 8) return win ? (const void *)gz_tilesolve_kernel<32, 8, true, 1> : (const void *)gz_tilesolve_kernel<32, 8, false, 1>;
    return nullptr;
}

}  // namespace gz4
