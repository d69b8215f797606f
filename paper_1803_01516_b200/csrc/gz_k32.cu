// gz_k32.cu -- v4 instances for chains of one or two 32-lane segments (16 < m <= 64).
#include "gz_common.cuh"

namespace gz4 {

const void *kernels_lp32(int R, bool win) {
    if (R == 1) return win ? (const void *)gz_tilesolve_kernel<32, 1, true, 1> : (const void *)gz_tilesolve_kernel<32, 1, false, 1>;
    if (R == 2) return win ? (const void *)gz_tilesolve_kernel<32, 2, true, 1> : (const void *)gz_tilesolve_kernel<32, 2, false, 1>;
    return nullptr;
}

}  // namespace gz4
