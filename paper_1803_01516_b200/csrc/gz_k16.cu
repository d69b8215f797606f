// gz_k16.cu -- v4 instances for chains of at most 16 positions (m <= 16), and
// the window-relative 16-lane instances of the level-1/2 fine solves.
#include "gz_common.cuh"

namespace gz4 {

const void *kernels_lp16(bool win, int occ, int rw) {
    if (rw == 1) return (const void *)gz_tilesolve_kernel<16, 1, true, 1, 1>;
    if (rw == 2) return (const void *)gz_tilesolve_kernel<16, 1, true, 1, 2>;
    if (occ == 2) return win ? (const void *)gz_tilesolve_kernel<16, 1, true, 2> : (const void *)gz_tilesolve_kernel<16, 1, false, 2>;
    return win ? (const void *)gz_tilesolve_kernel<16, 1, true, 1> : (const void *)gz_tilesolve_kernel<16, 1, false, 1>;
}

const void *pairs_kernel_lp16(int occ) {
    return occ == 2 ? (const void *)gz_pairs_kernel<16, 1, 2> : (const void *)gz_pairs_kernel<16, 1, 1>;
}

}  // namespace gz4
