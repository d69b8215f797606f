// gz_common.cuh -- device code shared by every translation unit of
// libgazecut_b200.so: the implicit graph (gz_graph.cuh), bit-word helpers
// (gz_bits.cuh), the per-chain warp machinery (gz_chain.cuh) and the v4 solve
// kernel template (gz_tilesolve.cuh).
//
// The v4 kernel instances are compiled in their own translation units
// (gz_k16.cu, gz_k32.cu, gz_k32w.cu, built in parallel) and handed to the host
// code in gz_solver.cu as launchable function pointers through
// gz4::kernel_for (declared below, defined in gz_solver.cu).
#pragma once

#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "gazecut_b200.h"
#include "gz_graph.cuh"

namespace gz {

// warp-reduced 64-bit counter add: one atomic per warp
__device__ __forceinline__ void warp_add_u64(unsigned long long *dst, long long v, int sys = 0) {
    unsigned long long x = (unsigned long long)v;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
    if ((threadIdx.x & 31) == 0 && x) {
        if (sys) atomicAdd_system(dst, x);
        else atomicAdd(dst, x);
    }
}

}  // namespace gz

#include "gz_bits.cuh"
#include "gz_chain.cuh"
#include "gz_tilesolve.cuh"

namespace gz4 {

// Launchable v4 instance for chains of LP lanes x R segments (RW > 0: the
// window-relative 16-lane instance over rows of 32 RW positions), or nullptr.
const void *kernel_for(int LP, int R, bool win, int occ, int rw);
// per translation unit
const void *kernels_lp16(bool win, int occ, int rw);
const void *kernels_lp32(int R, bool win);
const void *kernels_lp32w(int R, bool win);
// the batched pair-solve kernel (gz_pairs_kernel) for 16-lane chains, occupancy 1 or 2
const void *pairs_kernel_lp16(int occ);

}  // namespace gz4
