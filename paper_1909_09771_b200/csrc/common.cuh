// common.cuh -- shared helpers for the sm_100a NTD-PCG kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/ntdgpu.h"

typedef int64_t i64;

#define FULL_MASK 0xffffffffu

// Exactly-rounded fp64 ops that ptxas may not contract into FMA.  Used
// wherever bitwise parity with the reference (numba, no fastmath) is kept.
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }

__device__ __forceinline__ bool is_finite(double v) { return isfinite(v); }

// Named barrier over `nthreads` threads of the CTA (id 1..15; 0 = __syncthreads).
__device__ __forceinline__ void named_bar(int id, int nthreads)
{
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// L2 prefetch of a byte range (Hopper+ bulk prefetch; 16-B aligned, size%16==0).
__device__ __forceinline__ void prefetch_l2_bulk(const void *p, unsigned bytes)
{
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
__device__ __forceinline__ void prefetch_l2(const void *p)
{
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

namespace ntd {
void set_error(const char *where, cudaError_t e);
int check_launch(const char *where);
}  // namespace ntd

#define NTD_CHECK_LAUNCH(name) return ntd::check_launch(name)

namespace ntd {
// Blocks of 256 threads per system for a grid-stride kernel over `rows`
// rows: one full wave of the kernel on the GPU (SMs x resident blocks per SM,
// from the occupancy of this kernel instantiation), fewer for small systems.
// A fixed 8 blocks per SM left a partial second wave for kernels whose
// register count allows only 5-6 resident blocks.
template <auto K>
unsigned fill_grid(i64 rows)
{
    static int wave = 0;  // per kernel instantiation (same on every B200)
    if (wave == 0) {
        int occ = 0, sms = 0, dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, K, 256, 0);
        wave = (occ > 0 ? occ : 1) * (sms > 0 ? sms : 148);
    }
    const i64 b = (rows + 255) / 256;
    return (unsigned)(b < wave ? (b > 0 ? b : 1) : wave);
}
}  // namespace ntd
