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
// Per-system block cap of the bandwidth-bound row kernels (8 blocks per SM).
i64 rows_block_cap();
}  // namespace ntd

#define NTD_CHECK_LAUNCH(name) return ntd::check_launch(name)
