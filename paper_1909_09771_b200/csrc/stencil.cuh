// stencil.cuh -- one row of the 7-point SpMV in the reference's summation
// order (banded_core.py:105-118), exactly rounded, from the 7-band operator
// or its symmetric 4-band pack.  Shared by blas.cu and the slot-layout fused
// residuals in ntd.cu.
#pragma once
#include "common.cuh"

// One row of the reference SpMV (banded_core.py:105-118), exactly rounded.
__device__ __forceinline__ double spmv_row(const double *__restrict__ a, const double *__restrict__ x,
                                           i64 r, i64 n, i64 nx, i64 nxy)
{
    double s = mul_rn(a[3 * n + r], x[r]);
    if (r >= 1) s = add_rn(s, mul_rn(a[2 * n + r], x[r - 1]));
    if (r >= nx) s = add_rn(s, mul_rn(a[n + r], x[r - nx]));
    if (r >= nxy) s = add_rn(s, mul_rn(a[r], x[r - nxy]));
    if (r + 1 < n) s = add_rn(s, mul_rn(a[4 * n + r], x[r + 1]));
    if (r + nx < n) s = add_rn(s, mul_rn(a[5 * n + r], x[r + nx]));
    if (r + nxy < n) s = add_rn(s, mul_rn(a[6 * n + r], x[r + nxy]));
    return s;
}

// The same row from the symmetric packed operator (4 bands: 0, +1, +nx, +nxy):
// A[r][r-d] is read as A[r-d][r].  ntd_sym_pack only produces this layout when
// every mirrored pair is bitwise equal, so the result is bitwise spmv_row's.
__device__ __forceinline__ double spmv_row4(const double *__restrict__ a, const double *__restrict__ x,
                                            i64 r, i64 n, i64 nx, i64 nxy)
{
    double s = mul_rn(a[r], x[r]);
    if (r >= 1) s = add_rn(s, mul_rn(a[n + r - 1], x[r - 1]));
    if (r >= nx) s = add_rn(s, mul_rn(a[2 * n + r - nx], x[r - nx]));
    if (r >= nxy) s = add_rn(s, mul_rn(a[3 * n + r - nxy], x[r - nxy]));
    if (r + 1 < n) s = add_rn(s, mul_rn(a[n + r], x[r + 1]));
    if (r + nx < n) s = add_rn(s, mul_rn(a[2 * n + r], x[r + nx]));
    if (r + nxy < n) s = add_rn(s, mul_rn(a[3 * n + r], x[r + nxy]));
    return s;
}
template <int NB>
__device__ __forceinline__ double row_of(const double *__restrict__ a, const double *__restrict__ x, i64 r, i64 n,
                                         i64 nx, i64 nxy)
{
    if constexpr (NB == 4)
        return spmv_row4(a, x, r, n, nx, nxy);
    else
        return spmv_row(a, x, r, n, nx, nxy);
}

