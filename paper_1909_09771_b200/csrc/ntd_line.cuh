// ntd_line.cuh -- warp-level twisted tridiagonal line solve.
//
// One warp solves one grid line (nx cells) of the innermost NTD level,
// i.e. the reference's _line_solve = _line_lower + _line_upper
// (/root/reference/pkg/src/ntdprecon/ntd_solve.py:107-137), whose chained
// recurrences _chain_scaled / _chain_unit (ntd_solve.py:20-104) become
// warp-shuffle affine-map scans instead of the reference's K=4 lane
// composition.  Result agrees with the reference to rounding (<=1e-15 rel);
// the parity bar is 1e-10 (BASELINE.json north_star).
//
// Slot layout for a line of n cells with twist t = (n-1)/2 (ntd_solve.py:110):
//   half h = lane/16: 0 = ascending chain (cells 0..t-1), 1 = descending
//   chain (cells n-1..t+1); sub-lane s = lane%16 holds chain indices
//   j = s*K .. s*K+K-1 (cell j for h=0, cell n-1-j for h=1).  Slots past the
//   chain length are identity maps.  K = ceil(n/32).
#pragma once
#include "common.cuh"

template <int K>
struct LineGeom {
    int n, t, h, s, L;
    __device__ __forceinline__ LineGeom(int n_, int lane)
    {
        n = n_;
        t = (n - 1) / 2;
        h = lane >> 4;
        s = lane & 15;
        L = h ? (n - 1 - t) : t;
    }
    __device__ __forceinline__ int j(int k) const { return s * K + k; }
    __device__ __forceinline__ bool valid(int k) const { return s * K + k < L; }
    __device__ __forceinline__ int cell(int k) const { return h ? n - 1 - (s * K + k) : s * K + k; }
};

// Solve T x = rhs for one line.  Per slot: mr (1/pivot), offL (lower-phase
// coupling: l1 on the ascending chain, u1 on the descending one), offU
// (upper-phase coupling: u1 ascending, l1 descending), rhs.  Twist cell
// scalars (same in every lane): bt, mrt, l1t, u1t.  Out: x per slot, xt.
template <int K>
__device__ __forceinline__ void line_solve(const LineGeom<K> &g, const double (&mr)[K], const double (&offL)[K],
                                           const double (&offU)[K], const double (&rhs)[K], double bt, double mrt,
                                           double l1t, double u1t, double (&x)[K], double &xt)
{
    // ---- lower phase: x_j = (rhs_j - offL_j x_{j-1}) mr_j, x_{-1} = 0.
    // Each lane composes its K affine maps, a 16-lane Kogge-Stone scan gives
    // the carry into the lane, and the lane re-walks its K slots from it
    // (no per-slot prefix storage: keeps registers for operand prefetch).
    double A = 1.0, C = 0.0;
#pragma unroll
    for (int k = 0; k < K; k++) {
        if (g.valid(k)) {
            const double a = -offL[k] * mr[k];
            C = fma(a, C, rhs[k] * mr[k]);
            A = a * A;
        }
    }
#pragma unroll
    for (int d = 1; d < 16; d <<= 1) {
        const double Ao = __shfl_up_sync(FULL_MASK, A, d, 16);
        const double Co = __shfl_up_sync(FULL_MASK, C, d, 16);
        if (g.s >= d) {
            C = fma(A, Co, C);
            A = A * Ao;
        }
    }
    double xc = __shfl_up_sync(FULL_MASK, C, 1, 16);
    if (g.s == 0) xc = 0.0;
#pragma unroll
    for (int k = 0; k < K; k++) {
        if (g.valid(k)) xc = fma(-offL[k] * mr[k], xc, rhs[k] * mr[k]);
        x[k] = xc;  // padding slots carry the chain end through
    }
    // ---- twist row (ntd_solve.py:115-121)
    const double xa = __shfl_sync(FULL_MASK, x[K - 1], 15);
    const double xd = __shfl_sync(FULL_MASK, x[K - 1], 31);
    double acc = bt;
    if (g.t > 0) acc -= l1t * xa;
    if (g.t < g.n - 1) acc -= u1t * xd;
    xt = acc * mrt;
    // ---- upper phase (ntd_solve.py:124-131): x_j -= mr_j offU_j x_{j+1},
    // walking from the twist outward; slot order reversed.
    A = 1.0;
    C = 0.0;
#pragma unroll
    for (int k = K - 1; k >= 0; k--) {
        if (g.valid(k)) {
            const double a = -(mr[k] * offU[k]);
            C = fma(a, C, x[k]);
            A = a * A;
        }
    }
#pragma unroll
    for (int d = 1; d < 16; d <<= 1) {
        const double Ao = __shfl_down_sync(FULL_MASK, A, d, 16);
        const double Co = __shfl_down_sync(FULL_MASK, C, d, 16);
        if (g.s + d < 16) {
            C = fma(A, Co, C);
            A = A * Ao;
        }
    }
    const double An = __shfl_down_sync(FULL_MASK, A, 1, 16);
    const double Cn = __shfl_down_sync(FULL_MASK, C, 1, 16);
    xc = (g.s == 15) ? xt : fma(An, xt, Cn);
#pragma unroll
    for (int k = K - 1; k >= 0; k--) {
        if (g.valid(k)) {
            xc = fma(-(mr[k] * offU[k]), xc, x[k]);
            x[k] = xc;
        }
    }
}

// Load the per-slot factor operands of one line whose cells start at `base`.
template <int K>
__device__ __forceinline__ void load_line_factors(const LineGeom<K> &g, const double *__restrict__ mr,
                                                  const double *__restrict__ l1, const double *__restrict__ u1,
                                                  i64 base, double (&omr)[K], double (&offL)[K], double (&offU)[K],
                                                  double &mrt, double &l1t, double &u1t)
{
#pragma unroll
    for (int k = 0; k < K; k++) {
        if (g.valid(k)) {
            i64 c = base + g.cell(k);
            double vl = l1[c], vu = u1[c];
            omr[k] = mr[c];
            offL[k] = g.h ? vu : vl;
            offU[k] = g.h ? vl : vu;
        } else {
            omr[k] = 0.0;
            offL[k] = 0.0;
            offU[k] = 0.0;
        }
    }
    i64 ct = base + g.t;
    mrt = mr[ct];
    l1t = l1[ct];
    u1t = u1[ct];
}

// Load one per-slot array (0 in padding slots) plus its twist-cell value.
template <int K>
__device__ __forceinline__ void load_slots(const LineGeom<K> &g, const double *__restrict__ p, i64 base,
                                           double (&v)[K], double &vt)
{
#pragma unroll
    for (int k = 0; k < K; k++) v[k] = g.valid(k) ? p[base + g.cell(k)] : 0.0;
    vt = p[base + g.t];
}

template <int K>
__device__ __forceinline__ void store_slots(const LineGeom<K> &g, double *__restrict__ p, i64 base,
                                            const double (&v)[K], double vt)
{
#pragma unroll
    for (int k = 0; k < K; k++)
        if (g.valid(k)) p[base + g.cell(k)] = v[k];
    if ((threadIdx.x & 31) == 0) p[base + g.t] = vt;
}
