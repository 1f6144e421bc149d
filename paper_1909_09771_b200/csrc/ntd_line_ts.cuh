// ntd_line_ts.cuh -- two-sided line solve: every cell is a twist cell.
//
// The reference solves a factored line (ntd_solve.py:107-137) as a lower
// chain toward the twist row, the twist row, and an upper chain back out: two
// dependent scans per line.  For a tridiagonal T the same solution is
//     x_j = mu_j (f_j + g_j - r_j),
// with f the forward elimination of the rhs from the line's first cell
// (f_j = r_j - l_j f_{j-1} / delta_{j-1}), g the backward elimination from
// its last cell (g_j = r_j - u_j g_{j+1} / gamma_{j+1}) and 1 / mu_j =
// delta_j + gamma_j - d_j the twisted pivot *at cell j* (the reference's
// twist-row formula, ntd_solve.py:115-121, holds at every j when both
// eliminations are carried across the whole line).  f and g are independent
// first-order recurrences, so the two 32-lane scans run concurrently and the
// dependent chain per line is one scan deep instead of two.
//
// Scaled form (what the records hold): rho = mu r, f' = mu f, g' = mu g:
//     f'_j = rho_j + eF_j f'_{j-1},   eF_j = -l_j mu_j / (mu_{j-1} delta_{j-1})
//     g'_j = rho_j + eB_j g'_{j+1},   eB_j = -u_j mu_j / (mu_{j+1} gamma_{j+1})
//     x_j  = f'_j + g'_j - rho_j
// Lane l owns K consecutive cells.  Per lane the chains are composed as prefix
// maps (slot k: f'_k = pa_k cF + pf_k), the lane maps are scanned over the 32
// lanes (line_prep below) with multiplicative coefficients that depend only
// on the factor (PrepTS, prepared at setup), and each slot is finished with
// two FMAs once the carries arrive.
#pragma once
#include "common.cuh"

struct PrepTS {
    double m1, m2, m4, m8, e;  // forward: window multipliers of levels 1, 2, 4, 8 and the exclusive level (lane l-17)
    double n1, n2, n4, n8, f;  // backward
};

namespace ts {

// 64-bit shuffles, low half first: ptxas numbers the two result registers in
// issue order, and (low, high) in that order is an aligned register pair the
// following DFMA reads directly (the toolkit's double overload shuffles the
// high half first and costs two MOVs per shuffle in this kernel).
__device__ __forceinline__ double up(double v, int d)
{
    int lo, hi;
    asm("mov.b64 {%0, %1}, %2;" : "=r"(lo), "=r"(hi) : "d"(v));
    lo = __shfl_up_sync(FULL_MASK, lo, d);
    hi = __shfl_up_sync(FULL_MASK, hi, d);
    double r;
    asm("mov.b64 %0, {%1, %2};" : "=d"(r) : "r"(lo), "r"(hi));
    return r;
}
__device__ __forceinline__ double dn(double v, int d)
{
    int lo, hi;
    asm("mov.b64 {%0, %1}, %2;" : "=r"(lo), "=r"(hi) : "d"(v));
    lo = __shfl_down_sync(FULL_MASK, lo, d);
    hi = __shfl_down_sync(FULL_MASK, hi, d);
    double r;
    asm("mov.b64 %0, {%1, %2};" : "=d"(r) : "r"(lo), "r"(hi));
    return r;
}

// Factor-only scan coefficients of one line (setup; not on the apply path).
// The lane maps are scanned Kogge-Stone style: after the levels at distances
// 1, 2, 4, 8 lane l holds the composition of the 16 lanes ending at l
// (W_2d(l) = W_d(l) + M_d(l) W_d(l-d), M_d(l) the product of the lane
// multipliers of lanes l-d+1..l), and the exclusive carry of lane l is
// W_16(l-1) + M_16(l-1) W_16(l-17).  A shuffle costs a single warp ~6.5 issue
// cycles per 32-bit half, so the scan is shaped for the fewest shuffles (12
// per direction), not for the fewest levels.
template <int K>
__device__ __forceinline__ PrepTS line_prep(int l, const double (&eF)[K], const double (&eB)[K])
{
    PrepTS P;
    double A0 = 1.0, B0 = 1.0;
#pragma unroll
    for (int k = 0; k < K; k++) {
        A0 *= eF[k];
        B0 *= eB[k];
    }
    {  // forward: maps compose in increasing lane order
        const double M2 = A0 * up(A0, 1), M4 = M2 * up(M2, 2), M8 = M4 * up(M4, 4), M16 = M8 * up(M8, 8);
        const double e = up(M16, 1);
        P.m1 = l >= 1 ? A0 : 0.0;
        P.m2 = l >= 2 ? M2 : 0.0;
        P.m4 = l >= 4 ? M4 : 0.0;
        P.m8 = l >= 8 ? M8 : 0.0;
        P.e = l >= 17 ? e : 0.0;
    }
    {  // backward: maps compose in decreasing lane order
        const double M2 = B0 * dn(B0, 1), M4 = M2 * dn(M2, 2), M8 = M4 * dn(M4, 4), M16 = M8 * dn(M8, 8);
        const double f = dn(M16, 1);
        P.n1 = l <= 30 ? B0 : 0.0;
        P.n2 = l <= 29 ? M2 : 0.0;
        P.n4 = l <= 27 ? M4 : 0.0;
        P.n8 = l <= 23 ? M8 : 0.0;
        P.f = l <= 14 ? f : 0.0;
    }
    return P;
}

// One line (reference form, used by the micro-benchmarks): rho[k] = mu r of
// this lane's K cells, x[k] out.  The production kernel inlines the same
// sequence with its operand loads placed between the levels (ntd_apply_ts.cuh).
template <int K>
__device__ __forceinline__ void line_solve(const PrepTS &P, int l, const double (&eF)[K], const double (&eB)[K],
                                           const double (&rho)[K], double (&x)[K])
{
    double pf[K], pb[K], pa[K], qa[K];
    pf[0] = rho[0];
    pa[0] = eF[0];
    pb[K - 1] = rho[K - 1];
    qa[K - 1] = eB[K - 1];
#pragma unroll
    for (int k = 1; k < K; k++) {
        pf[k] = fma(eF[k], pf[k - 1], rho[k]);
        pa[k] = eF[k] * pa[k - 1];
        pb[K - 1 - k] = fma(eB[K - 1 - k], pb[K - k], rho[K - 1 - k]);
        qa[K - 1 - k] = eB[K - 1 - k] * qa[K - k];
    }
    double C = pf[K - 1], D = pb[0];
    C = fma(P.m1, up(C, 1), C);
    D = fma(P.n1, dn(D, 1), D);
    C = fma(P.m2, up(C, 2), C);
    D = fma(P.n2, dn(D, 2), D);
    C = fma(P.m4, up(C, 4), C);
    D = fma(P.n4, dn(D, 4), D);
    C = fma(P.m8, up(C, 8), C);
    D = fma(P.n8, dn(D, 8), D);
    const double u17 = up(C, 17), v17 = dn(D, 17), u1 = up(C, 1), v1 = dn(D, 1);
    const double cF = fma(P.e, u17, l >= 1 ? u1 : 0.0);
    const double cB = fma(P.f, v17, l <= 30 ? v1 : 0.0);
#pragma unroll
    for (int k = 0; k < K; k++) {
        const double R = k < K - 1 ? fma(eB[k], pb[k + 1 < K ? k + 1 : k], pf[k]) : pf[k];
        x[k] = fma(pa[k], cF, fma(qa[k], cB, R));
    }
}

}  // namespace ts
