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
// lanes in three sliding-window levels (4, 4, 2) whose multiplicative
// coefficients depend only on the factor (PrepTS, prepared at setup), and
// each slot is finished with two FMAs once the carries arrive.
#pragma once
#include "common.cuh"

struct PrepTS {
    double p1, p2, p3;  // forward level 1 (lanes l-1, l-2, l-3)
    double s1, s2, s3;  // forward level 2 (lanes l-4, l-8, l-12)
    double e1;          // forward level 3, exclusive (lane l-17)
    double q1, q2, q3;  // backward level 1 (lanes l+1, l+2, l+3)
    double t1, t2, t3;  // backward level 2 (lanes l+4, l+8, l+12)
    double f1;          // backward level 3, exclusive (lane l+17)
};

namespace ts {

__device__ __forceinline__ double up(double v, int d) { return __shfl_up_sync(FULL_MASK, v, d); }
__device__ __forceinline__ double dn(double v, int d) { return __shfl_down_sync(FULL_MASK, v, d); }

// Ordered shuffles for the solve: volatile asm statements keep their program
// order, so the forward and backward scans stay interleaved level by level
// (the warp issues in order; ptxas otherwise runs one scan after the other).
__device__ __forceinline__ double vup(double v, int d)
{
    int lo = __double2loint(v), hi = __double2hiint(v);
    asm volatile("shfl.sync.up.b32 %0, %0, %2, 0, 0xffffffff;\n\tshfl.sync.up.b32 %1, %1, %2, 0, 0xffffffff;"
                 : "+r"(lo), "+r"(hi)
                 : "r"(d));
    return __hiloint2double(hi, lo);
}
__device__ __forceinline__ double vdn(double v, int d)
{
    int lo = __double2loint(v), hi = __double2hiint(v);
    asm volatile("shfl.sync.down.b32 %0, %0, %2, 0x1f, 0xffffffff;\n\tshfl.sync.down.b32 %1, %1, %2, 0x1f, 0xffffffff;"
                 : "+r"(lo), "+r"(hi)
                 : "r"(d));
    return __hiloint2double(hi, lo);
}

// Factor-only scan coefficients of one line (setup; not on the apply path).
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
        const double a1 = up(A0, 1), a2 = up(A0, 2), a3 = up(A0, 3);
        const double A01 = A0 * a1, A012 = A01 * a2, A1 = A012 * (l >= 3 ? a3 : 1.0);
        P.p1 = l >= 1 ? A0 : 0.0;
        P.p2 = l >= 2 ? A01 : 0.0;
        P.p3 = l >= 3 ? A012 : 0.0;
        const double b4 = up(A1, 4), b8 = up(A1, 8), b12 = up(A1, 12);
        const double A14 = A1 * b4, A148 = A14 * b8, A2 = A148 * (l >= 12 ? b12 : 1.0);
        P.s1 = l >= 4 ? A1 : 0.0;
        P.s2 = l >= 8 ? A14 : 0.0;
        P.s3 = l >= 12 ? A148 : 0.0;
        const double c1 = up(A2, 1);
        P.e1 = l >= 17 ? c1 : 0.0;
    }
    {  // backward: maps compose in decreasing lane order
        const double a1 = dn(B0, 1), a2 = dn(B0, 2), a3 = dn(B0, 3);
        const double B01 = B0 * a1, B012 = B01 * a2, B1 = B012 * (l <= 28 ? a3 : 1.0);
        P.q1 = l <= 30 ? B0 : 0.0;
        P.q2 = l <= 29 ? B01 : 0.0;
        P.q3 = l <= 28 ? B012 : 0.0;
        const double b4 = dn(B1, 4), b8 = dn(B1, 8), b12 = dn(B1, 12);
        const double B14 = B1 * b4, B148 = B14 * b8, B2 = B148 * (l <= 19 ? b12 : 1.0);
        P.t1 = l <= 27 ? B1 : 0.0;
        P.t2 = l <= 23 ? B14 : 0.0;
        P.t3 = l <= 19 ? B148 : 0.0;
        const double c1 = dn(B2, 1);
        P.f1 = l <= 14 ? c1 : 0.0;
    }
    return P;
}

// Local (carry-free) part of a line solve: prefix maps of both chains and the
// carry-independent remainder R_k = pf_k + eB_k pb_{k+1} (= pf_k + pb_k - rho_k).
template <int K>
struct LocalTS {
    double pa[K], qa[K], R[K];
    double C0, D0;
};

// One line.  rho[k] = mu r (this lane's K cells), x[k] out.  `l` = lane.
// SUB: x = y - T^{-1} r instead (the level-2/3 upper sweeps), y passed in x.
template <int K, bool SUB = false, bool ORD = true>
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
    const double C0 = pf[K - 1], D0 = pb[0];
    // level 1
    auto U = [](double v, int d) { return ORD ? vup(v, d) : up(v, d); };
    auto Dn = [](double v, int d) { return ORD ? vdn(v, d) : dn(v, d); };
    const double c3 = U(C0, 3), d3 = Dn(D0, 3), c2 = U(C0, 2), d2 = Dn(D0, 2), c1 = U(C0, 1), d1 = Dn(D0, 1);
    const double C1 = fma(P.p1, c1, C0) + fma(P.p2, c2, P.p3 * c3);
    const double D1 = fma(P.q1, d1, D0) + fma(P.q2, d2, P.q3 * d3);
    // level 2
    const double c12 = U(C1, 12), c8 = U(C1, 8), c4 = U(C1, 4);
    const double d12 = Dn(D1, 12), d8 = Dn(D1, 8), d4 = Dn(D1, 4);
    const double C2 = fma(P.s1, c4, C1) + fma(P.s2, c8, P.s3 * c12);
    const double D2 = fma(P.t1, d4, D1) + fma(P.t2, d8, P.t3 * d12);
    // level 3: exclusive carries
    const double u17 = U(C2, 17), u1 = U(C2, 1);
    const double v17 = Dn(D2, 17), v1 = Dn(D2, 1);
    const double cF = fma(P.e1, u17, l >= 1 ? u1 : 0.0);
    const double cB = fma(P.f1, v17, l <= 30 ? v1 : 0.0);
#pragma unroll
    for (int k = 0; k < K; k++) {
        const double R = k < K - 1 ? fma(eB[k], pb[k + 1 < K ? k + 1 : k], pf[k]) : pf[k];
        if (SUB)
            x[k] = fma(-pa[k], cF, fma(-qa[k], cB, x[k] - R));
        else
            x[k] = fma(pa[k], cF, fma(qa[k], cB, R));
    }
}

}  // namespace ts
