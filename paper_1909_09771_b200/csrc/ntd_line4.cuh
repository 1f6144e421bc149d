// ntd_line4.cuh -- radix-4 two-level warp scans for the twisted line solve.
//
// Same mathematics as sl::line_solve (the reference's _line_solve,
// ntd_solve.py:107-137): a lower first-order chain per half-warp, the twist
// row, then an upper chain seeded by the twist value.  The 16-lane
// affine-map scans are done in two radix-4 levels; every multiplicative
// coefficient of the scan depends only on the factor, so it is prepared
// (line_prep) one line ahead, off the critical path, and the per-line work
// (line_solve4) only carries the right-hand-side chain:
//   lower:  compose -> 3 shuffles -> C1 -> 4 shuffles -> exclusive carry -> re-walk
//   twist:  2 shuffles                                    } concurrent
//   upper:  compose -> 3 shuffles -> D1 -> 4 shuffles     }
//           -> carry = Dex + Bex * x_twist -> re-walk
#pragma once
#include "common.cuh"

struct LinePrep {
    double p1, p2, p3;          // lower level-1 coefficients
    double e0, e1, e2, e3;      // lower level-2 (exclusive) coefficients
    double q1, q2, q3;          // upper level-1 coefficients
    double f0, f1, f2, f3, bex; // upper level-2 (exclusive) coefficients, seed factor
};

__device__ __forceinline__ double shup(double v, int d) { return __shfl_up_sync(FULL_MASK, v, d, 16); }
__device__ __forceinline__ double shdn(double v, int d) { return __shfl_down_sync(FULL_MASK, v, d, 16); }

// s = lane within the 16-lane half; aL/aU = chain coefficients of this lane's slots
template <int K>
__device__ __forceinline__ LinePrep line_prep(int s, const double (&aL)[K], const double (&aU)[K])
{
    // Branch-free: every lane-dependent choice is a single select (FSEL),
    // never a multi-way conditional (which compiles to divergent jumps).
    LinePrep P;
    double A0 = 1.0, B0 = 1.0;
#pragma unroll
    for (int k = 0; k < K; k++) {
        A0 *= aL[k];
        B0 *= aU[k];
    }
    const bool g1 = s >= 1, g2 = s >= 2, g3 = s >= 3;
    // lower: maps compose in increasing lane order
    const double a1 = shup(A0, 1), a2 = shup(A0, 2), a3 = shup(A0, 3);
    const double m1 = g1 ? a1 : 1.0, m2 = g2 ? a2 : 1.0, m3 = g3 ? a3 : 1.0;
    const double A01 = A0 * a1, A012 = A01 * a2;
    P.p1 = g1 ? A0 : 0.0;
    P.p2 = g2 ? A01 : 0.0;
    P.p3 = g3 ? A012 : 0.0;
    const double A1 = ((A0 * m1) * m2) * m3;
    const double b1 = shup(A1, 1), b5 = shup(A1, 5), b9 = shup(A1, 9);
    const double b15 = b1 * b5;
    P.e0 = g1 ? 1.0 : 0.0;
    P.e1 = s >= 5 ? b1 : 0.0;
    P.e2 = s >= 9 ? b15 : 0.0;
    P.e3 = s >= 13 ? b15 * b9 : 0.0;
    // upper: maps compose in decreasing lane order (seed enters lane 15)
    const bool h1 = s <= 14, h2 = s <= 13, h3 = s <= 12;
    const double c1 = shdn(B0, 1), c2 = shdn(B0, 2), c3 = shdn(B0, 3);
    const double n1 = h1 ? c1 : 1.0, n2 = h2 ? c2 : 1.0, n3 = h3 ? c3 : 1.0;
    const double B01 = B0 * c1, B012 = B01 * c2;
    P.q1 = h1 ? B0 : 0.0;
    P.q2 = h2 ? B01 : 0.0;
    P.q3 = h3 ? B012 : 0.0;
    const double B1 = ((B0 * n1) * n2) * n3;
    const double d1 = shdn(B1, 1), d5 = shdn(B1, 5), d9 = shdn(B1, 9), d13 = shdn(B1, 13);
    const bool k1 = s <= 14, k5 = s <= 10, k9 = s <= 6, k13 = s <= 2;
    const double o1 = k1 ? d1 : 1.0, o5 = k5 ? d5 : 1.0, o9 = k9 ? d9 : 1.0, o13 = k13 ? d13 : 1.0;
    P.f0 = k1 ? 1.0 : 0.0;
    P.f1 = k5 ? d1 : 0.0;
    const double d15 = d1 * d5;
    P.f2 = k9 ? d15 : 0.0;
    P.f3 = k13 ? d15 * d9 : 0.0;
    P.bex = ((o1 * o5) * o9) * o13;
    return P;
}

// Solve one line.  cr[k] = rhs[k]*mr[k] (the chain constants of the lower
// phase); twist row xt = bt*mrt + nlt*xa + nut*xd.
//
// The per-lane chain pieces are composed as prefix maps: slot k's value is
// PA_k * carry + PC_k with PC_k the composed constant after slot k (the
// compose's own intermediates) and PA_k the prefix product of the slot
// coefficients (factor-only, off the critical path), so once the scan has
// delivered the lane's carry every slot takes one FMA instead of a K-long
// re-walk; the compose starts from the first constant (fma(a, 0, c) == c).
// Same operator as the sequential form, rounded differently (<= 1e-15
// relative, far inside the 1e-10 apply bar).
template <int K>
__device__ __forceinline__ void line_solve4(const LinePrep &P, int n, int t, const double (&aL)[K],
                                            const double (&cr)[K], const double (&aU)[K], double btm, double nlt,
                                            double nut, double (&x)[K], double &xt)
{
    // ---- lower chain
    double pc[K], pa[K];
    pc[0] = cr[0];
    pa[0] = aL[0];
#pragma unroll
    for (int k = 1; k < K; k++) {
        pc[k] = fma(aL[k], pc[k - 1], cr[k]);
        pa[k] = aL[k] * pa[k - 1];
    }
    const double C0 = pc[K - 1];
    const double t1 = shup(C0, 1), t2 = shup(C0, 2), t3 = shup(C0, 3);
    const double C1 = fma(P.p1, t1, C0) + fma(P.p2, t2, P.p3 * t3);
    const double u1 = shup(C1, 1), u5 = shup(C1, 5), u9 = shup(C1, 9), u13 = shup(C1, 13);
    const double xl = fma(P.e0, u1, P.e1 * u5) + fma(P.e2, u9, P.e3 * u13);
#pragma unroll
    for (int k = 0; k < K; k++) x[k] = fma(pa[k], xl, pc[k]);
    // ---- twist row
    const double xa = __shfl_sync(FULL_MASK, x[K - 1], 15);
    const double xd = __shfl_sync(FULL_MASK, x[K - 1], 31);
    double acc = btm;
    if (t > 0) acc = fma(nlt, xa, acc);
    if (t < n - 1) acc = fma(nut, xd, acc);
    xt = acc;
    // ---- upper chain (independent of xt until the carry)
    double qc[K], qa[K];
    qc[K - 1] = x[K - 1];
    qa[K - 1] = aU[K - 1];
#pragma unroll
    for (int k = K - 2; k >= 0; k--) {
        qc[k] = fma(aU[k], qc[k + 1], x[k]);
        qa[k] = aU[k] * qa[k + 1];
    }
    const double D0 = qc[0];
    const double v1 = shdn(D0, 1), v2 = shdn(D0, 2), v3 = shdn(D0, 3);
    const double D1 = fma(P.q1, v1, D0) + fma(P.q2, v2, P.q3 * v3);
    const double w1 = shdn(D1, 1), w5 = shdn(D1, 5), w9 = shdn(D1, 9), w13 = shdn(D1, 13);
    const double dex = fma(P.f0, w1, P.f1 * w5) + fma(P.f2, w9, P.f3 * w13);
    const double xu = fma(P.bex, xt, dex);
#pragma unroll
    for (int k = 0; k < K; k++) x[k] = fma(qa[k], xu, qc[k]);
}
