#pragma once
// ntd.cu -- NTD preconditioner setup (factor_level3) and apply (ntd_apply)
// on sm_100a.
//
// Reference: /root/reference/pkg/src/ntdprecon/ntd_factor.py (setup) and
// ntd_solve.py (apply).  Mapping (one CTA of 4 warps per system):
//   level 3 (planes): the two twisted halves (ntd_solve.py:198-221 / :233-253,
//     ntd_factor.py:436-446) are two warp pairs; the twist plane is handled by
//     pair 0 between two __syncthreads.
//   level 2 (lines of a plane, _plane_solve ntd_solve.py:140-185 and
//     _factor_plane ntd_factor.py:147-219): the two halves are the two warps
//     of a pair; they meet at the twist line through a named barrier and a
//     shared-memory exchange of the neighbouring lines.
//   level 1 (cells of a line): one warp, shuffle scans (ntd_line.cuh).
// All level-2/3 couplings are diagonal (elementwise per cell), so a line's
// right-hand side only needs lines that the same lane layout already holds.
#include "common.cuh"
#include "ntd_line.cuh"

enum { M_LOWER3 = 0, M_UPPER3 = 1, M_SETUP = 2 };

struct FactorPtrs {
    const double *l1, *u1, *l2, *u2, *l3, *u3, *mr;
};

__device__ __forceinline__ FactorPtrs factor_ptrs(const double *pre, i64 n)
{
    FactorPtrs f;
    f.l1 = pre;
    f.u1 = pre + n;
    f.l2 = pre + 2 * n;
    f.u2 = pre + 3 * n;
    f.l3 = pre + 4 * n;
    f.u3 = pre + 5 * n;
    f.mr = pre + 6 * n;
    return f;
}

// What a plane solve reads as right-hand side and where it writes.
struct PlaneIO {
    // M_LOWER3: rhs = b - [hasM] l3*x[r-nxy] - [hasP] u3*x[r+nxy]; lower and
    //           final values -> x.
    // M_UPPER3: rhs = nbrUp ? u3*x[r+nxy] : l3*x[r-nxy]; lower -> xs;
    //           final: x[r] -= value.
    // M_SETUP:  rhs = useg[local]; lower -> ylow[local]; final -> out[local].
    const double *b;
    double *x, *xs;
    bool hasM, hasP, nbrUp;
    const double *useg;
    double *ylow, *out;
};

template <int K, int MODE>
__device__ __forceinline__ void rhs_lower(const FactorPtrs &F, const PlaneIO &io, const LineGeom<K> &g, i64 lb,
                                          i64 llocal, i64 nxy, double (&rhs)[K], double &rhst)
{
#pragma unroll
    for (int k = 0; k <= K; k++) {
        bool tw = (k == K);
        if (!tw && !g.valid(k)) {
            rhs[k] = 0.0;
            continue;
        }
        int c = tw ? g.t : g.cell(k);
        i64 r = lb + c;
        double v;
        if (MODE == M_LOWER3) {
            v = io.b[r];
            if (io.hasM) v -= F.l3[r] * io.x[r - nxy];
            if (io.hasP) v -= F.u3[r] * io.x[r + nxy];
        } else if (MODE == M_UPPER3) {
            v = io.nbrUp ? F.u3[r] * io.x[r + nxy] : F.l3[r] * io.x[r - nxy];
        } else {
            v = io.useg[llocal + c];
        }
        if (tw)
            rhst = v;
        else
            rhs[k] = v;
    }
}

template <int K, int MODE>
__device__ __forceinline__ void load_lowerstore(const PlaneIO &io, const LineGeom<K> &g, i64 lb, i64 llocal,
                                                double (&y)[K], double &yt)
{
    if (MODE == M_LOWER3)
        load_slots(g, io.x, lb, y, yt);
    else if (MODE == M_UPPER3)
        load_slots(g, io.xs, lb, y, yt);
    else
        load_slots(g, io.ylow, llocal, y, yt);
}

template <int K, int MODE>
__device__ __forceinline__ void store_lower(const PlaneIO &io, const LineGeom<K> &g, i64 lb, i64 llocal,
                                            const double (&y)[K], double yt)
{
    if (MODE == M_LOWER3)
        store_slots(g, io.x, lb, y, yt);
    else if (MODE == M_UPPER3)
        store_slots(g, io.xs, lb, y, yt);
    else
        store_slots(g, io.ylow, llocal, y, yt);
}

template <int K, int MODE>
__device__ __forceinline__ void finalize(const PlaneIO &io, const LineGeom<K> &g, i64 lb, i64 llocal,
                                         const double (&v)[K], double vt)
{
    if (MODE == M_LOWER3) {
        store_slots(g, io.x, lb, v, vt);
    } else if (MODE == M_UPPER3) {
        double xo[K], xot;
        load_slots(g, io.x, lb, xo, xot);
        double nv[K];
#pragma unroll
        for (int k = 0; k < K; k++) nv[k] = xo[k] - v[k];
        store_slots(g, io.x, lb, nv, xot - vt);
    } else {
        store_slots(g, io.out, llocal, v, vt);
    }
}

// Operands of one lower-phase line: factors, right-hand-side parts and the
// level-2 coupling.  Loaded one line ahead (register double buffer).
template <int K>
struct LOps {
    double mr[K], oL[K], oU[K], r0[K], c1[K], y1[K], cp[K];
    double mrt, l1t, u1t, r0t, c1t, y1t, cpt;
};
// Operands of one upper-phase line.
template <int K>
struct UOps {
    double mr[K], oL[K], oU[K], cp[K], y[K], xo[K];
    double mrt, l1t, u1t, cpt, yt, xot;
};

// Level-3 right-hand-side parts of a line: rhs = r0 - c1*y1 (M_LOWER3),
// c1*y1 (M_UPPER3) or r0 (M_SETUP).  For the twist plane (both neighbours)
// r0 already has the l3 term removed (loaded eagerly; one plane per apply).
template <int K, int MODE>
__device__ __forceinline__ void load_rhs_parts(const FactorPtrs &F, const PlaneIO &io, const LineGeom<K> &g, i64 lb,
                                               i64 ll, i64 nxy, LOps<K> &o)
{
#pragma unroll
    for (int k = 0; k <= K; k++) {
        const bool tw = k == K;
        double r0 = 0.0, c1 = 0.0, y1 = 0.0;
        if (tw || g.valid(k)) {
            const int c = tw ? g.t : g.cell(k);
            const i64 r = lb + c;
            if (MODE == M_LOWER3) {
                r0 = io.b[r];
                if (io.hasM && io.hasP) {
                    r0 -= F.l3[r] * io.x[r - nxy];
                    c1 = F.u3[r];
                    y1 = io.x[r + nxy];
                } else if (io.hasM) {
                    c1 = F.l3[r];
                    y1 = io.x[r - nxy];
                } else if (io.hasP) {
                    c1 = F.u3[r];
                    y1 = io.x[r + nxy];
                }
            } else if (MODE == M_UPPER3) {
                c1 = io.nbrUp ? F.u3[r] : F.l3[r];
                y1 = io.nbrUp ? io.x[r + nxy] : io.x[r - nxy];
            } else {
                r0 = io.useg[ll + c];
            }
        }
        if (tw) {
            o.r0t = r0;
            o.c1t = c1;
            o.y1t = y1;
        } else {
            o.r0[k] = r0;
            o.c1[k] = c1;
            o.y1[k] = y1;
        }
    }
}

template <int K, int MODE>
__device__ __forceinline__ void rhs_of(const LOps<K> &o, double (&rhs)[K], double &rhst)
{
#pragma unroll
    for (int k = 0; k < K; k++)
        rhs[k] = MODE == M_LOWER3 ? o.r0[k] - o.c1[k] * o.y1[k] : (MODE == M_UPPER3 ? o.c1[k] * o.y1[k] : o.r0[k]);
    rhst = MODE == M_LOWER3 ? o.r0t - o.c1t * o.y1t : (MODE == M_UPPER3 ? o.c1t * o.y1t : o.r0t);
}

template <int K, int MODE>
__device__ __forceinline__ void load_lops(const FactorPtrs &F, const PlaneIO &io, const LineGeom<K> &g, i64 pb,
                                          int q, int nx, i64 nxy, const double *cpl, bool has_cpl, LOps<K> &o)
{
    const i64 lb = pb + (i64)q * nx, ll = (i64)q * nx;
    load_line_factors(g, F.mr, F.l1, F.u1, lb, o.mr, o.oL, o.oU, o.mrt, o.l1t, o.u1t);
    load_rhs_parts<K, MODE>(F, io, g, lb, ll, nxy, o);
    if (has_cpl) {
        load_slots(g, cpl, lb, o.cp, o.cpt);
    } else {
#pragma unroll
        for (int k = 0; k < K; k++) o.cp[k] = 0.0;
        o.cpt = 0.0;
    }
}

template <int K, int MODE>
__device__ __forceinline__ void load_uops(const FactorPtrs &F, const PlaneIO &io, const LineGeom<K> &g, i64 pb,
                                          int q, int nx, const double *cpl, UOps<K> &o)
{
    const i64 lb = pb + (i64)q * nx, ll = (i64)q * nx;
    load_line_factors(g, F.mr, F.l1, F.u1, lb, o.mr, o.oL, o.oU, o.mrt, o.l1t, o.u1t);
    load_slots(g, cpl, lb, o.cp, o.cpt);
    load_lowerstore<K, MODE>(io, g, lb, ll, o.y, o.yt);
    if (MODE == M_UPPER3) load_slots(g, io.x, lb, o.xo, o.xot);
}

// Warp-cooperative L2 prefetch of rows [r0, r1) of an array.
__device__ __forceinline__ void prefetch_rows(const double *p, i64 r0, i64 r1)
{
    if (!p || r1 <= r0) return;
    const char *c = (const char *)(p + r0);
    const i64 bytes = (r1 - r0) * 8;
    for (i64 off = (i64)(threadIdx.x & 31) * 128; off < bytes; off += 32 * 128) prefetch_l2(c + off);
}

// Prefetch into L2 the part of plane `npb` this warp will touch.
__device__ __forceinline__ void prefetch_plane(const FactorPtrs &F, const double *e1, const double *e2, i64 npb,
                                               int nx, int ny, int w2)
{
    const int t2 = (ny - 1) / 2;
    const i64 r0 = npb + (w2 == 0 ? 0 : (i64)t2 * nx);
    const i64 r1 = npb + (w2 == 0 ? (i64)(t2 + 1) * nx : (i64)ny * nx);
    prefetch_rows(F.mr, r0, r1);
    prefetch_rows(F.l1, r0, r1);
    prefetch_rows(F.u1, r0, r1);
    prefetch_rows(F.l2, r0, r1);
    prefetch_rows(F.u2, r0, r1);
    prefetch_rows(e1, r0, r1);
    prefetch_rows(e2, r0, r1);
}

// Twisted solve of one factored plane (ntd_solve.py:140-185) by a warp pair.
// w2: warp within the pair (0 = ascending lines, 1 = descending lines).
// ex: this pair's shared exchange buffer [2 parity][2 warps][32K+1].
// next_pb >= 0: L2-prefetch that plane (arrays F.* and pf1/pf2) meanwhile.
template <int K, int MODE>
__device__ void plane_solve(const FactorPtrs &F, const PlaneIO &io, i64 pb, int nx, int ny, int w2, int bar_id,
                            double *ex, int &parity, i64 next_pb = -1, const double *pf1 = nullptr,
                            const double *pf2 = nullptr)
{
    const int lane = threadIdx.x & 31;
    const LineGeom<K> g(nx, lane);
    const i64 nxy = (i64)nx * ny;
    const int t2 = (ny - 1) / 2;
    if (next_pb >= 0) prefetch_plane(F, pf1, pf2, next_pb, nx, ny, w2);
    double xprev[K], xprevt = 0.0;
#pragma unroll
    for (int k = 0; k < K; k++) xprev[k] = 0.0;
    // ---------------- level-2 lower sweep, ends inward (ntd_solve.py:147-171)
    const int cnt = w2 == 0 ? t2 : (ny - 1 - t2);
    const double *cplL = w2 == 0 ? F.l2 : F.u2;  // b -= l2*x[r-nx] | u2*x[r+nx]
    auto qlow = [&](int i) { return w2 == 0 ? i : ny - 1 - i; };
    auto lower_body = [&](const LOps<K> &o, int i) {
        const int q = qlow(i);
        const i64 lb = pb + (i64)q * nx, ll = (i64)q * nx;
        double rhs[K], rhst;
        rhs_of<K, MODE>(o, rhs, rhst);
#pragma unroll
        for (int k = 0; k < K; k++) rhs[k] -= o.cp[k] * xprev[k];
        rhst -= o.cpt * xprevt;
        double x[K], xt;
        line_solve(g, o.mr, o.oL, o.oU, rhs, rhst, o.mrt, o.l1t, o.u1t, x, xt);
        store_lower<K, MODE>(io, g, lb, ll, x, xt);
#pragma unroll
        for (int k = 0; k < K; k++) xprev[k] = x[k];
        xprevt = xt;
    };
    {
        for (int i = 0; i < cnt; i++) {
            LOps<K> oa;
            load_lops<K, MODE>(F, io, g, pb, qlow(i), nx, nxy, cplL, i > 0, oa);
            lower_body(oa, i);
        }
    }
    // ---------------- exchange the lines next to the twist
    const int stride = 32 * K + 1;
    double *mine = ex + (parity * 2 + w2) * stride;
    double *other = ex + (parity * 2 + (1 - w2)) * stride;
#pragma unroll
    for (int k = 0; k < K; k++) mine[lane * K + k] = xprev[k];
    if (lane == 0) mine[32 * K] = xprevt;
    named_bar(bar_id, 64);
    parity ^= 1;
    double xo[K], xot = other[32 * K];
#pragma unroll
    for (int k = 0; k < K; k++) xo[k] = other[lane * K + k];
    // x_{t2-1} lives in warp 0, x_{t2+1} in warp 1
    double xa[K], xat, xd[K], xdt;
#pragma unroll
    for (int k = 0; k < K; k++) {
        xa[k] = w2 == 0 ? xprev[k] : xo[k];
        xd[k] = w2 == 0 ? xo[k] : xprev[k];
    }
    xat = w2 == 0 ? xprevt : xot;
    xdt = w2 == 0 ? xot : xprevt;
    // ---------------- twist line (ntd_solve.py:172-177), both warps; its
    // operands are read after the barrier (x of the twist line of the
    // neighbouring plane was written by the other warp).
    const double *cplU = w2 == 0 ? F.u2 : F.l2;  // bs = u2*x[r+nx] | l2*x[r-nx]
    double xT[K], xTt;
    UOps<K> ua, ub;
    {
        const int q = t2;
        const i64 lb = pb + (i64)q * nx, ll = (i64)q * nx;
        LOps<K> o;
        load_lops<K, MODE>(F, io, g, pb, q, nx, nxy, F.l2, t2 > 0, o);
        double cu[K], cut;
        if (t2 < ny - 1) load_slots(g, F.u2, lb, cu, cut);
        if (cnt > 0) load_uops<K, MODE>(F, io, g, pb, w2 == 0 ? t2 - 1 : t2 + 1, nx, cplU, ua);
        double rhs[K], rhst;
        rhs_of<K, MODE>(o, rhs, rhst);
#pragma unroll
        for (int k = 0; k < K; k++) rhs[k] -= o.cp[k] * xa[k];
        rhst -= o.cpt * xat;
        if (t2 < ny - 1) {
#pragma unroll
            for (int k = 0; k < K; k++) rhs[k] -= cu[k] * xd[k];
            rhst -= cut * xdt;
        }
        line_solve(g, o.mr, o.oL, o.oU, rhs, rhst, o.mrt, o.l1t, o.u1t, xT, xTt);
        if (w2 == 0) finalize<K, MODE>(io, g, lb, ll, xT, xTt);
    }
    // ---------------- level-2 upper sweep, twist outward (ntd_solve.py:178-185)
    double xn[K], xnt = xTt;
#pragma unroll
    for (int k = 0; k < K; k++) xn[k] = xT[k];
    auto qup = [&](int i) { return w2 == 0 ? t2 - 1 - i : t2 + 1 + i; };
    auto upper_body = [&](const UOps<K> &o, int i) {
        const int q = qup(i);
        const i64 lb = pb + (i64)q * nx, ll = (i64)q * nx;
        double bs[K], bst = o.cpt * xnt;
#pragma unroll
        for (int k = 0; k < K; k++) bs[k] = o.cp[k] * xn[k];
        double xs[K], xst;
        line_solve(g, o.mr, o.oL, o.oU, bs, bst, o.mrt, o.l1t, o.u1t, xs, xst);
#pragma unroll
        for (int k = 0; k < K; k++) xn[k] = o.y[k] - xs[k];
        xnt = o.yt - xst;
        if (MODE == M_UPPER3) {
            double nv[K];
#pragma unroll
            for (int k = 0; k < K; k++) nv[k] = o.xo[k] - xn[k];
            store_slots(g, io.x, lb, nv, o.xot - xnt);
        } else {
            finalize<K, MODE>(io, g, lb, ll, xn, xnt);
        }
    };
    for (int i = 0; i < cnt; i++) {
        if (i > 0) load_uops<K, MODE>(F, io, g, pb, qup(i), nx, cplU, ua);
        upper_body(ua, i);
    }
}

// ---- TMA / mbarrier helpers (1-D bulk copies)
__device__ __forceinline__ unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(void *bar, unsigned count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(void *bar, unsigned bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(void *bar, unsigned parity)
{
    unsigned ok = 0;
    const unsigned a = smem_u32(bar);
    while (!ok) {
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
            : "=r"(ok)
            : "r"(a), "r"(parity)
            : "memory");
    }
}
// Producer-side wait: poll with back-off so a waiting producer warp does not
// steal issue slots from the solver warp sharing its SM sub-partition.
__device__ __forceinline__ void mbar_wait_lazy(void *bar, unsigned parity)
{
    unsigned ok = 0;
    const unsigned a = smem_u32(bar);
    while (true) {
        asm volatile(
            "{ .reg .pred p; mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
            : "=r"(ok)
            : "r"(a), "r"(parity)
            : "memory");
        if (ok) break;
        __nanosleep(96);
    }
}
__device__ __forceinline__ void tma_load_1d(void *dst, const void *src, unsigned bytes, void *bar)
{
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

// =============================================================== apply
template <int K>
__global__ void __launch_bounds__(128) k_ntd_apply(const double *__restrict__ pre, const double *__restrict__ b,
                                                   double *x, double *work, int nx, int ny, int nz,
                                                   const int32_t *__restrict__ active)
{
    __shared__ double ex[2][2 * 2 * (32 * K + 1)];
    const i64 sys = blockIdx.x;
    if (active && !active[sys]) return;
    const i64 nxy = (i64)nx * ny, n = nxy * nz;
    const FactorPtrs F = factor_ptrs(pre + sys * 7 * n, n);
    const int warp = __shfl_sync(FULL_MASK, (int)(threadIdx.x >> 5), 0), pair = warp >> 1, w2 = warp & 1, bar = 1 + pair;
    double *myex = ex[pair];
    int parity = 0;
    PlaneIO io;
    io.b = b + sys * n;
    io.x = x + sys * n;
    io.xs = work + sys * n;
    io.useg = nullptr;
    io.ylow = io.out = nullptr;
    const int t3 = (nz - 1) / 2;
    // level-3 lower sweep, both halves (ntd_solve.py:198-221)
    io.nbrUp = false;
    if (pair == 0) {
        prefetch_plane(F, io.b, F.l3, 0, nx, ny, w2);
        for (int p = 0; p < t3; p++) {
            io.hasM = p > 0;
            io.hasP = false;
            plane_solve<K, M_LOWER3>(F, io, (i64)p * nxy, nx, ny, w2, bar, myex, parity, (i64)(p + 1) * nxy,
                                     io.b, F.l3);
        }
    } else {
        prefetch_plane(F, io.b, F.u3, (i64)(nz - 1) * nxy, nx, ny, w2);
        for (int p = nz - 1; p > t3; p--) {
            io.hasM = false;
            io.hasP = p < nz - 1;
            plane_solve<K, M_LOWER3>(F, io, (i64)p * nxy, nx, ny, w2, bar, myex, parity,
                                     p - 1 > t3 ? (i64)(p - 1) * nxy : -1, io.b, F.u3);
        }
    }
    __syncthreads();
    // twist plane (ntd_solve.py:222-232)
    if (pair == 0) {
        io.hasM = t3 > 0;
        io.hasP = t3 < nz - 1;
        plane_solve<K, M_LOWER3>(F, io, (i64)t3 * nxy, nx, ny, w2, bar, myex, parity);
    }
    __syncthreads();
    // level-3 upper sweep (ntd_solve.py:233-253)
    if (pair == 0) {
        io.nbrUp = true;
        if (t3 > 0) prefetch_plane(F, F.u3, io.x, (i64)(t3 - 1) * nxy, nx, ny, w2);
        for (int p = t3 - 1; p >= 0; p--)
            plane_solve<K, M_UPPER3>(F, io, (i64)p * nxy, nx, ny, w2, bar, myex, parity,
                                     p > 0 ? (i64)(p - 1) * nxy : -1, F.u3, io.x);
    } else {
        io.nbrUp = false;
        if (t3 + 1 < nz) prefetch_plane(F, F.l3, io.x, (i64)(t3 + 1) * nxy, nx, ny, w2);
        for (int p = t3 + 1; p < nz; p++)
            plane_solve<K, M_UPPER3>(F, io, (i64)p * nxy, nx, ny, w2, bar, myex, parity,
                                     p + 1 < nz ? (i64)(p + 1) * nxy : -1, F.l3, io.x);
    }
}

// =============================================================== factor
// Setup-side line and plane solves in the reference's exact operation order.
//
// The factorisation feeds nested solves back into the bands (correct_line:
// T_m^-1 u; correct_from: the nested plane solve of the neighbour), and on
// strongly heterogeneous fields (BASELINE config 5, kappa jumps of 1e6)
// rounding differences there are amplified to ~1e-10 in the bands.  So the
// setup does not use the warp-scan line solve of the apply: it restates
// _chain_scaled / _chain_unit (ntd_solve.py:20-104) with the reference's
// lane composition (CHAIN_LANES = 4, ntd_solve.py:17: `lanes` chunks of
// m // lanes composed into prefix maps, stitched sequentially, remainder
// walked sequentially), every operation exactly rounded in the reference's
// order.  The resulting factor is bitwise equal to the reference's.
constexpr int REF_LANES = 4;
static_assert(REF_LANES == 4, "chain_ref_finish picks among four chunk carries");
#ifdef FACTOR_TIMING
#include <cstdio>
__device__ unsigned long long g_ft[16];
#define FT0 const long long ft0_ = clock64();
#define FTA(i) if (threadIdx.x == 0) g_ft[i] += (unsigned long long)(clock64() - ft0_);
#define FTM(i) if (threadIdx.x == 0) { const long long now_ = clock64(); g_ft[i] += (unsigned long long)(now_ - ftm_); ftm_ = now_; }
#define FTM0 long long ftm_ = clock64();
#else
#define FT0
#define FTA(i)
#define FTM(i)
#define FTM0
#endif

// One chain of a line (both chains of a line run concurrently, one per
// half-warp h).  Chain position e = 0..m-1 is cell lo + e*step.
//   SCALED: x_e = (rhs_e - off_e x_{e-1}) dr_e, x_{-1} = x0 (_chain_scaled)
//   UNIT:   x_e = x_e - dr_e off_e x_{e-1}     (_chain_unit, in place)
// aw/cw: smem prefix maps (m each); car: smem carries (REF_LANES + 1).
template <bool SCALED>
__device__ __forceinline__ void chain_ref_compose(const double *__restrict__ x, const double *__restrict__ dr,
                                                  const double *__restrict__ off, const double *__restrict__ rhs,
                                                  int lo, int step, int m, double *__restrict__ aw,
                                                  double *__restrict__ cw, int sl)
{
    // sl: lane within the half-warp; lanes 0..REF_LANES-1 compose one chunk each
    if (m < 2 * REF_LANES || sl >= REF_LANES) return;
    const int chunk = m / REF_LANES, base = sl * chunk;
    // Cells are walked four at a time; the operands of the next four are requested before the
    // current four's dependent multiply-adds (the compiler does not move the loads above the
    // prefix-map stores by itself once this is inlined).  Running pointers: po/pd/pr at the batch's
    // first cell, pa/pc at its prefix-map slots; a batch past the chunk's end re-reads the last cell.
    const double *po = off + (lo + base * step), *pd = dr + (lo + base * step);
    const double *pr = (SCALED ? rhs : x) + (lo + base * step);
    double *pa = aw + base, *pc = cw + base;
    double aa, cc;
    {
        const double a = SCALED ? mul_rn(-po[0], pd[0]) : mul_rn(-pd[0], po[0]);
        aa = a;
        cc = SCALED ? mul_rn(pr[0], pd[0]) : pr[0];
        pa[0] = aa;
        pc[0] = cc;
    }
    double o[4], d[4], r[4];
    auto fetch = [&](int left, const double *qo, const double *qd, const double *qr, double (&oo)[4], double (&dd)[4],
                     double (&rr)[4]) {  // left: cells of the chunk from qo on (>= 1)
#pragma unroll
        for (int j = 0; j < 4; j++) {
            const int e = (j < left ? j : left - 1) * step;
            oo[j] = qo[e];
            dd[j] = qd[e];
            rr[j] = qr[e];
        }
    };
    int left = chunk - 1;  // cells not yet composed
    po += step;
    pd += step;
    pr += step;
    pa += 1;
    pc += 1;
    if (left > 0) fetch(left, po, pd, pr, o, d, r);
#pragma unroll 1
    for (; left > 0; left -= 4) {
        double on[4], dn[4], rn[4];
        const int nleft = left > 4 ? left - 4 : 1;
        const int adv4 = left > 4 ? 4 * step : 0;
        fetch(nleft, po + adv4, pd + adv4, pr + adv4, on, dn, rn);
#pragma unroll
        for (int j = 0; j < 4; j++) {
            if (j < left) {
                const double a = SCALED ? mul_rn(-o[j], d[j]) : mul_rn(-d[j], o[j]);
                aa = mul_rn(a, aa);
                cc = add_rn(mul_rn(a, cc), SCALED ? mul_rn(r[j], d[j]) : r[j]);
                pa[j] = aa;
                pc[j] = cc;
            }
        }
#pragma unroll
        for (int j = 0; j < 4; j++) {
            o[j] = on[j];
            d[j] = dn[j];
            r[j] = rn[j];
        }
        po += 4 * step;
        pd += 4 * step;
        pr += 4 * step;
        pa += 4;
        pc += 4;
    }
}

template <bool SCALED>
__device__ __forceinline__ void chain_ref_finish(double *x, const double *dr, const double *off, const double *rhs,
                                                 int lo, int step, int m, double x0, const double *aw,
                                                 const double *cw, double *car, int sl)
{
    // Both half-warps run this concurrently (their chains may take different
    // branches), so every path passes exactly two __syncwarp().
    if (m < 2 * REF_LANES) {  // scalar chain (also m <= 0: nothing)
        if (sl == 0) {
            double xp = x0;
            int p = lo;
            for (int it = 0; it < m; it++, p += step) {
                xp = SCALED ? mul_rn(sub_rn(rhs[p], mul_rn(off[p], xp)), dr[p])
                            : sub_rn(x[p], mul_rn(mul_rn(dr[p], off[p]), xp));
                x[p] = xp;
            }
        }
        __syncwarp();
        __syncwarp();
        return;
    }
    const int chunk = m / REF_LANES;
    if (sl == 0) {  // carries into each chunk, stitched in order
        double carry = x0;
        for (int l = 0; l < REF_LANES; l++) {
            car[l] = carry;
            const int e = l * chunk + chunk - 1;
            carry = add_rn(mul_rn(aw[e], carry), cw[e]);
        }
        car[REF_LANES] = carry;
    }
    __syncwarp();
    {
        // cells e = sl, sl + 16, ... of the composed part, four at a time, loads first; the carry of a
        // cell's chunk is picked by comparisons (no division per cell)
        const double c0 = car[0], c1 = car[1], c2 = car[2], c3 = car[3];
        const int total = REF_LANES * chunk;
        const double *pa = aw + sl, *pc = cw + sl;
        double *px = x + (lo + sl * step);
#pragma unroll 1
        for (int e = sl; e < total; e += 64, pa += 64, pc += 64, px += 64 * step) {
            double av[4], cv[4];
#pragma unroll
            for (int j = 0; j < 4; j++) {
                const int o16 = e + 16 * j < total ? 16 * j : 0;
                av[j] = pa[o16];
                cv[j] = pc[o16];
            }
#pragma unroll
            for (int j = 0; j < 4; j++) {
                const int ej = e + 16 * j;
                if (ej < total) {
                    const double cl = ej < chunk ? c0 : ej < 2 * chunk ? c1 : ej < 3 * chunk ? c2 : c3;
                    px[16 * j * step] = add_rn(mul_rn(av[j], cl), cv[j]);
                }
            }
        }
    }
    if (sl == 0) {  // remainder, sequential from the last carry
        double xp = car[REF_LANES];
        int p = lo + REF_LANES * chunk * step;
        for (int it = REF_LANES * chunk; it < m; it++, p += step) {
            xp = SCALED ? mul_rn(sub_rn(rhs[p], mul_rn(off[p], xp)), dr[p])
                        : sub_rn(x[p], mul_rn(mul_rn(dr[p], off[p]), xp));
            x[p] = xp;
        }
    }
    __syncwarp();
}

// _line_solve (ntd_solve.py:134-137) of one line of n <= 32K cells by one warp:
// x = T^-1 b with T's factor (mr, l1, u1; line-local global arrays).
//
// Everything a line touches is requested up front -- the factor, and whatever
// the caller's right-hand side is made of (ldf: loads of a cell into a RawLine;
// evf: RawLine -> rhs value) -- so a line costs ONE memory round trip;
// the chains then walk shared memory, and wf(cell, x, RawLine) stores the
// result.  (Before, the operands were read from global memory inside the
// composition's sequential chunk walks and the callers' elementwise steps
// around the solve were plain loops over the line whose loads could not pass
// the previous iteration's store: ~11 serialised round trips per loop at
// nx = 350.)  Same operations in the same order: bitwise the same result.
// On return s_x(lsm, n) holds x and, with KEEP, s_b(lsm, n) the rhs; s_l /
// s_u / s_mr still hold the line's factor.
// lsm: 7n doubles of smem (prefix maps 2n, then mr, l1, u1, x, b); car: 2 x
// (REF_LANES + 1) doubles of smem.
struct RawLine {  // (references to one cell's slots of five register arrays; unused ones fold away)
    double &a, &b, &c, &d, &e;
};
__device__ __forceinline__ double *s_mr_of(double *lsm, int n) { return lsm + 2 * n; }
__device__ __forceinline__ double *s_l_of(double *lsm, int n) { return lsm + 3 * n; }
__device__ __forceinline__ double *s_u_of(double *lsm, int n) { return lsm + 4 * n; }
__device__ __forceinline__ double *s_x_of(double *lsm, int n) { return lsm + 5 * n; }
__device__ __forceinline__ double *s_b_of(double *lsm, int n) { return lsm + 6 * n; }
constexpr int LSM_PER_WARP = 7;  // x nx doubles

template <int K, bool KEEP, class LF, class EF, class WF>
static __device__ __forceinline__ void line_solve_ref(LF &&ldf, EF &&evf, WF &&wf, const double *mr, const double *l1,
                                                      const double *u1, int n, double *lsm, double *car)
{
    const int lane = threadIdx.x & 31, h = lane >> 4, sl = lane & 15;
    const int t = (n - 1) / 2;
    FT0
    double *s_mr = s_mr_of(lsm, n), *s_l = s_l_of(lsm, n), *s_u = s_u_of(lsm, n), *s_x = s_x_of(lsm, n);
    double ra[K], rb[K], rc[K], rd[K], re[K];
    FTM0
    {
        double v[3][K];
        // (unconditional loads at a clamped cell: guarded loads end up in per-cell branches next to
        // their stores, one memory round trip per cell instead of one per line)
#pragma unroll
        for (int k = 0; k < K; k++) {
            const int c = min(lane + 32 * k, n - 1);
            v[0][k] = mr[c];
            v[1][k] = l1[c];
            v[2][k] = u1[c];
            ldf(c, RawLine{ra[k], rb[k], rc[k], rd[k], re[k]});
        }
#pragma unroll
        for (int k = 0; k < K; k++) {
            const int c = lane + 32 * k;
            if (c < n) {
                s_mr[c] = v[0][k];
                s_l[c] = v[1][k];
                s_u[c] = v[2][k];
                const double r = evf(RawLine{ra[k], rb[k], rc[k], rd[k], re[k]});
                s_x[c] = r;
                if (KEEP) s_b_of(lsm, n)[c] = r;
            }
        }
    }
    __syncwarp();
    FTM(9)
    // half 0: ascending chain over cells 0..t-1; half 1: descending n-1..t+1
    const int m = h == 0 ? t : n - 1 - t;
    const int lo = h == 0 ? 0 : n - 1, step = h == 0 ? 1 : -1;
    double *aw = lsm + (h == 0 ? 0 : 2 * t), *cw = aw + m;
    double *ch = car + h * (REF_LANES + 1);
    // _line_lower (ntd_solve.py:107-121); the rhs is consumed in place (x_e overwrites rhs_e)
    chain_ref_compose<true>(nullptr, s_mr, h == 0 ? s_l : s_u, s_x, lo, step, m, aw, cw, sl);
    __syncwarp();
    FTM(10)
    chain_ref_finish<true>(s_x, s_mr, h == 0 ? s_l : s_u, s_x, lo, step, m, 0.0, aw, cw, ch, sl);
    FTM(11)
    if (lane == 0) {
        double acc = s_x[t];
        if (t > 0) acc = sub_rn(acc, mul_rn(s_l[t], s_x[t - 1]));
        if (t < n - 1) acc = sub_rn(acc, mul_rn(s_u[t], s_x[t + 1]));
        s_x[t] = mul_rn(acc, s_mr[t]);
    }
    __syncwarp();
    // _line_upper (ntd_solve.py:124-131): outward from the twist
    const double xt = s_x[t];
    const int lo2 = h == 0 ? t - 1 : t + 1, step2 = -step;
    FTM(12)
    chain_ref_compose<false>(s_x, s_mr, h == 0 ? s_u : s_l, nullptr, lo2, step2, m, aw, cw, sl);
    __syncwarp();
    FTM(13)
    chain_ref_finish<false>(s_x, s_mr, h == 0 ? s_u : s_l, nullptr, lo2, step2, m, xt, aw, cw, ch, sl);
    FTM(14)
#pragma unroll
    for (int k = 0; k < K; k++) {
        const int c = lane + 32 * k;
        if (c < n) wf(c, s_x[c], RawLine{ra[k], rb[k], rc[k], rd[k], re[k]});
    }
    __syncwarp();
    FTM(15)
    FTA(2)
}

// _plane_solve (ntd_solve.py:140-185) of factored plane (F at offset pb) in
// the reference's order, by a warp pair (w2 = 0: lines 0..t2, w2 = 1: lines
// t2+1..ny-1; the two level-2 halves only meet at the twist line).
// rhs: plane-local right-hand side (read only); X: solution.  The reference's
// scratch copies (b, xs, bs) live in registers / shared memory per line: each
// line's right-hand side is formed from rhs, the coupling and the neighbour
// line as the line is staged, and the upper sweep's x -= xs is the solve's
// write-back.
template <int K>
static __device__ void plane_solve_ref(const FactorPtrs &F, i64 pb, const double *rhs, double *X, int nx, int ny,
                                       int w2, int bar_id, double *lsm, double *car)
{
    const int t2 = (ny - 1) / 2;
    const double *mr = F.mr + pb, *l1 = F.l1 + pb, *u1 = F.u1 + pb, *l2 = F.l2 + pb, *u2 = F.u2 + pb;
    // lower-sweep line at offset s: rhs - cpl * X[nb] (first line of the sweep: rhs)
    auto lower = [&](i64 s, const double *cpl, i64 nb, bool first) {
        line_solve_ref<K, false>(
            [&](int c, const RawLine &r) {
                r.a = rhs[s + c];
                if (!first) {
                    r.b = cpl[s + c];
                    r.c = X[s + c + nb];
                }
            },
            [&](const RawLine &r) { return first ? r.a : sub_rn(r.a, mul_rn(r.b, r.c)); },
            [&](int c, double v, const RawLine &) { X[s + c] = v; }, mr + s, l1 + s, u1 + s, nx, lsm, car);
    };
    // upper-sweep line: xs = T^-1 (cpl * X[nb]); x -= xs
    auto upper = [&](i64 s, const double *cpl, i64 nb) {
        line_solve_ref<K, false>(
            [&](int c, const RawLine &r) {
                r.a = cpl[s + c];
                r.b = X[s + c + nb];
                r.c = X[s + c];
            },
            [&](const RawLine &r) { return mul_rn(r.a, r.b); },
            [&](int c, double v, const RawLine &r) { X[s + c] = sub_rn(r.c, v); }, mr + s, l1 + s, u1 + s, nx, lsm,
            car);
    };
    // level-2 lower sweep, ends inward (ntd_solve.py:147-171)
    if (w2 == 0) {
        for (int q = 0; q < t2; q++) lower((i64)q * nx, l2, -nx, q == 0);
    } else {
        for (int q = ny - 1; q > t2; q--) lower((i64)q * nx, u2, nx, q == ny - 1);
    }
    __threadfence_block();
    named_bar(bar_id, 64);
    // twist line (ntd_solve.py:172-177)
    if (w2 == 0) {
        const i64 s = (i64)t2 * nx;
        const bool hm = t2 > 0, hp = t2 < ny - 1;
        line_solve_ref<K, false>(
            [&](int c, const RawLine &r) {
                r.a = rhs[s + c];
                if (hm) {
                    r.b = l2[s + c];
                    r.c = X[s + c - nx];
                }
                if (hp) {
                    r.d = u2[s + c];
                    r.e = X[s + c + nx];
                }
            },
            [&](const RawLine &r) {
                double v = r.a;
                if (hm) v = sub_rn(v, mul_rn(r.b, r.c));
                if (hp) v = sub_rn(v, mul_rn(r.d, r.e));
                return v;
            },
            [&](int c, double v, const RawLine &) { X[s + c] = v; }, mr + s, l1 + s, u1 + s, nx, lsm, car);
    }
    __threadfence_block();
    named_bar(bar_id, 64);
    // level-2 upper sweep, twist outward (ntd_solve.py:178-185)
    if (w2 == 0) {
        for (int q = t2 - 1; q >= 0; q--) upper((i64)q * nx, u2, nx);
    } else {
        for (int q = t2 + 1; q < ny; q++) upper((i64)q * nx, l2, -nx);
    }
    __threadfence_block();
    named_bar(bar_id, 64);
}

// Per-pair global scratch (plane-local, nxy each).
enum { S_PC0 = 0, S_PC1 = 5, S_W = 10, S_BETA, S_QD, S_TDW, S_PER_PAIR };

struct PairScratch {
    double *base;
    i64 nxy;
    __device__ double *at(int k) const { return base + k * nxy; }
};

// status codes (ntdgpu.h)
struct ErrState {
    int code;
    i64 plane, row;
};

__device__ __forceinline__ void set_err(volatile int *ecode, i64 *eplane, i64 *erow, int code, i64 plane, i64 row)
{
    if (*ecode == 0) {
        *eplane = plane;
        *erow = row;
        __threadfence_block();
        *ecode = code;
    }
}

// _line_factor (ntd_factor.py:80-110) on one line: exact, sequential pivots.
// td/tl/tu are global (plane-local) arrays; mr output global.  smem per warp:
// sd[nx] diag, sc[nx] products, sm[nx] reciprocals.  Returns -1 or bad cell.
static __device__ int line_factor_warp(const double *__restrict__ td, const double *__restrict__ tl,
                                const double *__restrict__ tu, double *__restrict__ mr, int nx, double *sd,
                                double *sc, double *sm)
{
    const int lane = threadIdx.x & 31;
    const int t = (nx - 1) / 2;
    FT0
    for (int c = lane; c < nx; c += 32) {
        sd[c] = td[c];
        double p = 0.0;
        if (c < t && c > 0) p = mul_rn(tl[c], tu[c - 1]);
        if (c > t && c < nx - 1) p = mul_rn(tu[c], tl[c + 1]);
        sc[c] = p;
    }
    __syncwarp();
    int bad = -1;
    if (lane == 0 || lane == 16) {
        // Lane 0 walks the ascending pivots, lane 16 the descending ones -- in ONE loop, so the two
        // recurrences run concurrently (as two branches of a warp they ran one after the other).
        // The first cell needs no special case (its product sc is an exact 0 and m starts at 0), and a
        // bad pivot is recorded without leaving the loop: what follows it is never used, the line fails.
        const bool asc = lane == 0;
        const int cnt = asc ? t : nx - 1 - t, stp = asc ? 1 : -1;
        int i = asc ? 0 : nx - 1;
        double m = 0.0;
        // (the next cell's operands are read before this cell's dependent multiply, subtract and
        // reciprocal, so their shared-memory latency is off the recurrence; the line has a twist cell
        // past each walk, so the look-ahead stays inside the line)
        double dn = sd[i], cn = sc[i];
        for (int it = 0; it < cnt; it++, i += stp) {
            const double d = dn, cc = cn;
            dn = sd[i + stp];
            cn = sc[i + stp];
            const double piv = sub_rn(d, mul_rn(cc, m));
            if (bad < 0 && (piv == 0.0 || !isfinite(piv))) bad = i;
            m = __drcp_rn(piv);  // == 1.0 / piv (both correctly rounded)
            sm[i] = m;
        }
    }
    int bad_a = __shfl_sync(FULL_MASK, bad, 0);
    int bad_d = __shfl_sync(FULL_MASK, bad, 16);
    __syncwarp();
    if (bad_a >= 0) return bad_a;
    if (bad_d >= 0) return bad_d;
    int badt = -1;
    if (lane == 0) {
        double piv = sd[t];
        if (t > 0) piv = sub_rn(piv, mul_rn(mul_rn(tl[t], tu[t - 1]), sm[t - 1]));
        if (t < nx - 1) piv = sub_rn(piv, mul_rn(mul_rn(tu[t], tl[t + 1]), sm[t + 1]));
        if (piv == 0.0 || !isfinite(piv))
            badt = t;
        else
            sm[t] = 1.0 / piv;
    }
    badt = __shfl_sync(FULL_MASK, badt, 0);
    __syncwarp();
    if (badt >= 0) return badt;
    for (int c = lane; c < nx; c += 32) mr[c] = sm[c];
    __syncwarp();
    FTA(7)
    return -1;
}

// _correct_line (ntd_factor.py:113-144): line q corrected through factored
// line m.  P* are the plane's corrected bands (plane-local), L1G/U1G/MRG the
// plane's factor outputs.  w = T_m^-1 u, beta and the neighbours' beta / u
// stay in shared memory (line_solve_ref leaves x, the rhs and line m's l1 / u1
// there).  Returns -1 or bad plane-local row.
template <int K>
__device__ i64 correct_line_warp(int q, int m, const double *P_l2, const double *P_u2, double *TDW, double *L1G,
                                 double *U1G, const double *MRG, int nx, double *lsm, double *car)
{
    const int lane = threadIdx.x & 31;
    const i64 sq = (i64)q * nx, sm = (i64)m * nx;
    FT0
    const double *src = m < q ? P_u2 : P_l2;
    line_solve_ref<K, true>(
        [&](int c, const RawLine &r) { r.a = src[sm + c]; },
        [&](const RawLine &r) { return r.a; }, [&](int, double, const RawLine &) {}, MRG + sm, L1G + sm, U1G + sm, nx,
        lsm, car);
    double *s_w = s_x_of(lsm, nx), *s_uu = s_b_of(lsm, nx);
    const double *s_l1m = s_l_of(lsm, nx), *s_u1m = s_u_of(lsm, nx);
    // what the update reads from global memory, requested before the divisions below
    const double *rsp = m < q ? P_l2 : P_u2;
    double rs[K], tdm[K], tdq[K], l1q[K], u1q[K];
#pragma unroll
    for (int k = 0; k < K; k++) {
        const int c = min(lane + 32 * k, nx - 1);
        rs[k] = rsp[sq + c];
        tdm[k] = TDW[sm + c];
        tdq[k] = TDW[sq + c];
        l1q[k] = L1G[sq + c];
        u1q[k] = U1G[sq + c];
    }
    // beta = w/u where u != 0 (first non-finite -> error)
    int badk = 0x7fffffff;
#pragma unroll
    for (int k = 0; k < K; k++) {
        const int c = lane + 32 * k;
        if (c < nx) {
            const double u = s_uu[c];
            const double bet = u != 0.0 ? s_w[c] / u : 0.0;
            if (!isfinite(bet) && c < badk) badk = c;
            s_w[c] = bet;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) badk = min(badk, __shfl_xor_sync(FULL_MASK, badk, o));
    __syncwarp();
    if (badk != 0x7fffffff) return sm + badk;
#pragma unroll
    for (int k = 0; k < K; k++) {
        const int c = lane + 32 * k;
        if (c < nx) {
            const double bet = s_w[c];
            const double inner = sub_rn(mul_rn(2.0, bet), mul_rn(mul_rn(bet, tdm[k]), bet));
            TDW[sq + c] = sub_rn(tdq[k], mul_rn(mul_rn(rs[k], inner), s_uu[c]));
            if (c >= 1)
                L1G[sq + c] = add_rn(l1q[k], mul_rn(mul_rn(mul_rn(mul_rn(rs[k], bet), s_l1m[c]), s_w[c - 1]),
                                                    s_uu[c - 1]));
            if (c + 1 < nx)
                U1G[sq + c] = add_rn(u1q[k], mul_rn(mul_rn(mul_rn(mul_rn(rs[k], bet), s_u1m[c]), s_w[c + 1]),
                                                    s_uu[c + 1]));
        }
    }
    __syncwarp();
    FTA(8)
    return -1;
}

struct FactorCtx {
    const double *a;  // (7,N) of this system: -nxy,-nx,-1,0,+1,+nx,+nxy
    double *pre;      // (7,N) output l1,u1,l2,u2,l3,u3,mr
    i64 n, nxy;
    int nx, ny, nz;
};

// _factor_plane (ntd_factor.py:147-219) by a warp pair on the corrected plane
// bands P (plane-local, 5 arrays).  Returns via err* (pair-shared).
template <int K>
__device__ void factor_plane_pair(const FactorCtx &c, i64 pb, const double *P[5], const PairScratch &S, int w2,
                                  int bar_id, volatile int *ecode, i64 *eplane, i64 *erow, int plane,
                                  double *lsm, volatile i64 *wbad, double *car)
{
    const int lane = threadIdx.x & 31;
    const int nx = c.nx, ny = c.ny, t2 = (ny - 1) / 2;
    double *L1G = c.pre + pb, *U1G = c.pre + c.n + pb, *MRG = c.pre + 6 * c.n + pb;
    double *TDW = S.at(S_TDW);
    double *sd = lsm, *sc = lsm + nx, *sm = lsm + 2 * nx;
    auto init_line = [&](int q) {
        i64 sq = (i64)q * nx;
        for (int cc = lane; cc < nx; cc += 32) {
            TDW[sq + cc] = P[0][sq + cc];
            L1G[sq + cc] = P[1][sq + cc];
            U1G[sq + cc] = P[2][sq + cc];
        }
        __syncwarp();
    };
    // each warp: (code, cell-row) of its first failure
    int mcode = 0;
    i64 mrow = -1;
    const int cnt = w2 == 0 ? t2 : (ny - 1 - t2);
    for (int i = 0; i < cnt && !mcode; i++) {
        int q = w2 == 0 ? i : ny - 1 - i;
        init_line(q);
        if (i > 0) {
            i64 st = correct_line_warp<K>(q, w2 == 0 ? q - 1 : q + 1, P[3], P[4], TDW, L1G, U1G, MRG, nx, lsm, car);
            if (st >= 0) {
                mcode = 2;
                mrow = st;
                break;
            }
        }
        int st = line_factor_warp(TDW + (i64)q * nx, L1G + (i64)q * nx, U1G + (i64)q * nx, MRG + (i64)q * nx, nx,
                                  sd, sc, sm);
        if (st >= 0) {
            mcode = 1;
            mrow = (i64)q * nx + st;
        }
    }
    if (lane == 0) {
        wbad[w2] = mcode;
        wbad[2 + w2] = mrow;
    }
    named_bar(bar_id, 64);
    int c0 = (int)wbad[0], c1 = (int)wbad[1];
    if (c0 || c1) {
        if (w2 == 0 && lane == 0) {
            int cc = c0 ? c0 : c1;
            i64 rr = wbad[2 + (c0 ? 0 : 1)];
            set_err(ecode, eplane, erow, cc, plane, pb + rr);
        }
        named_bar(bar_id, 64);
        return;
    }
    if (w2 == 0) {
        const int q = t2;
        init_line(q);
        i64 st = -1;
        int code = 0;
        if (t2 > 0) {
            st = correct_line_warp<K>(q, q - 1, P[3], P[4], TDW, L1G, U1G, MRG, nx, lsm, car);
            if (st >= 0) code = 2;
        }
        if (!code && t2 < ny - 1) {
            st = correct_line_warp<K>(q, q + 1, P[3], P[4], TDW, L1G, U1G, MRG, nx, lsm, car);
            if (st >= 0) code = 2;
        }
        if (!code) {
            int s2 = line_factor_warp(TDW + (i64)q * nx, L1G + (i64)q * nx, U1G + (i64)q * nx, MRG + (i64)q * nx, nx,
                                      sd, sc, sm);
            if (s2 >= 0) {
                code = 1;
                st = (i64)q * nx + s2;
            }
        }
        if (code && lane == 0) set_err(ecode, eplane, erow, code, plane, pb + st);
    }
    named_bar(bar_id, 64);
}

// correct_from (ntd_factor.py:378-404) for plane p through factored neighbour
// m, whose corrected (pre-factor) bands are Q.  Updates P in place.
template <int K>
__device__ void correct_from_pair(const FactorCtx &c, int p, int m, double *P[5], const double *Q[5],
                                  const PairScratch &S, int w2, int bar_id, double *ex, int &parity,
                                  volatile int *ecode, i64 *eplane, i64 *erow, volatile int *flag, double *lsm,
                                  double *car)
{
    const i64 nxy = c.nxy, n = c.n;
    const int nx = c.nx;
    const int tid = threadIdx.x & 63;
    const FactorPtrs F = factor_ptrs(c.pre, n);
    const double *useg = (m < p ? c.a + 6 * n : c.a) + (i64)m * nxy;  // u3 | l3 = copies of A's +-nxy
    const double *rowscale = (m < p ? c.a : c.a + 6 * n) + (i64)p * nxy;
    double *W = S.at(S_W), *BETA = S.at(S_BETA), *QD = S.at(S_QD);
    // _apply_factored_plane (ntd_factor.py:336-348): w = nested solve of plane m on u
    {
        FT0
        plane_solve_ref<K>(F, (i64)m * nxy, useg, W, c.nx, c.ny, w2, bar_id, lsm, car);
        FTA(1)
    }
    FT0
    // beta (_beta_from :242-249), qw (_plane_band_action :266-274), qd shift (:393-399)
    int fb = 0, fq = 0;
    // The plane loops below are elementwise over distinct scratch planes, walked by the pair's 64
    // threads: with the pointers held in no-alias locals (not re-read from the pointer arrays, which
    // live in local memory) every load of an iteration is issued before its first store, one memory
    // round trip per iteration instead of one per band.
    {
        const double *__restrict__ q0 = Q[0], *__restrict__ q1 = Q[1], *__restrict__ q2 = Q[2],
                     *__restrict__ q3 = Q[3], *__restrict__ q4 = Q[4];
        const double *__restrict__ us = useg, *__restrict__ Wr = W;
        double *__restrict__ Bo = BETA, *__restrict__ Qo = QD;
#pragma unroll 4
        for (i64 k = tid; k < nxy; k += 64) {
            double u = us[k], w = Wr[k];
            double bet = u != 0.0 ? w / u : 0.0;
            if (!isfinite(bet)) fb = 1;
            Bo[k] = bet;
            double qw = mul_rn(q0[k], w);
            if (k >= 1) qw = add_rn(qw, mul_rn(q1[k], Wr[k - 1]));
            if (k + 1 < nxy) qw = add_rn(qw, mul_rn(q2[k], Wr[k + 1]));
            if (k >= nx) qw = add_rn(qw, mul_rn(q3[k], Wr[k - nx]));
            if (k + nx < nxy) qw = add_rn(qw, mul_rn(q4[k], Wr[k + nx]));
            double qd = q0[k];
            if (w != 0.0) qd = add_rn(qd, sub_rn(u, qw) / w);
            if (!isfinite(qd)) fq = 1;
            Qo[k] = qd;
        }
    }
    if (fb) flag[0] = 1;
    if (fq) flag[1] = 1;
    named_bar(bar_id, 64);
    FTA(3)
    if (flag[0] || flag[1]) {
        if (tid == 0) set_err(ecode, eplane, erow, flag[0] ? 2 : 3, p, -1);
        named_bar(bar_id, 64);
        return;
    }
    // _plane_correction (ntd_factor.py:222-239)
    {
        FT0
        double *__restrict__ p0 = P[0], *__restrict__ p1 = P[1], *__restrict__ p2 = P[2], *__restrict__ p3 = P[3],
                            *__restrict__ p4 = P[4];
        const double *__restrict__ q1 = Q[1], *__restrict__ q2 = Q[2], *__restrict__ q3 = Q[3],
                     *__restrict__ q4 = Q[4];
        const double *__restrict__ us = useg, *__restrict__ rsc = rowscale, *__restrict__ Br = BETA,
                     *__restrict__ Qr = QD;
#pragma unroll 4
        for (i64 k = tid; k < nxy; k += 64) {
            double rs = rsc[k], bet = Br[k];
            double inner = sub_rn(mul_rn(2.0, bet), mul_rn(mul_rn(bet, Qr[k]), bet));
            p0[k] = sub_rn(p0[k], mul_rn(mul_rn(rs, inner), us[k]));
            double rb = mul_rn(rs, bet);
            if (k >= 1) p1[k] = add_rn(p1[k], mul_rn(mul_rn(mul_rn(rb, q1[k]), Br[k - 1]), us[k - 1]));
            if (k + 1 < nxy) p2[k] = add_rn(p2[k], mul_rn(mul_rn(mul_rn(rb, q2[k]), Br[k + 1]), us[k + 1]));
            if (k >= nx) p3[k] = add_rn(p3[k], mul_rn(mul_rn(mul_rn(rb, q3[k]), Br[k - nx]), us[k - nx]));
            if (k + nx < nxy) p4[k] = add_rn(p4[k], mul_rn(mul_rn(mul_rn(rb, q4[k]), Br[k + nx]), us[k + nx]));
        }
        named_bar(bar_id, 64);
        FTA(4)
    }
}

// plane_bands_of (ntd_factor.py:372-376): d, -1, +1, -nx, +nx of plane p
static __device__ void load_plane_bands(const FactorCtx &c, int p, double *P[5], int bar_id)
{
    const int tid = threadIdx.x & 63;
    const i64 pb = (i64)p * c.nxy, n = c.n;
    double *__restrict__ p0 = P[0], *__restrict__ p1 = P[1], *__restrict__ p2 = P[2], *__restrict__ p3 = P[3],
                        *__restrict__ p4 = P[4];
    const double *__restrict__ a = c.a + pb;
    FT0
#pragma unroll 4
    for (i64 k = tid; k < c.nxy; k += 64) {
        p0[k] = a[3 * n + k];
        p1[k] = a[2 * n + k];
        p2[k] = a[4 * n + k];
        p3[k] = a[1 * n + k];
        p4[k] = a[5 * n + k];
    }
    named_bar(bar_id, 64);
    FTA(0)
}

// factor_one (ntd_factor.py:406-419)
template <int K>
__device__ void factor_one_pair(const FactorCtx &c, int p, double *P[5], const PairScratch &S, int w2, int bar_id,
                                volatile int *ecode, i64 *eplane, i64 *erow, double *lsm, volatile i64 *wbad,
                                double *car)
{
    const int tid = threadIdx.x & 63;
    const i64 pb = (i64)p * c.nxy, n = c.n;
    FT0
    {
        const double *__restrict__ p3 = P[3], *__restrict__ p4 = P[4];
        double *__restrict__ o2 = c.pre + 2 * n + pb, *__restrict__ o3 = c.pre + 3 * n + pb;
#pragma unroll 4
        for (i64 k = tid; k < c.nxy; k += 64) {
            o2[k] = p3[k];
            o3[k] = p4[k];
        }
    }
    named_bar(bar_id, 64);
    FTA(5)
    const double *Pc[5] = {P[0], P[1], P[2], P[3], P[4]};
    {
        FT0
        factor_plane_pair<K>(c, pb, Pc, S, w2, bar_id, ecode, eplane, erow, p, lsm, wbad, car);
        FTA(6)
    }
}

template <int K>
__global__ void __launch_bounds__(128) k_ntd_factor(const double *__restrict__ a, double *pre, double *work,
                                                    int64_t *status, int nx, int ny, int nz)
{
    extern __shared__ double lsm_all[];  // 4 warps x LSM_PER_WARP x nx (line_solve_ref)
    __shared__ double ex[2][2 * 2 * (32 * K + 1)];
    __shared__ int ecode_s[2];
    __shared__ i64 eplane_s[2], erow_s[2];
    __shared__ i64 wbad_s[2][4];
    __shared__ int flag_s[2][2];
    __shared__ int last_p[2];
    __shared__ double car_s[4][2 * (REF_LANES + 1)];  // chain carries, per warp
    const i64 sys = blockIdx.x;
    const i64 nxy = (i64)nx * ny, n = nxy * nz;
    FactorCtx c;
    c.a = a + sys * 7 * n;
    c.pre = pre + sys * 7 * n;
    c.n = n;
    c.nxy = nxy;
    c.nx = nx;
    c.ny = ny;
    c.nz = nz;
    const int warp = __shfl_sync(FULL_MASK, (int)(threadIdx.x >> 5), 0), pair = warp >> 1, w2 = warp & 1, bar = 1 + pair;
    double *lsm = lsm_all + warp * LSM_PER_WARP * nx;
    double *car = car_s[warp];
    if (threadIdx.x < 2) {
        ecode_s[threadIdx.x] = 0;
        eplane_s[threadIdx.x] = -1;
        erow_s[threadIdx.x] = -1;
        last_p[threadIdx.x] = -1;
        flag_s[threadIdx.x][0] = flag_s[threadIdx.x][1] = 0;
    }
    // zero the factor (factor_level3 :365-369) and copy l3/u3 (:363-364)
    for (i64 k = threadIdx.x; k < n; k += blockDim.x) {
        c.pre[k] = 0.0;
        c.pre[n + k] = 0.0;
        c.pre[2 * n + k] = 0.0;
        c.pre[3 * n + k] = 0.0;
        c.pre[4 * n + k] = c.a[k];
        c.pre[5 * n + k] = c.a[6 * n + k];
        c.pre[6 * n + k] = 0.0;
    }
    __syncthreads();
    PairScratch S[2];
    for (int h = 0; h < 2; h++) {
        S[h].base = work + (sys * 2 + h) * S_PER_PAIR * nxy;
        S[h].nxy = nxy;
    }
    const PairScratch &MS = S[pair];
    volatile int *ecode = &ecode_s[pair];
    double *bufA[5], *bufB[5];
    for (int b = 0; b < 5; b++) {
        bufA[b] = MS.at(S_PC0 + b);
        bufB[b] = MS.at(S_PC1 + b);
    }
    double **Pcur = bufA, **Pprev = bufB;
    int parity = 0;
    const int t3 = (nz - 1) / 2;
    // run_half (ntd_factor.py:425-434)
    {
        int cntp = pair == 0 ? t3 : (nz - 1 - t3);
        int prev_p = -1;
        for (int i = 0; i < cntp; i++) {
            int p = pair == 0 ? i : nz - 1 - i;
            load_plane_bands(c, p, Pcur, bar);
            if (prev_p >= 0) {
                if ((threadIdx.x & 63) == 0) flag_s[pair][0] = flag_s[pair][1] = 0;
                named_bar(bar, 64);
                const double *Q[5] = {Pprev[0], Pprev[1], Pprev[2], Pprev[3], Pprev[4]};
                correct_from_pair<K>(c, p, prev_p, Pcur, Q, MS, w2, bar, ex[pair], parity, ecode, &eplane_s[pair],
                                     &erow_s[pair], flag_s[pair], lsm, car);
                if (*ecode) break;
            }
            factor_one_pair<K>(c, p, Pcur, MS, w2, bar, ecode, &eplane_s[pair], &erow_s[pair], lsm, wbad_s[pair],
                               car);
            if (*ecode) break;
            double **tmp = Pcur;
            Pcur = Pprev;
            Pprev = tmp;
            prev_p = p;
        }
        if ((threadIdx.x & 63) == 0) last_p[pair] = prev_p;
    }
    __syncthreads();
    // twist plane, corrected from both sides (ntd_factor.py:448-453)
    if (pair == 0 && !ecode_s[0] && !ecode_s[1]) {
        double *Pt[5];
        for (int b = 0; b < 5; b++) Pt[b] = Pcur[b];  // pair 0's free buffer
        load_plane_bands(c, t3, Pt, bar);
        int pa = last_p[0], pd = last_p[1];
        if (pa >= 0) {
            if ((threadIdx.x & 63) == 0) flag_s[0][0] = flag_s[0][1] = 0;
            named_bar(bar, 64);
            const double *Q[5] = {Pprev[0], Pprev[1], Pprev[2], Pprev[3], Pprev[4]};
            correct_from_pair<K>(c, t3, pa, Pt, Q, MS, w2, bar, ex[0], parity, ecode, &eplane_s[0], &erow_s[0],
                                 flag_s[0], lsm, car);
        }
        if (!*ecode && pd >= 0) {
            // pair 1's last corrected bands: its "Pprev" after the final swap
            int cnt1 = nz - 1 - t3;
            double *Q1[5];
            for (int b = 0; b < 5; b++) Q1[b] = S[1].at(((cnt1 & 1) ? S_PC0 : S_PC1) + b);
            if ((threadIdx.x & 63) == 0) flag_s[0][0] = flag_s[0][1] = 0;
            named_bar(bar, 64);
            const double *Q[5] = {Q1[0], Q1[1], Q1[2], Q1[3], Q1[4]};
            correct_from_pair<K>(c, t3, pd, Pt, Q, MS, w2, bar, ex[0], parity, ecode, &eplane_s[0], &erow_s[0],
                                 flag_s[0], lsm, car);
        }
        if (!*ecode)
            factor_one_pair<K>(c, t3, Pt, MS, w2, bar, ecode, &eplane_s[0], &erow_s[0], lsm, wbad_s[0], car);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        // the ascending half's error is reported first (fut_a.result(), :442)
        int h = ecode_s[0] ? 0 : (ecode_s[1] ? 1 : -1);
        status[sys * 3 + 0] = h >= 0 ? ecode_s[h] : 0;
        status[sys * 3 + 1] = h >= 0 ? eplane_s[h] : -1;
        status[sys * 3 + 2] = h >= 0 ? erow_s[h] : -1;
#ifdef FACTOR_TIMING
        if (sys == 0)
            printf("factor timing (warp 0, Mcycles): load_bands %llu  plane_solve %llu  [line_solve %llu]  beta/qd %llu  "
                   "plane_corr %llu  copy %llu  factor_plane %llu  [line_factor %llu  correct_line %llu]\n",
                   g_ft[0] >> 20, g_ft[1] >> 20, g_ft[2] >> 20, g_ft[3] >> 20, g_ft[4] >> 20, g_ft[5] >> 20,
                   g_ft[6] >> 20, g_ft[7] >> 20, g_ft[8] >> 20);
        if (sys == 0)
            printf("  line_solve parts: stage %llu  compose1 %llu  finish1 %llu  twist %llu  compose2 %llu  finish2 %llu  "
                   "writeback %llu\n", g_ft[9] >> 20, g_ft[10] >> 20, g_ft[11] >> 20, g_ft[12] >> 20, g_ft[13] >> 20,
                   g_ft[14] >> 20, g_ft[15] >> 20);
#endif
    }
}


// ---- per-K launchers (instantiated in ntd_k<K>.cu)
template <int K>
int launch_apply_k(const double *pre, const double *b, double *x, double *work, int nx, int ny, int nz, i64 batch,
                   const int32_t *active, cudaStream_t st);
template <int K>
int launch_factor_k(const double *a, double *pre, double *work, int64_t *status, int nx, int ny, int nz, i64 batch,
                    cudaStream_t st);

#define NTD_INSTANTIATE(K)                                                                                        \
    template <>                                                                                                    \
    int launch_apply_k<K>(const double *pre, const double *b, double *x, double *work, int nx, int ny, int nz,     \
                          i64 batch, const int32_t *active, cudaStream_t st)                                       \
    {                                                                                                              \
        k_ntd_apply<K><<<(unsigned)batch, 128, 0, st>>>(pre, b, x, work, nx, ny, nz, active);                      \
        return ntd::check_launch("ntd_apply");                                                                     \
    }                                                                                                              \
    template <>                                                                                                    \
    int launch_factor_k<K>(const double *a, double *pre, double *work, int64_t *status, int nx, int ny, int nz,    \
                           i64 batch, cudaStream_t st)                                                             \
    {                                                                                                              \
        size_t smem = sizeof(double) * 4 * LSM_PER_WARP * (size_t)nx;                                             \
        cudaError_t e = cudaFuncSetAttribute(k_ntd_factor<K>, cudaFuncAttributeMaxDynamicSharedMemorySize,         \
                                             (int)(smem > 48 * 1024 ? smem : 48 * 1024));                          \
        if (e != cudaSuccess) {                                                                                    \
            ntd::set_error("ntd_factor smem", e);                                                                  \
            return NTD_ELAUNCH;                                                                                    \
        }                                                                                                          \
        k_ntd_factor<K><<<(unsigned)batch, 128, smem, st>>>(a, pre, work, status, nx, ny, nz);                     \
        return ntd::check_launch("ntd_factor");                                                                    \
    }
