// ntd_apply_sl.cuh -- the production NTD apply (ntd_solve.py:107-322) on sm_100a.
//
// Mapping: one CTA per system; 4 solver warps (pair = level-3 half, warp of
// a pair = level-2 half, one warp per grid line) + 4 producer warps (producer
// w+4 feeds solver w from the same SM sub-partition).
//
// Slot layout (SL).  Every per-line array the apply touches is stored in
// "slot layout": a line of n cells becomes a record of LR = 32K+2 doubles
//     [ascending region 16K | twist cell | descending region 16K | 0]
// where region index r holds chain position j = r - P (P = 16K - chain
// length, start padding: r < P holds 0).  Lane s of half h owns slots
// k = 0..K-1 at region index s*K + k, so its K values are contiguous
// (immediate-offset shared loads, fully coalesced global loads/stores) and
// padded slots are zero maps that need no branches.  The factor (and its
// chain coefficients NL = -(l1*m), NU = -(u1*m)) is converted to SL once at
// setup (ntd_solve_bands); b is converted on entry and x back on exit.
//
// Per line step the solver waits on an mbarrier, reads its slots from a
// D-deep ring of line records streamed by 1-D bulk TMA (issued by the
// producer warp), forms the right-hand side, runs two 16-lane Kogge-Stone
// affine scans (ntd_line: lower and upper chains of the twisted line
// solve) and stores x.  x-dependent operands (neighbour plane, lower-sweep
// values of this plane) are loaded by the solver one line ahead.
#pragma once
#include "ntd_kernels.cuh"
#include "ntd_line4.cuh"

namespace sl {

#ifndef NTD_SL_PREFETCH_PLANES
#define NTD_SL_PREFETCH_PLANES 0
#endif
constexpr bool PREFETCH_PLANES = NTD_SL_PREFETCH_PLANES;  // whole-next-plane L2 prefetch (off: the TMA ring runs far enough ahead)

enum { SL_MR = 0, SL_NL, SL_NU, SL_L2, SL_U2, SL_L3, SL_U3, SL_N };  // solve arrays (SL)
constexpr int NPREP = 15;  // LinePrep coefficients per lane, stored [coef][lane] after the arrays

__host__ __device__ constexpr int lr_of(int K) { return 32 * K + 2; }
// doubles per line of the solve record: 7 SL arrays + the line's scan coefficients
__host__ __device__ constexpr int recd_of(int K) { return SL_N * lr_of(K) + NPREP * 32; }
// ring stage: one solve record + one extra line (b or xo)
__host__ __device__ constexpr int stage_of(int K) { return recd_of(K) + lr_of(K); }

__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
__device__ __forceinline__ void mbar_arrive(void *bar)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// index of cell c of a line of n cells inside its SL record
__device__ __forceinline__ int sl_index(int c, int n, int K)
{
    const int t = (n - 1) / 2;
    if (c == t) return 16 * K;
    if (c < t) return c + (16 * K - t);                       // asc: r = j + P0, j = c
    return 16 * K + 1 + (n - 1 - c) + (16 * K - (n - 1 - t));  // desc: r = j + P1, j = n-1-c
}

// natural (B, N) <-> SL (B, N_SL).  One thread per SL element / cell.
static __global__ void k_to_sl(const double *__restrict__ src, double *__restrict__ dst, int nx, i64 lines, int K,
                        i64 batch)
{
    const int LR = lr_of(K);
    const i64 total = lines * LR * batch;
    const int t = (nx - 1) / 2;
    const int P0 = 16 * K - t, P1 = 16 * K - (nx - 1 - t);
    for (i64 e = blockIdx.x * (i64)blockDim.x + threadIdx.x; e < total; e += (i64)gridDim.x * blockDim.x) {
        const i64 line = e / LR;  // global line over batch
        const int r = (int)(e - line * LR);
        int c = -1;
        if (r < 16 * K) {
            const int j = r - P0;
            if (j >= 0) c = j;
        } else if (r == 16 * K) {
            c = t;
        } else if (r < 32 * K + 1) {
            const int j = r - (16 * K + 1) - P1;
            if (j >= 0) c = nx - 1 - j;
        }
        dst[e] = c >= 0 ? src[line * nx + c] : 0.0;
    }
}

static __global__ void k_from_sl(const double *__restrict__ src, double *__restrict__ dst, int nx, i64 lines, int K,
                          i64 batch)
{
    const int LR = lr_of(K);
    const i64 total = lines * nx * batch;
    for (i64 e = blockIdx.x * (i64)blockDim.x + threadIdx.x; e < total; e += (i64)gridDim.x * blockDim.x) {
        const i64 line = e / nx;
        const int c = (int)(e - line * nx);
        dst[e] = src[line * LR + sl_index(c, nx, K)];
    }
}

// solve arrays in SL from a factor (B,7,N): mr, -(l1 mr), -(u1 mr), l2, u2, l3, u3
static __global__ void k_solve_sl(const double *__restrict__ pre, double *__restrict__ solve, int nx, i64 lines, int K,
                           i64 batch)
{
    const int LR = lr_of(K);
    const i64 nsl = lines * LR, n = lines * nx;
    const i64 total = nsl * batch;
    const int t = (nx - 1) / 2;
    const int P0 = 16 * K - t, P1 = 16 * K - (nx - 1 - t);
    for (i64 e = blockIdx.x * (i64)blockDim.x + threadIdx.x; e < total; e += (i64)gridDim.x * blockDim.x) {
        const i64 s = e / nsl, el = e - s * nsl;
        const i64 line = el / LR;
        const int r = (int)(el - line * LR);
        int c = -1;
        if (r < 16 * K) {
            const int j = r - P0;
            if (j >= 0) c = j;
        } else if (r == 16 * K) {
            c = t;
        } else if (r < 32 * K + 1) {
            const int j = r - (16 * K + 1) - P1;
            if (j >= 0) c = nx - 1 - j;
        }
        const double *p = pre + s * 7 * n;
        // record-major: [system][line][array][LR] -> one bulk copy per line
        double *o = solve + (s * lines + line) * (i64)(SL_N * LR + NPREP * 32) + r;
        const i64 g = line * nx + c;
        const double m = c >= 0 ? p[6 * n + g] : 0.0;
        o[SL_MR * LR] = m;
        o[SL_NL * LR] = c >= 0 ? -(p[g] * m) : 0.0;
        o[SL_NU * LR] = c >= 0 ? -(p[n + g] * m) : 0.0;
        o[SL_L2 * LR] = c >= 0 ? p[2 * n + g] : 0.0;
        o[SL_U2 * LR] = c >= 0 ? p[3 * n + g] : 0.0;
        o[SL_L3 * LR] = c >= 0 ? p[4 * n + g] : 0.0;
        o[SL_U3 * LR] = c >= 0 ? p[5 * n + g] : 0.0;
    }
}

// twist row: xt = bt*mt + NLt*xa + NUt*xd (= (bt - l1t xa - u1t xd) mt)
template <int K>
__device__ __forceinline__ void line_solve(int s, int n, int t, const double (&aL)[K], const double (&mr)[K],
                                           const double (&aU)[K], const double (&rhs)[K], double bt, double mrt,
                                           double nlt, double nut, double (&x)[K], double &xt)
{
    double A = 1.0, C = 0.0;
#pragma unroll
    for (int k = 0; k < K; k++) {
        C = fma(aL[k], C, rhs[k] * mr[k]);
        A = aL[k] * A;
    }
#pragma unroll
    for (int d = 1; d < 16; d <<= 1) {
        const double Ao = __shfl_up_sync(FULL_MASK, A, d, 16);
        const double Co = __shfl_up_sync(FULL_MASK, C, d, 16);
        if (s >= d) {
            C = fma(A, Co, C);
            A = A * Ao;
        }
    }
    double xc = __shfl_up_sync(FULL_MASK, C, 1, 16);
    if (s == 0) xc = 0.0;
#pragma unroll
    for (int k = 0; k < K; k++) {
        xc = fma(aL[k], xc, rhs[k] * mr[k]);
        x[k] = xc;
    }
    const double xa = __shfl_sync(FULL_MASK, x[K - 1], 15);
    const double xd = __shfl_sync(FULL_MASK, x[K - 1], 31);
    double acc = bt * mrt;
    if (t > 0) acc = fma(nlt, xa, acc);
    if (t < n - 1) acc = fma(nut, xd, acc);
    xt = acc;
    A = 1.0;
    C = 0.0;
#pragma unroll
    for (int k = K - 1; k >= 0; k--) {
        C = fma(aU[k], C, x[k]);
        A = aU[k] * A;
    }
#pragma unroll
    for (int d = 1; d < 16; d <<= 1) {
        const double Ao = __shfl_down_sync(FULL_MASK, A, d, 16);
        const double Co = __shfl_down_sync(FULL_MASK, C, d, 16);
        if (s + d < 16) {
            C = fma(A, Co, C);
            A = A * Ao;
        }
    }
    const double An = __shfl_down_sync(FULL_MASK, A, 1, 16);
    const double Cn = __shfl_down_sync(FULL_MASK, C, 1, 16);
    xc = (s == 15) ? xt : fma(An, xt, Cn);
#pragma unroll
    for (int k = K - 1; k >= 0; k--) {
        xc = fma(aU[k], xc, x[k]);
        x[k] = xc;
    }
}

// ---------------------------------------------------------------- data
struct SlArrays {  // one system, SL
    const double *solve;  // record-major solve records [line][recd_of(K)]
    const double *b;
    double *x, *xs;
    i64 nsl;
};

// per-lane slot access (lane base inside a record)
template <int K>
struct LaneSl {
    int base;  // element index of slot 0 within a record
    int tw;    // twist element (16K)
    bool desc;
    __device__ __forceinline__ LaneSl(int lane)
    {
        desc = lane >= 16;
        base = (desc ? 16 * K + 1 : 0) + (lane & 15) * K;
        tw = 16 * K;
    }
};

template <int K>
__device__ __forceinline__ void ld_rec(const double *rec, const LaneSl<K> &L, double (&v)[K], double &vt)
{
#pragma unroll
    for (int k = 0; k < K; k++) v[k] = rec[L.base + k];
    vt = rec[L.tw];
}
template <int K>
__device__ __forceinline__ void ld_rec(const double *rec, const LaneSl<K> &L, double (&v)[K])
{
#pragma unroll
    for (int k = 0; k < K; k++) v[k] = rec[L.base + k];
}
template <int K>
__device__ __forceinline__ void st_rec(double *rec, const LaneSl<K> &L, const double (&v)[K], double vt, int lane)
{
    (void)lane;
#pragma unroll
    for (int k = 0; k < K; k++) rec[L.base + k] = v[k];
    rec[L.tw] = vt;  // every lane holds the same twist value: branch-free
}

// ring of D stages x RSEG line records per solver warp
constexpr int G_X = SL_N;      // ring segment holding b (lower lines of LOWER3) or xo (upper lines of UPPER3)
constexpr int G_PREP = SL_N + 1;  // the record's scan coefficients

template <int K, int D>
struct Ring {
    double *base;
    unsigned long long *full, *empty;
    __device__ __forceinline__ double *seg(int st, int g) const
    {
        double *b0 = base + (size_t)st * stage_of(K);
        return g < SL_N ? b0 + g * lr_of(K) : (g == G_X ? b0 + recd_of(K) : b0 + SL_N * lr_of(K));
    }
};

struct PlaneDesc {
    i64 prec;      // record index of the plane's first line (plane * ny)
    int mode;      // M_LOWER3 / M_UPPER3
    bool hasM, hasP, nbrUp;
    bool up;       // lower sweep: the level-3 neighbour is plane p+1 (descending half)
};

struct Seq {
    int cnt, t2, ny, w2;
    __device__ __forceinline__ int qlow(int i) const { return w2 == 0 ? i : ny - 1 - i; }
    __device__ __forceinline__ int qup(int i) const { return w2 == 0 ? t2 - 1 - i : t2 + 1 + i; }
};

__device__ __forceinline__ LinePrep read_prep(const double *pp, int lane)
{
    LinePrep P;
    P.p1 = pp[0 * 32 + lane];
    P.p2 = pp[1 * 32 + lane];
    P.p3 = pp[2 * 32 + lane];
    P.e0 = pp[3 * 32 + lane];
    P.e1 = pp[4 * 32 + lane];
    P.e2 = pp[5 * 32 + lane];
    P.e3 = pp[6 * 32 + lane];
    P.q1 = pp[7 * 32 + lane];
    P.q2 = pp[8 * 32 + lane];
    P.q3 = pp[9 * 32 + lane];
    P.f0 = pp[10 * 32 + lane];
    P.f1 = pp[11 * 32 + lane];
    P.f2 = pp[12 * 32 + lane];
    P.f3 = pp[13 * 32 + lane];
    P.bex = pp[14 * 32 + lane];
    return P;
}

// scan coefficients of every line (setup): one warp per line
template <int K>
__global__ void k_prep_sl(double *__restrict__ solve, i64 lines_total)
{
    constexpr int LR = lr_of(K);
    const int lane = threadIdx.x & 31;
    const i64 line = (blockIdx.x * (i64)blockDim.x + threadIdx.x) >> 5;
    if (line >= lines_total) return;
    double *rec = solve + line * (i64)recd_of(K);
    const LaneSl<K> L(lane);
    double aL[K], aU[K];
    ld_rec(rec + (L.desc ? SL_NU : SL_NL) * LR, L, aL);
    ld_rec(rec + (L.desc ? SL_NL : SL_NU) * LR, L, aU);
    const LinePrep P = line_prep<K>(lane & 15, aL, aU);
    double *pp = rec + SL_N * LR;
    const double v[NPREP] = {P.p1, P.p2, P.p3, P.e0, P.e1, P.e2, P.e3, P.q1, P.q2, P.q3, P.f0, P.f1, P.f2, P.f3, P.bex};
#pragma unroll
    for (int c = 0; c < NPREP; c++) pp[c * 32 + lane] = v[c];
}

// ---------------- producer: bulk copies of one plane's line records
template <int K, int D>
__device__ void produce_plane(const SlArrays &S, const PlaneDesc &P, const Seq &Q, const Ring<K, D> &R,
                              unsigned &rec)
{
    const int lane = threadIdx.x & 31;
    constexpr int LR = lr_of(K);
    const unsigned rbytes = LR * 8u;
    const unsigned recbytes = recd_of(K) * 8u;
    for (int ph = 0; ph < 2; ph++) {
        for (int i = 0; i < Q.cnt; i++, rec++) {
            if (lane == 0) {
                const int st = rec % D;
                if (rec >= (unsigned)D) mbar_wait_lazy(&R.empty[st], ((rec / D) + 1) & 1);
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                unsigned long long *bar = &R.full[st];
                const int q = ph == 0 ? Q.qlow(i) : Q.qup(i);
                const i64 line = P.prec + q;
                const bool extra = ph == 0 ? P.mode == M_LOWER3 : P.mode == M_UPPER3;
                mbar_expect_tx(bar, recbytes + (extra ? rbytes : 0u));
                tma_load_1d(R.seg(st, 0), S.solve + line * (i64)recd_of(K), recbytes, bar);
                if (extra) tma_load_1d(R.seg(st, G_X), (ph == 0 ? S.b : S.x) + line * (i64)LR, rbytes, bar);
            }
        }
    }
    __syncwarp();
}

// ---------------- solver: one plane
template <int K, int D, int MODE, bool TWO>
__device__ void solve_plane(const SlArrays &S, const PlaneDesc &P, const Seq &Q, int nx, int bar_id, double *ex,
                            int &parity, const Ring<K, D> &R, const LaneSl<K> &L, unsigned &rec)
{
    constexpr int LR = lr_of(K);
    const int lane = threadIdx.x & 31, s = lane & 15, w2 = Q.w2;
    const int ny = Q.ny, t2 = Q.t2, cnt = Q.cnt, t = (nx - 1) / 2;
    const i64 plr = (i64)ny * LR;  // plane stride in SL
    const bool lower3 = P.mode == M_LOWER3;
    // x-dependent neighbour planes
    // Neighbour planes.  A missing neighbour has an exactly-zero l3/u3
    // coefficient (first/last plane), so it is pointed at this plane's own
    // (finite, zero-initialised) x record instead of branching.
    const double *y1, *y2 = S.x;
    int gC1;
    if (lower3) {
        if (TWO) {
            gC1 = SL_L3;
            y1 = P.hasM ? S.x - plr : S.x;
            y2 = P.hasP ? S.x + plr : S.x;
        } else if (P.up) {
            gC1 = SL_U3;
            y1 = P.hasP ? S.x + plr : S.x;
        } else {
            gC1 = SL_L3;
            y1 = P.hasM ? S.x - plr : S.x;
        }
    } else {
        gC1 = P.nbrUp ? SL_U3 : SL_L3;
        y1 = P.nbrUp ? S.x + plr : S.x - plr;
    }
    double *xlow = lower3 ? S.x : S.xs;  // lower-sweep store of this plane
    const int gL = L.desc ? SL_NU : SL_NL, gU = L.desc ? SL_NL : SL_NU;
    const int gCL = w2 == 0 ? SL_L2 : SL_U2, gCU = w2 == 0 ? SL_U2 : SL_L2;
    auto recp = [&](const double *base, int q) { return base + (P.prec + q) * (i64)LR; };
    auto srec = [&](int a, int q) { return S.solve + (P.prec + q) * (i64)recd_of(K) + a * LR; };
    auto recw = [&](double *base, int q) { return base + (P.prec + q) * (i64)LR; };
    double xprev[K], xprevt = 0.0;
#pragma unroll
    for (int k = 0; k < K; k++) xprev[k] = 0.0;
    // ---------------- level-2 lower sweep (ntd_solve.py:147-171)
    double n1[K], n1t = 0.0, n2[K], n2t = 0.0;
#pragma unroll
    for (int k = 0; k < K; k++) n1[k] = n2[k] = 0.0;
    if (cnt > 0) {
        ld_rec(recp(y1, Q.qlow(0)), L, n1, n1t);
        if (TWO) ld_rec(recp(y2, Q.qlow(0)), L, n2, n2t);
    }
    for (int i = 0; i < cnt; i++, rec++) {
        double v1[K], v1t = n1t, v2[K], v2t = n2t;
#pragma unroll
        for (int k = 0; k < K; k++) {
            v1[k] = n1[k];
            v2[k] = n2[k];
        }
        if (i + 1 < cnt) {
            ld_rec(recp(y1, Q.qlow(i + 1)), L, n1, n1t);
            if (TWO) ld_rec(recp(y2, Q.qlow(i + 1)), L, n2, n2t);
        }
        const int st = rec % D;
        TSTAMP(q1);
        mbar_wait(&R.full[st], (rec / D) & 1);
        TSTAMP(q2);
        TACC(0, q1, q2);
        double aL[K], mr[K], aU[K], rhs[K], mrt, nlt, nut, rhst;
        ld_rec(R.seg(st, SL_MR), L, mr, mrt);
        ld_rec(R.seg(st, gL), L, aL);
        ld_rec(R.seg(st, gU), L, aU);
        nlt = R.seg(st, SL_NL)[L.tw];
        nut = R.seg(st, SL_NU)[L.tw];
        if (lower3) {
            ld_rec(R.seg(st, G_X), L, rhs, rhst);
            {
                double c[K], ct;
                ld_rec(R.seg(st, gC1), L, c, ct);
#pragma unroll
                for (int k = 0; k < K; k++) rhs[k] -= c[k] * v1[k];
                rhst -= ct * v1t;
            }
            if (TWO) {
                double c[K], ct;
                ld_rec(R.seg(st, SL_U3), L, c, ct);
#pragma unroll
                for (int k = 0; k < K; k++) rhs[k] -= c[k] * v2[k];
                rhst -= ct * v2t;
            }
        } else {
            double c[K], ct;
            ld_rec(R.seg(st, gC1), L, c, ct);
#pragma unroll
            for (int k = 0; k < K; k++) rhs[k] = c[k] * v1[k];
            rhst = ct * v1t;
        }
        {
            double cp[K], cpt;  // line 0: xprev = 0, so the term vanishes
            ld_rec(R.seg(st, gCL), L, cp, cpt);
#pragma unroll
            for (int k = 0; k < K; k++) rhs[k] -= cp[k] * xprev[k];
            rhst -= cpt * xprevt;
        }
        const int st_rel = st;
        TSTAMP(q3);
        TACC(1, q2, q3);
        double x[K], xt;
        { const LinePrep PP_ = read_prep(R.seg(st_rel, G_PREP), lane); double cr_[K];
#pragma unroll
        for (int k_ = 0; k_ < K; k_++) cr_[k_] = (rhs)[k_] * mr[k_];
        line_solve4<K>(PP_, nx, t, aL, cr_, aU, (rhst) * mrt, nlt, nut, x, xt); }
        TSTAMP(q4);
        TACC(2, q3, q4);
        mbar_arrive(&R.empty[st_rel]);
        st_rec(recw(xlow, Q.qlow(i)), L, x, xt, lane);
        TSTAMP(q5);
        TACC(3, q4, q5);
#pragma unroll
        for (int k = 0; k < K; k++) xprev[k] = x[k];
        xprevt = xt;
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
    double xa[K], xat, xd[K], xdt;
    {
        double xo[K], xot = other[32 * K];
#pragma unroll
        for (int k = 0; k < K; k++) xo[k] = other[lane * K + k];
#pragma unroll
        for (int k = 0; k < K; k++) {
            xa[k] = w2 == 0 ? xprev[k] : xo[k];
            xd[k] = w2 == 0 ? xo[k] : xprev[k];
        }
        xat = w2 == 0 ? xprevt : xot;
        xdt = w2 == 0 ? xot : xprevt;
    }
    // ---------------- twist line (ntd_solve.py:172-177), direct loads after
    // the barrier (the neighbour plane's twist line was written by warp 0)
    double xn[K], xnt;
    double yv[K], yvt = 0.0;
    {
        const int q = t2;
        double aL[K], mr[K], aU[K], mrt, nlt, nut, rhs[K], rhst;
        ld_rec(srec(SL_MR, q), L, mr, mrt);
        ld_rec(srec(gL, q), L, aL);
        ld_rec(srec(gU, q), L, aU);
        nlt = srec(SL_NL, q)[L.tw];
        nut = srec(SL_NU, q)[L.tw];
        if (lower3) {
            ld_rec(recp(S.b, q), L, rhs, rhst);
            if (P.hasM) {
                double c[K], ct, y[K], yt;
                ld_rec(srec(SL_L3, q), L, c, ct);
                ld_rec(recp(S.x - plr, q), L, y, yt);
#pragma unroll
                for (int k = 0; k < K; k++) rhs[k] -= c[k] * y[k];
                rhst -= ct * yt;
            }
            if (P.hasP) {
                double c[K], ct, y[K], yt;
                ld_rec(srec(SL_U3, q), L, c, ct);
                ld_rec(recp(S.x + plr, q), L, y, yt);
#pragma unroll
                for (int k = 0; k < K; k++) rhs[k] -= c[k] * y[k];
                rhst -= ct * yt;
            }
        } else {
            double c[K], ct, y[K], yt;
            ld_rec(srec(gC1, q), L, c, ct);
            ld_rec(recp(y1, q), L, y, yt);
#pragma unroll
            for (int k = 0; k < K; k++) rhs[k] = c[k] * y[k];
            rhst = ct * yt;
        }
        if (t2 > 0) {
            double c[K], ct;
            ld_rec(srec(SL_L2, q), L, c, ct);
#pragma unroll
            for (int k = 0; k < K; k++) rhs[k] -= c[k] * xa[k];
            rhst -= ct * xat;
        }
        if (t2 < ny - 1) {
            double c[K], ct;
            ld_rec(srec(SL_U2, q), L, c, ct);
#pragma unroll
            for (int k = 0; k < K; k++) rhs[k] -= c[k] * xd[k];
            rhst -= ct * xdt;
        }
        if (cnt > 0) ld_rec(recp(xlow, Q.qup(0)), L, yv, yvt);  // first upper line's lower value
        { const LinePrep PP_ = line_prep<K>(s, aL, aU); double cr_[K];
#pragma unroll
        for (int k_ = 0; k_ < K; k_++) cr_[k_] = (rhs)[k_] * mr[k_];
        line_solve4<K>(PP_, nx, t, aL, cr_, aU, (rhst) * mrt, nlt, nut, xn, xnt); }
        if (w2 == 0) {
            if (lower3) {
                st_rec(recw(S.x, q), L, xn, xnt, lane);
            } else {
                double xo[K], xot, nv[K];
                ld_rec(recp(S.x, q), L, xo, xot);
#pragma unroll
                for (int k = 0; k < K; k++) nv[k] = xo[k] - xn[k];
                st_rec(recw(S.x, q), L, nv, xot - xnt, lane);
            }
        }
    }
    // ---------------- level-2 upper sweep (ntd_solve.py:178-185)
    for (int i = 0; i < cnt; i++, rec++) {
        double y[K], yt = yvt;
#pragma unroll
        for (int k = 0; k < K; k++) y[k] = yv[k];
        if (i + 1 < cnt) ld_rec(recp(xlow, Q.qup(i + 1)), L, yv, yvt);
        const int st = rec % D;
        mbar_wait(&R.full[st], (rec / D) & 1);
        double aL[K], mr[K], aU[K], cp[K], mrt, nlt, nut, cpt;
        ld_rec(R.seg(st, SL_MR), L, mr, mrt);
        ld_rec(R.seg(st, gL), L, aL);
        ld_rec(R.seg(st, gU), L, aU);
        nlt = R.seg(st, SL_NL)[L.tw];
        nut = R.seg(st, SL_NU)[L.tw];
        ld_rec(R.seg(st, gCU), L, cp, cpt);
        double xo[K], xot = 0.0;
        if (!lower3) ld_rec(R.seg(st, G_X), L, xo, xot);
        const int st_rel = st;
        double bs[K];
#pragma unroll
        for (int k = 0; k < K; k++) bs[k] = cp[k] * xn[k];
        double xs[K], xst;
        { const LinePrep PP_ = read_prep(R.seg(st_rel, G_PREP), lane); double cr_[K];
#pragma unroll
        for (int k_ = 0; k_ < K; k_++) cr_[k_] = (bs)[k_] * mr[k_];
        line_solve4<K>(PP_, nx, t, aL, cr_, aU, (cpt * xnt) * mrt, nlt, nut, xs, xst); }
        mbar_arrive(&R.empty[st_rel]);
#pragma unroll
        for (int k = 0; k < K; k++) xn[k] = y[k] - xs[k];
        xnt = yt - xst;
        if (!lower3) {
            double nv[K];
#pragma unroll
            for (int k = 0; k < K; k++) nv[k] = xo[k] - xn[k];
            st_rec(recw(S.x, Q.qup(i)), L, nv, xot - xnt, lane);
        } else {
            st_rec(recw(S.x, Q.qup(i)), L, xn, xnt, lane);
        }
    }
}

// L2 prefetch of one plane's SL records this warp will read (producers)
__device__ __forceinline__ void prefetch_sl(const double *p, i64 r0, i64 r1)
{
    if (!p || r1 <= r0) return;
    const char *c = (const char *)(p + r0);
    const i64 bytes = (r1 - r0) * 8;
    for (i64 off = (i64)(threadIdx.x & 31) * 128; off < bytes; off += 32 * 128) prefetch_l2(c + off);
}

template <int K, int D>
__global__ void __launch_bounds__(256, 1) k_apply(const double *__restrict__ solve, const double *__restrict__ bsl,
                                                  double *xsl, double *xssl, int nx, int ny, int nz,
                                                  const int32_t *__restrict__ active)
{
    extern __shared__ __align__(128) double sl_ring[];
    __shared__ double ex[2][2 * 2 * (32 * K + 1)];
    __shared__ __align__(8) unsigned long long bars[4][2 * D];
    constexpr int LR = lr_of(K);
    const i64 sys = blockIdx.x;
    if (active && !active[sys]) return;
    const i64 nsl = (i64)nz * ny * LR;
    SlArrays S;
    S.solve = solve + sys * (i64)nz * ny * recd_of(K);
    S.b = bsl + sys * nsl;
    S.x = xsl + sys * nsl;
    S.xs = xssl + sys * nsl;
    S.nsl = nsl;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const bool producer = warp >= 4;
    const int sw = warp & 3, pair = sw >> 1, w2 = sw & 1, bar = 1 + pair;
    Ring<K, D> R;
    R.base = sl_ring + (size_t)sw * D * stage_of(K);
    R.full = bars[sw];
    R.empty = bars[sw] + D;
    if (!producer && lane == 0) {
        for (int st = 0; st < D; st++) {
            mbar_init(&R.full[st], 1);
            mbar_init(&R.empty[st], 32);  // every solver lane arrives: no divergent branch
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const LaneSl<K> L(lane);
    Seq Q;
    Q.ny = ny;
    Q.t2 = (ny - 1) / 2;
    Q.w2 = w2;
    Q.cnt = w2 == 0 ? Q.t2 : (ny - 1 - Q.t2);
    unsigned rec = 0;
    double *myex = ex[pair];
    int parity = 0;
    const int t3 = (nz - 1) / 2;
    const i64 plr = (i64)ny * LR;
    // warp's row range of a plane (for L2 prefetch)
    const i64 wr0 = w2 == 0 ? 0 : (i64)Q.t2 * LR, wr1 = w2 == 0 ? (i64)(Q.t2 + 1) * LR : plr;
    auto prefetch_plane_sl = [&](int p, bool upper) {
        if (!PREFETCH_PLANES) return;
        const i64 b0 = (i64)p * plr;
        prefetch_sl(S.solve, (b0 + wr0) / LR * recd_of(K), (b0 + wr1) / LR * recd_of(K));
        prefetch_sl(upper ? S.x : S.b, b0 + wr0, b0 + wr1);
    };
    // level-3 lower sweep (ntd_solve.py:198-221)
    const int nlow = pair == 0 ? t3 : nz - 1 - t3;
    if (producer) prefetch_plane_sl(pair == 0 ? 0 : nz - 1, false);
    for (int i = 0; i < nlow; i++) {
        const int p = pair == 0 ? i : nz - 1 - i;
        PlaneDesc P;
        P.prec = (i64)p * ny;
        P.mode = M_LOWER3;
        P.hasM = pair == 0 && p > 0;
        P.hasP = pair == 1 && p < nz - 1;
        P.nbrUp = false;
        P.up = pair == 1;
        if (producer) {
            if (i + 1 < nlow) prefetch_plane_sl(pair == 0 ? p + 1 : p - 1, false);
            produce_plane<K, D>(S, P, Q, R, rec);
        } else {
            solve_plane<K, D, M_LOWER3, false>(S, P, Q, nx, bar, myex, parity, R, L, rec);
        }
    }
    __syncthreads();
    // twist plane (ntd_solve.py:222-232): pair 0, both level-3 neighbours
    if (pair == 0) {
        PlaneDesc P;
        P.prec = (i64)t3 * ny;
        P.mode = M_LOWER3;
        P.hasM = t3 > 0;
        P.hasP = t3 < nz - 1;
        P.nbrUp = false;
        P.up = false;
        if (producer) {
            fence_proxy_async();
            produce_plane<K, D>(S, P, Q, R, rec);
        } else {
            solve_plane<K, D, M_LOWER3, true>(S, P, Q, nx, bar, myex, parity, R, L, rec);
        }
    }
    __syncthreads();
    if (producer) fence_proxy_async();  // x (read as xo) was written by generic stores
    // level-3 upper sweep (ntd_solve.py:233-253)
    if (producer && nlow > 0) prefetch_plane_sl(pair == 0 ? t3 - 1 : t3 + 1, true);
    for (int i = 0; i < nlow; i++) {
        const int p = pair == 0 ? t3 - 1 - i : t3 + 1 + i;
        PlaneDesc P;
        P.prec = (i64)p * ny;
        P.mode = M_UPPER3;
        P.hasM = P.hasP = false;
        P.nbrUp = pair == 0;
        P.up = false;
        if (producer) {
            if (i + 1 < nlow) prefetch_plane_sl(pair == 0 ? p - 1 : p + 1, true);
            produce_plane<K, D>(S, P, Q, R, rec);
        } else {
            solve_plane<K, D, M_UPPER3, false>(S, P, Q, nx, bar, myex, parity, R, L, rec);
        }
    }
}

}  // namespace sl

template <int K>
int launch_prep_sl_k(double *solve, i64 lines_total, cudaStream_t st);
template <int K>
int launch_apply_sl_k(const double *solve, const double *bsl, double *xsl, double *xssl, int nx, int ny, int nz,
                      i64 batch, const int32_t *active, cudaStream_t st, int depth);

#define NTD_INSTANTIATE_SL(K)                                                                                     \
    template <>                                                                                                    \
    int launch_prep_sl_k<K>(double *solve, i64 lines_total, cudaStream_t st)                                      \
    {                                                                                                              \
        const i64 threads = lines_total * 32;                                                                      \
        sl::k_prep_sl<K><<<(unsigned)((threads + 255) / 256), 256, 0, st>>>(solve, lines_total);                  \
        return ntd::check_launch("ntd_solve_bands prep");                                                          \
    }                                                                                                              \
    template <>                                                                                                    \
    int launch_apply_sl_k<K>(const double *solve, const double *bsl, double *xsl, double *xssl, int nx, int ny,    \
                             int nz, i64 batch, const int32_t *active, cudaStream_t st, int depth)                 \
    {                                                                                                              \
        size_t smem = (size_t)4 * depth * sl::stage_of(K) * 8;                                                     \
        cudaError_t e = depth == 4                                                                                 \
            ? cudaFuncSetAttribute(sl::k_apply<K, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)      \
            : cudaFuncSetAttribute(sl::k_apply<K, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);     \
        if (e != cudaSuccess) {                                                                                    \
            ntd::set_error("ntd_apply smem", e);                                                                   \
            return NTD_ELAUNCH;                                                                                    \
        }                                                                                                          \
        if (depth == 4)                                                                                            \
            sl::k_apply<K, 4><<<(unsigned)batch, 256, smem, st>>>(solve, bsl, xsl, xssl, nx, ny, nz, active);      \
        else                                                                                                       \
            sl::k_apply<K, 2><<<(unsigned)batch, 256, smem, st>>>(solve, bsl, xsl, xssl, nx, ny, nz, active);      \
        return ntd::check_launch("ntd_apply");                                                                     \
    }
