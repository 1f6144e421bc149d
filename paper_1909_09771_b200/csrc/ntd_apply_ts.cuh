// ntd_apply_ts.cuh -- the production NTD apply (ntd_solve.py:107-322) on sm_100a,
// two-sided line solves (ntd_line_ts.cuh).
//
// Mapping: one CTA (or a cluster of two CTAs, one level-3 half each) per
// system; a solver warp per level-2 half (one warp per grid line), a producer
// warp per solver warp streaming line records by 1-D bulk TMA into an
// mbarrier ring.
//
// Lane layout (TS).  A line of n <= 32K cells is a record of LR = 32K doubles;
// cell c lives at element (c % K) * 32 + c / K: lane l owns the K consecutive
// cells lK .. lK+K-1 and its slot k is element 32k + l, so every warp access
// is one conflict-free, fully coalesced row of 32 doubles.  Elements of cells
// >= n are zero in every array (zero maps: no branches).
//
// Solve record of one line (record-major, [system][line][RECD]), derived once
// at setup from the factor (ntd_solve_bands):
//   [ EFB (eF, eB pairs, 2 LR) | PREP (NPREP x 32, pairs) | L2' | U2' | L3' | U3' ]
// eF / eB are the scaled elimination multipliers of the two-sided solve,
// PREP the factor-only scan coefficients, and the couplings are pre-multiplied
// by mu (the twisted pivot reciprocal at the cell): c' = c mu, as is the
// right-hand side on entry (b' = b mu).  The mu of every cell follows the
// records ([system][line][LR]) for the kernels that form b'.
#pragma once
#include "ntd_kernels.cuh"
#include "ntd_line_ts.cuh"

namespace ts {

constexpr int NPREP = 12;  // stored PrepTS coefficients per lane; p1 and q1 are rebuilt
__host__ __device__ constexpr int lr_of(int K) { return 32 * K; }
__host__ __device__ constexpr int o_efb(int K) { return 0; }
__host__ __device__ constexpr int o_prep(int K) { return 2 * lr_of(K); }
__host__ __device__ constexpr int blk_of(int K) { return 2 * lr_of(K) + NPREP * 32; }  // [EFB|PREP]
__host__ __device__ constexpr int o_l2(int K) { return blk_of(K); }
__host__ __device__ constexpr int o_u2(int K) { return blk_of(K) + lr_of(K); }
__host__ __device__ constexpr int o_l3(int K) { return blk_of(K) + 2 * lr_of(K); }
__host__ __device__ constexpr int o_u3(int K) { return blk_of(K) + 3 * lr_of(K); }
__host__ __device__ constexpr int recd_of(int K) { return blk_of(K) + 4 * lr_of(K); }
// ring stage: [block | S0: in-plane coupling | S1: C1 | S2: C2 | X: b' or xo | S4: second in-plane coupling (twist line)]
__host__ __device__ constexpr int rs0_of(int K) { return blk_of(K); }
__host__ __device__ constexpr int rs1_of(int K) { return blk_of(K) + lr_of(K); }
__host__ __device__ constexpr int rs2_of(int K) { return blk_of(K) + 2 * lr_of(K); }
__host__ __device__ constexpr int rx_of(int K) { return blk_of(K) + 3 * lr_of(K); }
__host__ __device__ constexpr int rs4_of(int K) { return blk_of(K) + 4 * lr_of(K); }
__host__ __device__ constexpr int stage_of(int K) { return blk_of(K) + 5 * lr_of(K); }

constexpr int SMEM_MAX = 232448 - 1024;
__host__ __device__ constexpr int clamp8(int d) { return d > 8 ? 8 : d; }
// static shared memory: the twist exchange (2 parities x 2 warps x LR per pair) + barriers
__host__ __device__ constexpr int static_smem_of(int K, int NP) { return NP * 4 * lr_of(K) * 8 + 2 * NP * 2 * 8 * 8; }
// ring depth of the one-CTA kernel (4 solver warps) and the split kernel (2)
__host__ __device__ constexpr int depth_of(int K) { return clamp8((SMEM_MAX - static_smem_of(K, 2)) / (4 * stage_of(K) * 8)); }
__host__ __device__ constexpr int depth2_of(int K) { return clamp8((SMEM_MAX - static_smem_of(K, 1)) / (2 * stage_of(K) * 8)); }
// split kernel with plane buffers sized for ny <= 32K+1 (a half-plane of 16K+1 lines per solver warp); < 2: none
__host__ __device__ constexpr int depth_smb_of(int K)
{
    return clamp8((SMEM_MAX - static_smem_of(K, 1) - 2 * (16 * K + 1) * lr_of(K) * 8) / (2 * stage_of(K) * 8));
}

__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
__device__ __forceinline__ void mbar_arrive(void *bar)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// element of cell c inside its TS record / cell of element r (-1: padding)
__host__ __device__ __forceinline__ int ts_index(int c, int K) { return (c % K) * 32 + c / K; }
__host__ __device__ __forceinline__ int ts_cell(int r, int nx, int K)
{
    const int c = (r & 31) * K + (r >> 5);
    return c < nx ? c : -1;
}

// b (B, N) -> b' = b mu in TS (B, N_TS).  One thread per TS element.
static __global__ void k_to_ts(const double *__restrict__ src, const double *__restrict__ mu, double *__restrict__ dst,
                               int nx, i64 lines, int K, i64 batch)
{
    const int LR = lr_of(K);
    const i64 total = lines * LR * batch;
    for (i64 e = blockIdx.x * (i64)blockDim.x + threadIdx.x; e < total; e += (i64)gridDim.x * blockDim.x) {
        const i64 line = e / LR;  // global line over the batch
        const int c = ts_cell((int)(e - line * LR), nx, K);
        dst[e] = c >= 0 ? src[line * nx + c] * mu[e] : 0.0;
    }
}

// x in TS -> natural; systems masked off by `active` get x = 0
static __global__ void k_from_ts(const double *__restrict__ src, double *__restrict__ dst, int nx, i64 lines, int K,
                                 i64 batch, const int32_t *__restrict__ active)
{
    const int LR = lr_of(K);
    const i64 total = lines * nx * batch;
    for (i64 e = blockIdx.x * (i64)blockDim.x + threadIdx.x; e < total; e += (i64)gridDim.x * blockDim.x) {
        const i64 line = e / nx;
        const int c = (int)(e - line * nx);
        const bool on = !active || active[line / lines];
        dst[e] = on ? src[line * LR + ts_index(c, K)] : 0.0;
    }
}

// Solve records from a factor (B,7,N); one thread per line, three passes
// along the line (the record's own slots hold the intermediate pivots).
//   T of the line (ntd_solve.py:107-131): sub-diagonal l1, super-diagonal u1,
//   twisted pivots 1/m with the twist at t = (nx-1)/2; its diagonal follows
//   from the pivot recurrences (ntd_factor.py:86-110).
//   pass 1 (ascending):  d, forward pivots delta (= 1/m left of the twist)
//   pass 2 (descending): backward pivots gamma (= 1/m right of it), nu = delta + gamma - d, eB
//   pass 3 (ascending):  mu = 1/nu, eF, couplings c mu
// The record and mu buffers are zero-filled before (padding elements).
static __global__ void k_solve_ts(const double *__restrict__ pre, double *__restrict__ solve, double *__restrict__ mu_out,
                                  int nx, i64 lines, int K, i64 batch)
{
    const int LR = lr_of(K), RECD = recd_of(K);
    const i64 n = lines * nx;
    const i64 gl = blockIdx.x * (i64)blockDim.x + threadIdx.x;  // global line
    if (gl >= lines * batch) return;
    const i64 s = gl / lines, line = gl - s * lines;
    const double *p = pre + s * 7 * n + line * nx;
    const double *l1 = p, *u1 = p + n, *l2 = p + 2 * n, *u2 = p + 3 * n, *l3 = p + 4 * n, *u3 = p + 5 * n, *mr = p + 6 * n;
    double *rec = solve + gl * (i64)RECD;
    double *mu = mu_out + gl * (i64)LR;
    const int t = (nx - 1) / 2;
    double *DE = rec + o_l2(K), *DD = rec + o_u2(K), *NU = rec + o_l3(K), *GA = rec + o_u3(K);  // scratch
    // pass 1
    double dprev = 0.0;
    for (int c = 0; c < nx; c++) {
        const double M = 1.0 / mr[c];
        double d = M;
        if (c <= t && c > 0) d += (l1[c] * u1[c - 1]) * mr[c - 1];
        if (c >= t && c < nx - 1) d += (u1[c] * l1[c + 1]) * mr[c + 1];
        double de = M;
        if (c >= t) de = c > 0 ? d - (l1[c] * u1[c - 1]) / dprev : d;
        const int e = ts_index(c, K);
        DD[e] = d;
        DE[e] = de;
        dprev = de;
    }
    // pass 2
    double gnext = 0.0, nunext = 0.0;
    for (int c = nx - 1; c >= 0; c--) {
        const int e = ts_index(c, K);
        const double d = DD[e];
        double ga = 1.0 / mr[c];
        if (c <= t) ga = c < nx - 1 ? d - (u1[c] * l1[c + 1]) / gnext : d;
        const double nu = c == t ? 1.0 / mr[c] : (DE[e] + ga) - d;
        rec[o_efb(K) + 2 * e + 1] = c < nx - 1 ? -(u1[c] * nunext) / (gnext * nu) : 0.0;
        NU[e] = nu;
        GA[e] = ga;
        gnext = ga;
        nunext = nu;
    }
    // pass 3
    double deprev = 0.0, nuprev = 0.0;
    for (int c = 0; c < nx; c++) {
        const int e = ts_index(c, K);
        const double nu = NU[e], de = DE[e];
        const double m = c == t ? mr[c] : 1.0 / nu;
        rec[o_efb(K) + 2 * e] = c > 0 ? -(l1[c] * nuprev) / (deprev * nu) : 0.0;
        mu[e] = m;
        rec[o_l2(K) + e] = l2[c] * m;
        rec[o_u2(K) + e] = u2[c] * m;
        rec[o_l3(K) + e] = l3[c] * m;
        rec[o_u3(K) + e] = u3[c] * m;
        deprev = de;
        nuprev = nu;
    }
}

// ---------------------------------------------------------------- data
struct TsArrays {  // one system, TS
    const double *solve;  // record-major solve records [line][recd_of(K)]
    const double *b;      // b' = b mu
    double *x, *xs;
    const double *zero;   // one plane of zero records: the missing level-3 neighbour
};

template <int K>
__device__ __forceinline__ void ld_rec(const double *rec, int lane, double (&v)[K])
{
#pragma unroll
    for (int k = 0; k < K; k++) v[k] = rec[k * 32 + lane];
}
template <int K>
__device__ __forceinline__ void st_rec(double *rec, int lane, const double (&v)[K])
{
#pragma unroll
    for (int k = 0; k < K; k++) rec[k * 32 + lane] = v[k];
}

// ring of D stages per solver warp
template <int K, int D>
struct Ring {
    double *base;
    unsigned long long *full, *empty;
    __device__ __forceinline__ double *stage(unsigned st) const { return base + (size_t)st * stage_of(K); }
};

struct PlaneDesc {
    bool nbuf;   // SMB: the level-3 neighbour y1 is the plane this warp processed last (in its smem buffer)
    i64 prec;    // record index of the plane's first line (plane * ny)
    int mode;    // M_LOWER3 / M_UPPER3
    int c1;      // record offset of the level-3 coupling C1 (two: L3 then U3 = C2)
    bool two;    // both level-3 neighbours (twist plane)
    bool hasM, hasP, nbrUp;
    bool up;     // lower sweep: the level-3 neighbour is plane p+1 (descending half)
};

struct Seq {
    int cnt, t2, ny, w2;
    __device__ __forceinline__ int qlow(int i) const { return w2 == 0 ? i : ny - 1 - i; }
    __device__ __forceinline__ int qup(int i) const { return w2 == 0 ? t2 - 1 - i : t2 + 1 + i; }
    // line of record k of a plane: lower sweep, twist line, upper sweep
    __device__ __forceinline__ int qrec(int k) const { return k < cnt ? qlow(k) : k == cnt ? t2 : qup(k - cnt - 1); }
};

// scan coefficients of every line (setup): one warp per line
template <int K>
__global__ void k_prep_ts(double *__restrict__ solve, i64 lines_total)
{
    const int lane = threadIdx.x & 31;
    const i64 line = (blockIdx.x * (i64)blockDim.x + threadIdx.x) >> 5;
    if (line >= lines_total) return;
    double *rec = solve + line * (i64)recd_of(K);
    double eF[K], eB[K];
#pragma unroll
    for (int k = 0; k < K; k++) {
        eF[k] = rec[o_efb(K) + 2 * (k * 32 + lane)];
        eB[k] = rec[o_efb(K) + 2 * (k * 32 + lane) + 1];
    }
    const PrepTS P = line_prep<K>(lane, eF, eB);
    double *pp = rec + o_prep(K);
    const double v[NPREP] = {P.p2, P.p3, P.s1, P.s2, P.s3, P.e1, P.q2, P.q3, P.t1, P.t2, P.t3, P.f1};
#pragma unroll
    for (int c = 0; c < NPREP; c++) pp[(c >> 1) * 64 + 2 * lane + (c & 1)] = v[c];
}

// ---------------- producer: bulk copies of what each line step reads
//   lower sweep:  block, in-plane coupling (L2' / U2' by half), C1 (+C2), b' (LOWER3)
//   twist line:   block, L2', U2', C1 (+C2), b' (LOWER3) / xo (UPPER3)
//   upper sweep:  block, in-plane coupling (U2' / L2'), xo (UPPER3)
__device__ __forceinline__ void mbar_wait_producer(void *bar, unsigned parity)
{
    unsigned ok = 0;
    const unsigned a = smem_u32(bar);
    while (!ok) {
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3; selp.u32 %0, 1, 0, p; }"
            : "=r"(ok)
            : "r"(a), "r"(parity), "r"(1000000u)
            : "memory");
    }
}

template <int K>
__device__ __forceinline__ void rec_copy(const TsArrays &S, const PlaneDesc &P, const Seq &Q, int k, double *dst,
                                         unsigned long long *bar)
{
    constexpr int LR = lr_of(K);
    constexpr unsigned lb = LR * 8u, bb = blk_of(K) * 8u;
    const bool lower3 = P.mode == M_LOWER3;
    const int ph = k < Q.cnt ? 0 : k == Q.cnt ? 1 : 2;
    const i64 line = P.prec + Q.qrec(k);
    const double *src = S.solve + line * (i64)recd_of(K);
    const int cpl = ph == 1 ? o_l2(K) : ((ph == 0) == (Q.w2 == 0) ? o_l2(K) : o_u2(K));
    const unsigned nc = ph < 2 ? (P.two ? 2u : 1u) : 0u;
    const bool extra = ph == 0 ? lower3 : ph == 1 ? true : !lower3;
    const double *xsrc = (lower3 ? S.b : S.x) + line * (i64)LR;
    mbar_expect_tx(bar, bb + lb + nc * lb + (extra ? lb : 0u) + (ph == 1 ? lb : 0u));
    tma_load_1d(dst, src, bb, bar);
    tma_load_1d(dst + rs0_of(K), src + cpl, lb, bar);
    if (nc) tma_load_1d(dst + rs1_of(K), src + P.c1, nc * lb, bar);
    if (extra) tma_load_1d(dst + rx_of(K), xsrc, lb, bar);
    if (ph == 1) tma_load_1d(dst + rs4_of(K), src + o_u2(K), lb, bar);
}

template <int K, int D>
__device__ void produce_plane(const TsArrays &S, const PlaneDesc &P, const Seq &Q, const Ring<K, D> &R, unsigned &rec)
{
    const int lane = threadIdx.x & 31;
    const int n = 2 * Q.cnt + 1;
    if (lane == 0) {
        for (int k = 0; k < n; k++, rec++) {
            const unsigned st = rec % D;
            if (rec >= (unsigned)D) mbar_wait_producer(&R.empty[st], ((rec / D) + 1) & 1);
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            rec_copy<K>(S, P, Q, k, R.stage(st), &R.full[st]);
        }
    } else {
        rec += n;
    }
    __syncwarp();
}

__device__ __forceinline__ bool mbar_test(void *bar, unsigned parity)
{
    unsigned ok;
    asm volatile("{ .reg .pred p; mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(ok)
                 : "r"(smem_u32(bar)), "r"(parity)
                 : "memory");
    return ok != 0;
}

// Ring operands of one line step.  ld_* only issues the shared-memory loads;
// the x-independent constants are formed after the current line's solve.
template <int K>
struct Ops {
    double eF[K], eB[K], cp[K], pt[K];
    double pr[NPREP];  // p2 p3 s1 s2 s3 e1 q2 q3 t1 t2 t3 f1
};

template <int K>
__device__ __forceinline__ void ld_common(Ops<K> &o, const double *sg, int lane)
{
    const double2 *efb = reinterpret_cast<const double2 *>(sg + o_efb(K));
#pragma unroll
    for (int k = 0; k < K; k++) {
        const double2 v = efb[k * 32 + lane];
        o.eF[k] = v.x;
        o.eB[k] = v.y;
    }
    const double2 *pp = reinterpret_cast<const double2 *>(sg + o_prep(K));
#pragma unroll
    for (int c = 0; c < NPREP / 2; c++) {
        const double2 v = pp[c * 32 + lane];
        o.pr[2 * c] = v.x;
        o.pr[2 * c + 1] = v.y;
    }
    ld_rec(sg + rs0_of(K), lane, o.cp);
}

// One line: x = T^{-1} r for rho = mu r (SUB: x = y - T^{-1} r, y passed in x).
template <int K, bool SUB>
__device__ __forceinline__ void solve_line(const Ops<K> &o, int l, const double (&rho)[K], double (&x)[K])
{
    double pf[K], pb[K], pa[K], qa[K];
    pf[0] = rho[0];
    pa[0] = o.eF[0];
    pb[K - 1] = rho[K - 1];
    qa[K - 1] = o.eB[K - 1];
#pragma unroll
    for (int k = 1; k < K; k++) {
        pf[k] = fma(o.eF[k], pf[k - 1], rho[k]);
        pa[k] = o.eF[k] * pa[k - 1];
        pb[K - 1 - k] = fma(o.eB[K - 1 - k], pb[K - k], rho[K - 1 - k]);
        qa[K - 1 - k] = o.eB[K - 1 - k] * qa[K - k];
    }
    const double p1 = l >= 1 ? pa[K - 1] : 0.0, q1 = l <= 30 ? qa[0] : 0.0;
    const double C0 = pf[K - 1], D0 = pb[0];
    // level 1 (windows of 4 lanes)
    const double c3 = up(C0, 3), d3 = dn(D0, 3), c2 = up(C0, 2), d2 = dn(D0, 2), c1 = up(C0, 1), d1 = dn(D0, 1);
    const double C1 = fma(p1, c1, C0) + fma(o.pr[0], c2, o.pr[1] * c3);
    const double D1 = fma(q1, d1, D0) + fma(o.pr[6], d2, o.pr[7] * d3);
    // level 2 (windows of 16 lanes)
    const double c12 = up(C1, 12), d12 = dn(D1, 12), c8 = up(C1, 8), d8 = dn(D1, 8), c4 = up(C1, 4), d4 = dn(D1, 4);
    const double C2 = fma(o.pr[2], c4, C1) + fma(o.pr[3], c8, o.pr[4] * c12);
    const double D2 = fma(o.pr[8], d4, D1) + fma(o.pr[9], d8, o.pr[10] * d12);
    // level 3: exclusive carries
    const double u17 = up(C2, 17), v17 = dn(D2, 17), u1 = up(C2, 1), v1 = dn(D2, 1);
    const double cF = fma(o.pr[5], u17, l >= 1 ? u1 : 0.0);
    const double cB = fma(o.pr[11], v17, l <= 30 ? v1 : 0.0);
#pragma unroll
    for (int k = 0; k < K; k++) {
        const double R = k < K - 1 ? fma(o.eB[k], pb[k + 1 < K ? k + 1 : k], pf[k]) : pf[k];
        if (SUB)
            x[k] = fma(-pa[k], cF, fma(-qa[k], cB, x[k] - R));
        else
            x[k] = fma(pa[k], cF, fma(qa[k], cB, R));
    }
}

// ---------------- solver: one plane
// SMB: the warp keeps its half of the plane it processed last in shared
// memory (pbuf, lines lo_line.. of the half incl. the twist line): each line
// slot holds the neighbour plane's final x until this plane's lower sweep
// replaces it with the lower-sweep value, which the upper sweep replaces with
// this plane's final x.  The solver then issues no global loads per line.
template <int K, int D, int MODE, bool TWO, bool SMB>
__device__ void solve_plane(const TsArrays &S, const PlaneDesc &P, const Seq &Q, int bar_id, double *ex, int &parity,
                            const Ring<K, D> &R, unsigned &rec, double *pbuf)
{
    constexpr int LR = lr_of(K);
    const int lane = threadIdx.x & 31, w2 = Q.w2;
    const int ny = Q.ny, t2 = Q.t2, cnt = Q.cnt;
    const i64 plr = (i64)ny * LR;  // plane stride in TS
    constexpr bool lower3 = MODE == M_LOWER3;
    constexpr bool PIPE = K <= 5;
    // Plane bases (line q of a plane at base + q*LR).  A missing level-3
    // neighbour (first/last plane) has an exactly-zero coupling; it reads the
    // zero plane instead of branching.
    double *xpl = S.x + P.prec * LR;
    const double *y1, *y2 = S.zero;
    if (lower3) {
        if (TWO) {
            y1 = P.hasM ? xpl - plr : S.zero;
            y2 = P.hasP ? xpl + plr : S.zero;
        } else if (P.up) {
            y1 = P.hasP ? xpl + plr : S.zero;
        } else {
            y1 = P.hasM ? xpl - plr : S.zero;
        }
    } else {
        y1 = P.nbrUp ? xpl + plr : xpl - plr;
    }
    double *xlow = (lower3 ? S.x : S.xs) + P.prec * LR;  // lower-sweep store of this plane
    if constexpr (SMB) {
        double *bq = pbuf - (i64)(w2 == 0 ? 0 : t2) * LR;  // line q of this half at bq + q*LR
        xlow = bq;
        if (P.nbuf) y1 = bq;
    }
    auto full = [&](unsigned r) { return &R.full[r % D]; };
    auto par = [&](unsigned r) { return (r / D) & 1u; };
    // raw operands of a lower-sweep line, and its x-independent constants
    //   LOWER3: pt = b' - C1' y1 (- C2' y2);  UPPER3: pt = C1' y1
    struct Raw {
        double bx[K], c1[K], c2[K], n1[K], n2[K];
    };
    auto ld_lower = [&](Ops<K> &o, Raw &w, const double *sg, int q) {
        ld_common(o, sg, lane);
        if (lower3) ld_rec(sg + rx_of(K), lane, w.bx);
        ld_rec(sg + rs1_of(K), lane, w.c1);
        ld_rec(y1 + q * LR, lane, w.n1);
        if (TWO) {
            ld_rec(sg + rs2_of(K), lane, w.c2);
            ld_rec(y2 + q * LR, lane, w.n2);
        }
    };
    auto fin_lower = [&](Ops<K> &o, const Raw &w) {
#pragma unroll
        for (int k = 0; k < K; k++) {
            double v = lower3 ? fma(-w.c1[k], w.n1[k], w.bx[k]) : w.c1[k] * w.n1[k];
            if (TWO) v = fma(-w.c2[k], w.n2[k], v);
            o.pt[k] = v;
        }
    };
    double xprev[K];
#pragma unroll
    for (int k = 0; k < K; k++) xprev[k] = 0.0;
    // ---------------- level-2 lower sweep (ntd_solve.py:147-171)
    // Software-pipelined (PIPE): the operands of line i+1 are loaded while
    // line i solves, so the serial chain per line is rho = pt - cp' xprev and
    // the scans.  The full barrier of record i+2 is tested at the top of step
    // i and the result consumed after the solve.
    Ops<K> cur;
    if (PIPE && cnt > 0) {
        Raw w;
        mbar_wait(full(rec), par(rec));
        ld_lower(cur, w, R.stage(rec % D), Q.qlow(0));
        fin_lower(cur, w);
        if (cnt > 1) mbar_wait(full(rec + 1), par(rec + 1));
    }
#pragma unroll 2  // ping-pong registers: no copies of in-flight loads
    for (int i = 0; i < cnt; i++, rec++) {
        const unsigned st = rec % D;
        Ops<K> nxo;
        Raw w;
        bool ok2 = true;
        if (PIPE) {
            if (i + 2 < cnt) ok2 = mbar_test(full(rec + 2), par(rec + 2));
            ld_lower(nxo, w, R.stage((rec + 1) % D), Q.qlow(i + 1 < cnt ? i + 1 : i));  // unused past the sweep
        } else {
            mbar_wait(full(rec), par(rec));
            ld_lower(cur, w, R.stage(st), Q.qlow(i));
            fin_lower(cur, w);
        }
        double rho[K], x[K];
#pragma unroll
        for (int k = 0; k < K; k++) rho[k] = fma(-cur.cp[k], xprev[k], cur.pt[k]);  // line 0: xprev = 0
        solve_line<K, false>(cur, lane, rho, x);
        mbar_arrive(&R.empty[st]);  // every operand of stage st has been consumed
        st_rec(xlow + Q.qlow(i) * LR, lane, x);
#pragma unroll
        for (int k = 0; k < K; k++) xprev[k] = x[k];
        if (PIPE) {
            fin_lower(nxo, w);
            if (i + 2 < cnt && !ok2) mbar_wait(full(rec + 2), par(rec + 2));
            cur = nxo;
        }
    }
    // ---------------- exchange the lines next to the twist
    double *mine = ex + (parity * 2 + w2) * LR;
    const double *other = ex + (parity * 2 + (1 - w2)) * LR;
    st_rec(mine, lane, xprev);
    named_bar(bar_id, 64);
    parity ^= 1;
    double xo_[K];
    ld_rec(other, lane, xo_);
    // ---------------- twist line (ntd_solve.py:172-177): its record follows the lower-sweep records
    double xn[K];
    {
        Ops<K> tw;
        Raw w;
        double u2c[K], xo[K];
        const unsigned st = rec % D;
        const double *sg = R.stage(st);
        mbar_wait(full(rec), par(rec));
        ld_lower(tw, w, sg, t2);
        ld_rec(sg + rs4_of(K), lane, u2c);
        if (!lower3) ld_rec(sg + rx_of(K), lane, xo);
        fin_lower(tw, w);
        double rho[K];
#pragma unroll
        for (int k = 0; k < K; k++) {
            const double xa = w2 == 0 ? xprev[k] : xo_[k], xd = w2 == 0 ? xo_[k] : xprev[k];
            double v = tw.pt[k];
            if (t2 > 0) v = fma(-tw.cp[k], xa, v);
            if (t2 < ny - 1) v = fma(-u2c[k], xd, v);
            rho[k] = v;
        }
        solve_line<K, false>(tw, lane, rho, xn);
        double nv[K];
#pragma unroll
        for (int k = 0; k < K; k++) nv[k] = lower3 ? xn[k] : xo[k] - xn[k];  // UPPER3: final = xo - value
        mbar_arrive(&R.empty[st]);
        rec++;
        if (w2 == 0) st_rec(xpl + t2 * LR, lane, nv);
        if constexpr (SMB) st_rec(xlow + t2 * LR, lane, nv);  // both warps keep the twist line
    }
    // ---------------- level-2 upper sweep (ntd_solve.py:178-185)
    //   value_q = y_q - T_q^{-1}(cp' value_prev);  LOWER3: x_q = value_q;  UPPER3: x_q = xo_q - value_q
    auto ld_upper = [&](Ops<K> &o, double (&y)[K], double (&xo)[K], const double *sg, int q) {
        ld_common(o, sg, lane);
        ld_rec(xlow + q * LR, lane, y);
        if (!lower3) ld_rec(sg + rx_of(K), lane, xo);
    };
    double ycur[K], xocur[K];
    if (PIPE && cnt > 0) {
        mbar_wait(full(rec), par(rec));
        ld_upper(cur, ycur, xocur, R.stage(rec % D), Q.qup(0));
        if (cnt > 1) mbar_wait(full(rec + 1), par(rec + 1));
    }
#pragma unroll 2
    for (int i = 0; i < cnt; i++, rec++) {
        const unsigned st = rec % D;
        Ops<K> nxo;
        double ynx[K], xonx[K];
        bool ok2 = true;
        if (PIPE) {
            if (i + 2 < cnt) ok2 = mbar_test(full(rec + 2), par(rec + 2));
            ld_upper(nxo, ynx, xonx, R.stage((rec + 1) % D), Q.qup(i + 1 < cnt ? i + 1 : i));
        } else {
            mbar_wait(full(rec), par(rec));
            ld_upper(cur, ycur, xocur, R.stage(st), Q.qup(i));
        }
        double rho[K];
#pragma unroll
        for (int k = 0; k < K; k++) rho[k] = cur.cp[k] * xn[k];
#pragma unroll
        for (int k = 0; k < K; k++) xn[k] = ycur[k];
        solve_line<K, true>(cur, lane, rho, xn);
        double nv[K];
#pragma unroll
        for (int k = 0; k < K; k++) nv[k] = lower3 ? xn[k] : xocur[k] - xn[k];
        mbar_arrive(&R.empty[st]);
        st_rec(xpl + Q.qup(i) * LR, lane, nv);
        if constexpr (SMB) st_rec(xlow + Q.qup(i) * LR, lane, nv);  // (xlow is the buffer)
        if (PIPE) {
            if (i + 2 < cnt && !ok2) mbar_wait(full(rec + 2), par(rec + 2));
            cur = nxo;
#pragma unroll
            for (int k = 0; k < K; k++) {
                ycur[k] = ynx[k];
                xocur[k] = xonx[k];
            }
        }
    }
}

__device__ __forceinline__ void cluster_sync_all()
{
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// NP = 2: one CTA per system, both level-3 halves (warp pairs) on one SM.
// NP = 1: a cluster of two CTAs per system, one level-3 half each on its own
// SM (solver and producer warps then each have an SM sub-partition to
// themselves); the level-3 phase boundaries are cluster barriers.
// SMB (split kernel only): each solver warp keeps its half of the last
// processed plane in shared memory after the ring (solve_plane).
template <int K, int D, int NP, bool SMB = false>
__global__ void __launch_bounds__(128 * NP, 1) k_apply(const double *__restrict__ solve, const double *__restrict__ bsl,
                                                       double *xsl, double *xssl, const double *__restrict__ zpl,
                                                       int nx, int ny, int nz, const int32_t *__restrict__ active)
{
    extern __shared__ __align__(128) double ts_ring[];
    __shared__ __align__(16) double ex[NP][2 * 2 * lr_of(K)];
    __shared__ __align__(8) unsigned long long bars[2 * NP][2 * D];
    constexpr int LR = lr_of(K);
    const i64 sys = NP == 2 ? blockIdx.x : blockIdx.x >> 1;
    if (active && !active[sys]) return;  // both CTAs of a cluster leave together
    const i64 nsl = (i64)nz * ny * LR;
    TsArrays S;
    S.solve = solve + sys * (i64)nz * ny * recd_of(K);
    S.b = bsl + sys * nsl;
    S.x = xsl + sys * nsl;
    S.xs = xssl + sys * nsl;
    S.zero = zpl;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const bool producer = warp >= 2 * NP;
    const int sw = warp & (2 * NP - 1);  // solver warp this warp is (or feeds)
    const int pair = NP == 2 ? sw >> 1 : (int)(blockIdx.x & 1), w2 = sw & 1, bar = NP == 2 ? 1 + pair : 1;
    Ring<K, D> R;
    R.base = ts_ring + (size_t)sw * D * stage_of(K);
    // SMB plane buffer of this solver warp: max(t2+1, ny-t2) lines
    const int bl = (ny - 1) / 2 + 1 > ny - (ny - 1) / 2 ? (ny - 1) / 2 + 1 : ny - (ny - 1) / 2;
    double *pbuf = ts_ring + (size_t)2 * NP * D * stage_of(K) + (size_t)sw * bl * LR;
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
    auto phase_sync = [&]() {
        if constexpr (NP == 2)
            __syncthreads();
        else
            cluster_sync_all();
    };
    Seq Q;
    Q.ny = ny;
    Q.t2 = (ny - 1) / 2;
    Q.w2 = w2;
    Q.cnt = w2 == 0 ? Q.t2 : (ny - 1 - Q.t2);
    unsigned rec = 0;
    double *myex = ex[NP == 2 ? pair : 0];
    int parity = 0;
    const int t3 = (nz - 1) / 2;
    // The warp pair's plane schedule: level-3 lower sweep (ntd_solve.py:198-221),
    // the twist plane for pair 0 (222-232), level-3 upper sweep (233-253).
    const int nlow = pair == 0 ? t3 : nz - 1 - t3;
    const int ntw = pair == 0 ? 1 : 0;
    auto desc = [&](int idx) {
        PlaneDesc P;
        // the neighbour is the plane this pair processed last, except for
        // each sweep's first plane (none / another pair's) and the twist
        // plane's upper neighbour (y2, pair 1's)
        P.nbuf = idx > 0 && !(pair == 1 && idx == nlow);
        P.two = false;
        P.hasM = P.hasP = P.nbrUp = P.up = false;
        if (idx < nlow) {
            const int p = pair == 0 ? idx : nz - 1 - idx;
            P.prec = (i64)p * ny;
            P.mode = M_LOWER3;
            P.hasM = pair == 0 && p > 0;
            P.hasP = pair == 1 && p < nz - 1;
            P.up = pair == 1;
            P.c1 = P.up ? o_u3(K) : o_l3(K);
        } else if (idx < nlow + ntw) {
            P.prec = (i64)t3 * ny;
            P.mode = M_LOWER3;
            P.two = true;
            P.hasM = t3 > 0;
            P.hasP = t3 < nz - 1;
            P.c1 = o_l3(K);  // L3 then U3 (contiguous)
        } else {
            const int u = idx - nlow - ntw;
            const int p = pair == 0 ? t3 - 1 - u : t3 + 1 + u;
            P.prec = (i64)p * ny;
            P.mode = M_UPPER3;
            P.nbrUp = pair == 0;
            P.c1 = P.nbrUp ? o_u3(K) : o_l3(K);
        }
        return P;
    };
    const int nplanes = 2 * nlow + ntw;
    for (int i = 0; i < nlow; i++) {
        if (producer)
            produce_plane<K, D>(S, desc(i), Q, R, rec);
        else
            solve_plane<K, D, M_LOWER3, false, SMB>(S, desc(i), Q, bar, myex, parity, R, rec, pbuf);
    }
    phase_sync();
    if (pair == 0) {
        if (producer) {
            fence_proxy_async();
            produce_plane<K, D>(S, desc(nlow), Q, R, rec);
        } else {
            solve_plane<K, D, M_LOWER3, true, SMB>(S, desc(nlow), Q, bar, myex, parity, R, rec, pbuf);
        }
    }
    phase_sync();
    if (producer) fence_proxy_async();  // x (read as xo) was written by generic stores
    for (int i = nlow + ntw; i < nplanes; i++) {
        if (producer)
            produce_plane<K, D>(S, desc(i), Q, R, rec);
        else
            solve_plane<K, D, M_UPPER3, false, SMB>(S, desc(i), Q, bar, myex, parity, R, rec, pbuf);
    }
}

}  // namespace ts

template <int K>
int launch_prep_ts_k(double *solve, i64 lines_total, cudaStream_t st);
template <int K>
int launch_apply_ts_k(const double *solve, const double *bsl, double *xsl, double *xssl, const double *zpl, int nx,
                      int ny, int nz, i64 batch, const int32_t *active, cudaStream_t st, int ctas_per_system = 1);

template <int K, int D, bool SMB>
int launch_apply_ts_cluster(const double *solve, const double *bsl, double *xsl, double *xssl, const double *zpl,
                            int nx, int ny, int nz, i64 batch, const int32_t *active, cudaStream_t st, int bl)
{
    const size_t smem = (size_t)2 * D * ts::stage_of(K) * 8 + (SMB ? (size_t)2 * bl * ts::lr_of(K) * 8 : 0);
    cudaError_t e = cudaFuncSetAttribute(ts::k_apply<K, D, 1, SMB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) {
        ntd::set_error("ntd_apply smem", e);
        return NTD_ELAUNCH;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(2 * batch));
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, ts::k_apply<K, D, 1, SMB>, solve, bsl, xsl, xssl, zpl, nx, ny, nz, active);
    if (e != cudaSuccess) {
        ntd::set_error("ntd_apply (cluster)", e);
        return NTD_ELAUNCH;
    }
    return ntd::check_launch("ntd_apply");
}

#define NTD_INSTANTIATE_TS(K)                                                                                     \
    template <>                                                                                                    \
    int launch_prep_ts_k<K>(double *solve, i64 lines_total, cudaStream_t st)                                      \
    {                                                                                                              \
        const i64 threads = lines_total * 32;                                                                      \
        ts::k_prep_ts<K><<<(unsigned)((threads + 255) / 256), 256, 0, st>>>(solve, lines_total);                  \
        return ntd::check_launch("ntd_solve_bands prep");                                                          \
    }                                                                                                              \
    template <>                                                                                                    \
    int launch_apply_ts_k<K>(const double *solve, const double *bsl, double *xsl, double *xssl, const double *zpl,   \
                             int nx, int ny, int nz, i64 batch, const int32_t *active, cudaStream_t st,            \
                             int ctas_per_system)                                                                  \
    {                                                                                                              \
        const int bl_ = (ny - 1) / 2 + 1 > ny - (ny - 1) / 2 ? (ny - 1) / 2 + 1 : ny - (ny - 1) / 2;             \
        if (ctas_per_system == 2) {                                                                                \
            if constexpr (ts::depth_smb_of(K) >= 2) {                                                              \
                if (bl_ <= 16 * K + 1)                                                                             \
                    return launch_apply_ts_cluster<K, ts::depth_smb_of(K), true>(solve, bsl, xsl, xssl, zpl, nx,   \
                                                                                 ny, nz, batch, active, st, bl_);  \
            }                                                                                                      \
            return launch_apply_ts_cluster<K, ts::depth2_of(K), false>(solve, bsl, xsl, xssl, zpl, nx, ny, nz,     \
                                                                       batch, active, st, bl_);                    \
        }                                                                                                          \
        constexpr int D = ts::depth_of(K);                                                                         \
        const size_t smem = (size_t)4 * D * ts::stage_of(K) * 8;                                                   \
        cudaError_t e = cudaFuncSetAttribute(ts::k_apply<K, D, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,    \
                                             (int)smem);                                                           \
        if (e != cudaSuccess) {                                                                                    \
            ntd::set_error("ntd_apply smem", e);                                                                   \
            return NTD_ELAUNCH;                                                                                    \
        }                                                                                                          \
        ts::k_apply<K, D, 2><<<(unsigned)batch, 256, smem, st>>>(solve, bsl, xsl, xssl, zpl, nx, ny, nz, active);  \
        return ntd::check_launch("ntd_apply");                                                                     \
    }
