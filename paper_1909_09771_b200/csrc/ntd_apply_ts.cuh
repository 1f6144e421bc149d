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
//   [ L3' | L2' | EFB (eF, eB pairs, 2 LR) | PREP (NPREP x 32, pairs) | U2' | U3' ]
// eF / eB are the scaled elimination multipliers of the two-sided solve,
// PREP the factor-only scan coefficients, and the couplings are pre-multiplied
// by mu (the twisted pivot reciprocal at the cell): c' = c mu, as is the
// right-hand side on entry (b' = b mu).  The mu of every cell follows the
// records ([system][line][LR]) for the kernels that form b'.
#pragma once
#include "ntd_kernels.cuh"
#include "ntd_line_ts.cuh"
#include <type_traits>

namespace ts {

constexpr int NPREP = 8;  // stored PrepTS coefficients per lane (m2 m4 m8 e, n2 n4 n8 f); m1 and n1 are rebuilt
__host__ __device__ constexpr int lr_of(int K) { return 32 * K; }
// record: [ L3' | L2' | EFB | PREP | U2' | U3' ] -- whatever a line step reads is one contiguous range
// (the in-plane couplings sit next to the block: an upper-sweep step copies nothing it does not read)
__host__ __device__ constexpr int o_l3(int K) { return 0; }
__host__ __device__ constexpr int o_l2(int K) { return lr_of(K); }
__host__ __device__ constexpr int o_efb(int K) { return 2 * lr_of(K); }
__host__ __device__ constexpr int o_prep(int K) { return 4 * lr_of(K); }
__host__ __device__ constexpr int o_u2(int K) { return 4 * lr_of(K) + NPREP * 32; }
__host__ __device__ constexpr int o_u3(int K) { return 5 * lr_of(K) + NPREP * 32; }
__host__ __device__ constexpr int recd_of(int K) { return 6 * lr_of(K) + NPREP * 32; }
// ring stage: [ record | X: b' or xo ]
__host__ __device__ constexpr int rx_of(int K) { return recd_of(K); }
__host__ __device__ constexpr int stage_of(int K) { return recd_of(K) + lr_of(K); }

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
    return clamp8((SMEM_MAX - static_smem_of(K, 1) - (2 * (16 * K + 1) + 1) * lr_of(K) * 8) / (2 * stage_of(K) * 8));
}

__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
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
    const double v[NPREP] = {P.m2, P.m4, P.m8, P.e, P.n2, P.n4, P.n8, P.f};
#pragma unroll
    for (int c = 0; c < NPREP; c++) pp[(c >> 1) * 64 + 2 * lane + (c & 1)] = v[c];
}

// ---------------- producer: bulk copies of what each line step reads
//   lower sweep:  block, in-plane coupling (L2' / U2' by half), C1 (+C2), b' (LOWER3)
//   twist line:   block, L2', U2', C1 (+C2), b' (LOWER3) / xo (UPPER3)
//   upper sweep:  block, in-plane coupling (U2' / L2'), xo (UPPER3)
__device__ __forceinline__ void mbar_wait_a(unsigned bar, unsigned parity);
__device__ __forceinline__ void mbar_expect_tx_a(unsigned bar, unsigned bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
// The bulk copies of one record, issued by ONE lane.  A record costs that
// lane several hundred cycles (barrier wait, byte count, 4-5 copy
// instructions), more than a line step of the solver, so a producer warp
// works on NB consecutive records at a time, one per lane (produce_range).
__device__ __forceinline__ void tma_load_a(unsigned dst, const void *src, unsigned bytes, unsigned bar)
{
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}
template <int K>
__device__ __forceinline__ void rec_copy(const TsArrays &S, const PlaneDesc &P, const Seq &Q, int k, unsigned dst,
                                         unsigned bar)
{
    constexpr int LR = lr_of(K);
    constexpr unsigned lb = LR * 8u;
    const bool lower3 = P.mode == M_LOWER3;
    const int ph = k < Q.cnt ? 0 : k == Q.cnt ? 1 : 2;
    const i64 line = P.prec + Q.qrec(k);
    const double *src = S.solve + line * (i64)recd_of(K);
    // what the step reads: the in-plane coupling of its sweep (both for the twist line), the level-3
    // coupling(s) of a lower-sweep / twist line, the block; the record orders them so that this is
    // one range [lo, hi) (at most one unused coupling inside it)
    const bool l2 = ph == 1 || ((ph == 0) == (Q.w2 == 0)), u2 = ph == 1 || !l2;
    const bool l3 = ph < 2 && (P.two || P.c1 == o_l3(K)), u3 = ph < 2 && (P.two || P.c1 == o_u3(K));
    const int lo = l3 ? o_l3(K) : l2 ? o_l2(K) : o_efb(K);
    const int hi = u3 ? recd_of(K) : u2 ? o_u3(K) : o_u2(K);
    const bool extra = ph == 0 ? lower3 : ph == 1 ? true : !lower3;
    const double *xsrc = (lower3 ? S.b : S.x) + line * (i64)LR;
    mbar_expect_tx_a(bar, (unsigned)(hi - lo) * 8u + (extra ? lb : 0u));
    tma_load_a(dst + (unsigned)lo * 8u, src + lo, (unsigned)(hi - lo) * 8u, bar);
    if (extra) tma_load_a(dst + rx_of(K) * 8u, xsrc, lb, bar);
}

// records of planes idx0 .. idx1-1 of this warp's schedule (one level-3 phase)
template <int K, int D, class DescF>
__device__ void produce_range(const TsArrays &S, DescF &&desc, int idx0, int idx1, const Seq &Q, unsigned ring_a,
                              unsigned bars_a, unsigned &rec)
{
    constexpr int NB = D >= 8 ? 4 : D >= 4 ? 2 : 1;  // records in flight per step: half the ring at most
    constexpr unsigned SB = stage_of(K) * 8;
    const int lane = threadIdx.x & 31;
    const int n = 2 * Q.cnt + 1, total = (idx1 - idx0) * n;
    for (int g = 0; g < total; g += NB) {
        const int my = g + lane;
        if (lane < NB && my < total) {
            const int pl = my / n, k = my - pl * n;
            const PlaneDesc P = desc(idx0 + pl);
            const unsigned r = rec + (unsigned)my, st = r % D;
            // (no proxy fence: the solver only read the stage, and its release of the stage's
            // empty barrier orders those reads before the copies issued after this wait)
            if (r >= (unsigned)D) mbar_wait_a(bars_a + (D + st) * 8, ((r / D) + 1) & 1);
            rec_copy<K>(S, P, Q, k, ring_a + st * SB, bars_a + st * 8);
        }
        __syncwarp();
    }
    rec += (unsigned)total;
}

// ---- explicit accesses of the solver.  volatile: kept in program order among
// themselves and with the mbarrier operations, so the next line's operands
// are requested at chosen points of the current line's scans (the warp issues
// in order: a load placed early delays the chain, placed late it stalls the
// next line), and addressed with 32-bit shared addresses + immediates.
__device__ __forceinline__ double lds(unsigned a)
{
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ double2 lds2(unsigned a)
{
    double2 v;
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a));
    return v;
}
__device__ __forceinline__ void sts(unsigned a, double v) { asm volatile("st.shared.f64 [%0], %1;" ::"r"(a), "d"(v)); }
__device__ __forceinline__ double ldg(const double *p)
{
    double v;
    asm volatile("ld.global.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ void stg(double *p, double v) { asm volatile("st.global.f64 [%0], %1;" ::"l"(p), "d"(v)); }
// a line of the plane buffer (shared address) or of a global plane; byte offsets
__device__ __forceinline__ double ldb(unsigned a) { return lds(a); }
__device__ __forceinline__ double ldb(double *p) { return ldg(p); }
__device__ __forceinline__ void stb(unsigned a, double v) { sts(a, v); }
__device__ __forceinline__ void stb(double *p, double v) { stg(p, v); }
__device__ __forceinline__ unsigned adv(unsigned a, int bytes) { return a + bytes; }
__device__ __forceinline__ double *adv(double *p, int bytes) { return (double *)((char *)p + bytes); }
template <bool SMB>
struct BufT {
    typedef unsigned type;
};
template <>
struct BufT<false> {
    typedef double *type;
};

__device__ __forceinline__ void mbar_wait_a(unsigned bar, unsigned parity)
{
    unsigned ok = 0;
    while (!ok) {
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
            : "=r"(ok)
            : "r"(bar), "r"(parity)
            : "memory");
    }
}
__device__ __forceinline__ bool mbar_test_a(unsigned bar, unsigned parity)
{
    unsigned ok;
    asm volatile("{ .reg .pred p; mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(ok)
                 : "r"(bar), "r"(parity)
                 : "memory");
    return __all_sync(FULL_MASK, ok != 0);  // (warp-uniform by construction; the vote lets the compiler know)
}
// one lane releases a stage (barrier count 1): the warp's loads of the stage
// precede it in program order, and a 32-lane arrive would serialise 32 atomics
__device__ __forceinline__ void mbar_arrive_if(unsigned bar, bool on)
{
    asm volatile("{ .reg .pred p; setp.ne.u32 p, %1, 0; @p mbarrier.arrive.shared::cta.b64 _, [%0]; }" ::"r"(bar),
                 "r"((unsigned)on)
                 : "memory");
}

// Operands of one line step.
template <int K>
struct Ops {
    double eF[K], eB[K], cp[K], pt[K];
    double pr[NPREP];  // m2 m4 m8 e n2 n4 n8 f
};
template <int K>
struct Raw {  // x-independent inputs of a lower-sweep line: pt = bx - c1 n1 (- c2 n2)  or  c1 n1
    double bx[K], c1[K], c2[K], n1[K], n2[K];
};

template <int K>
__device__ __forceinline__ void ld_row(double (&v)[K], unsigned a)
{
#pragma unroll
    for (int k = 0; k < K; k++) v[k] = lds(a + k * 256);
}
template <int K, class BA>
__device__ __forceinline__ void ld_buf(double (&v)[K], BA a)
{
#pragma unroll
    for (int k = 0; k < K; k++) v[k] = ldb(adv(a, k * 256));
}
template <int K, class BA>
__device__ __forceinline__ void st_buf(BA a, const double (&v)[K])
{
#pragma unroll
    for (int k = 0; k < K; k++) stb(adv(a, k * 256), v[k]);
}
template <int A, int B, class F>
__device__ __forceinline__ void static_for(F &&f)
{
    if constexpr (A < B) {
        f(std::integral_constant<int, A>{});
        static_for<A + 1, B>(f);
    }
}
constexpr int NHOOK = 5;  // shuffle rounds of a line solve (4 levels + the exclusive level)

// One line: x = T^{-1} r for rho = mu r (SUB: x = y - T^{-1} r, y passed in x).
// hook(j), j = 0..4, runs right after the shuffles of round j are issued and
// hook(5) once the carries are formed: the caller requests a share of the
// next line's operands behind every round, so its loads fill the shuffle
// latencies instead of queueing in front of the next round's shuffles (a
// warp's shared-memory loads and shuffles go through the same in-order queue,
// ~6 cycles each).
template <int K, bool SUB, class FH>
__device__ __forceinline__ void solve_line(const Ops<K> &o, int l, const double (&rho)[K], double (&x)[K], FH &&hook)
{
    double pf[K], pb[K], pa[K], qa[K], Rr[K];
    pf[0] = rho[0];
    pa[0] = o.eF[0];
    pb[K - 1] = rho[K - 1];
    qa[K - 1] = o.eB[K - 1];
#pragma unroll
    for (int k = 1; k < K; k++) {
        pf[k] = fma(o.eF[k], pf[k - 1], rho[k]);
        pb[K - 1 - k] = fma(o.eB[K - 1 - k], pb[K - k], rho[K - 1 - k]);
    }
    double C = pf[K - 1], D = pb[0];
    // Kogge-Stone levels at distances 1, 2, 4, 8 (ntd_line_ts.cuh), both directions interleaved
    const double c1 = up(C, 1), d1 = dn(D, 1);
    hook(std::integral_constant<int, 0>{});
#pragma unroll
    for (int k = 1; k < K; k++) {
        pa[k] = o.eF[k] * pa[k - 1];
        qa[K - 1 - k] = o.eB[K - 1 - k] * qa[K - k];
    }
#pragma unroll
    for (int k = 0; k < K; k++) Rr[k] = k < K - 1 ? fma(o.eB[k], pb[k + 1 < K ? k + 1 : k], pf[k]) : pf[k];
    // (no lane masks on the level-1 multipliers and on the carries: the multiplier of a line's first
    // cell and of its last cell -- and of every padding cell -- is an exact zero, so lane 0's pa[] and
    // lane 31's qa[] are zeros and whatever finite value the edge shuffles return drops out)
    C = fma(pa[K - 1], c1, C);
    D = fma(qa[0], d1, D);
    const double c2 = up(C, 2), d2 = dn(D, 2);
    hook(std::integral_constant<int, 1>{});
    C = fma(o.pr[0], c2, C);
    D = fma(o.pr[4], d2, D);
    const double c4 = up(C, 4), d4 = dn(D, 4);
    hook(std::integral_constant<int, 2>{});
    C = fma(o.pr[1], c4, C);
    D = fma(o.pr[5], d4, D);
    const double c8 = up(C, 8), d8 = dn(D, 8);
    hook(std::integral_constant<int, 3>{});
    C = fma(o.pr[2], c8, C);
    D = fma(o.pr[6], d8, D);
    // exclusive carries
    const double u17 = up(C, 17), v17 = dn(D, 17), u1 = up(C, 1), v1 = dn(D, 1);
    hook(std::integral_constant<int, 4>{});
    const double cF = fma(o.pr[3], u17, u1);
    const double cB = fma(o.pr[7], v17, v1);
    hook(std::integral_constant<int, 5>{});
#pragma unroll
    for (int k = 0; k < K; k++) {
        if (SUB)
            x[k] = fma(-pa[k], cF, fma(-qa[k], cB, x[k] - Rr[k]));
        else
            x[k] = fma(pa[k], cF, fma(qa[k], cB, Rr[k]));
    }
}

// ---------------- solver: one plane
// Plane buffer (SMB): the warp keeps its half of the plane it processed last
// in shared memory (lines lo_line.. of the half incl. the twist line): each
// line slot holds the neighbour plane's final x until this plane's lower
// sweep replaces it with the lower-sweep value, which the upper sweep
// replaces with this plane's final x.  Without it (wide or tall planes) the
// same lines are read from / written to the global planes.
//
// A plane is 2 cnt + 1 records (lower lines, twist line, upper lines); step r
// solves record r while the operands of record r+1 are loaded (hooks of
// solve_line), so the serial chain per line is rho = pt - cp' xprev and the
// scans.  full(r+2) is tested during step r and the result consumed in step
// r+1 (an mbarrier test has a long latency: never wait on it in place).
template <int K, int D, int MODE, bool TWO, bool SMB>
__device__ void solve_plane(const TsArrays &S, const PlaneDesc &P, const Seq &Q, int bar_id, unsigned ex_a, int &parity,
                            unsigned ring_a, unsigned bars_a, unsigned &rec, unsigned pbuf_a)
{
    typedef typename BufT<SMB>::type BA;
    constexpr int LR = lr_of(K), LB = LR * 8;
    constexpr unsigned SB = stage_of(K) * 8;
    constexpr bool lower3 = MODE == M_LOWER3;
    const int lane = threadIdx.x & 31, w2 = Q.w2;
    const int ny = Q.ny, t2 = Q.t2, cnt = Q.cnt;
    const unsigned l8 = lane * 8, l16 = lane * 16;
    const i64 plr = (i64)ny * LR;  // plane stride in TS
    // Plane bases (line q of a plane at base + q*LR), this lane's column.  A
    // missing level-3 neighbour (first/last plane) has an exactly-zero
    // coupling; it reads the zero plane instead of branching.
    double *xpl = S.x + P.prec * LR + lane;
    const double *y1, *y2 = S.zero + lane;
    if (lower3) {
        if (TWO) {
            y1 = P.hasM ? xpl - plr : S.zero + lane;
            y2 = P.hasP ? xpl + plr : S.zero + lane;
        } else if (P.up) {
            y1 = P.hasP ? xpl + plr : S.zero + lane;
        } else {
            y1 = P.hasM ? xpl - plr : S.zero + lane;
        }
    } else {
        y1 = P.nbrUp ? xpl + plr : xpl - plr;
    }
    // line q of this plane's own values (xl) and of the level-3 neighbour (yn)
    BA xl, yn;
    const int q0 = cnt == 0 ? t2 : (w2 == 0 ? 0 : ny - 1), dq = w2 == 0 ? 1 : -1;
    if constexpr (SMB) {
        const unsigned bq = pbuf_a - (unsigned)((w2 == 0 ? 0 : t2) * LB) + l8;  // line q at bq + q*LB
        if (!P.nbuf) {  // prime the buffer with the neighbour plane (a sweep's first plane)
            constexpr int CH = K <= 4 ? 8 : 2;  // lines in flight
            const int qa_ = w2 == 0 ? 0 : t2, qb_ = w2 == 0 ? t2 : ny - 1;
            for (int q = qa_; q <= qb_; q += CH) {
                double v[CH][K];
#pragma unroll
                for (int j = 0; j < CH; j++)
#pragma unroll
                    for (int k = 0; k < K; k++) v[j][k] = ldg(y1 + (i64)(q + j <= qb_ ? q + j : qb_) * LR + k * 32);
#pragma unroll
                for (int j = 0; j < CH; j++)
#pragma unroll
                    for (int k = 0; k < K; k++) sts(bq + (q + j <= qb_ ? q + j : qb_) * LB + k * 256, v[j][k]);
            }
        }
        xl = yn = bq + q0 * LB;
    } else {
        xl = (lower3 ? S.x : S.xs) + P.prec * LR + lane + (i64)q0 * LR;
        yn = const_cast<double *>(y1) + (i64)q0 * LR;
    }
    const double *y2p = y2 + (i64)q0 * LR;
    const int dqB = dq * LB;
    auto sa = [&](unsigned r) { return ring_a + (r % D) * SB; };
    auto full = [&](unsigned r) { return bars_a + (r % D) * 8; };
    auto empty = [&](unsigned r) { return bars_a + (D + r % D) * 8; };
    auto par = [&](unsigned r) { return (r / D) & 1u; };
    // in-plane coupling of the lower sweep (and of the twist line's first neighbour) / of the upper sweep
    const unsigned cpL = (unsigned)(w2 == 0 || cnt == 0 ? o_l2(K) : o_u2(K)) * 8 + l8;
    const unsigned cpU = (unsigned)(w2 == 0 ? o_u2(K) : o_l2(K)) * 8 + l8;
    const unsigned c1o = (unsigned)P.c1 * 8 + l8;
    // The operand loads of a record as a list of NL_L / NL_U single loads; share j of NHOOK is issued
    // behind shuffle round j of the line being solved (share = -1: all of them).
    //   lower-type record: c1, n1, [bx], [c2, n2], cp, eF|eB pairs, scan coefficient pairs
    //   upper-type record: cp, y, [xo], eF|eB pairs, scan coefficient pairs
    constexpr int NL_L = K * (4 + (lower3 ? 1 : 0) + (TWO ? 2 : 0)) + NPREP / 2;
    constexpr int NL_U = K * (3 + (lower3 ? 0 : 1)) + NPREP / 2;
    // (narrow lines; wide lines use the lists only for a plane's first record and place their loads
    // by register lifetime, below)
    auto item_L = [&](auto I, auto WN, Ops<K> &o, Raw<K> &w, unsigned s, BA ya, const double *y2q, unsigned cpo) {
        constexpr int i = decltype(I)::value;
        constexpr bool wn = decltype(WN)::value;
        constexpr int nb = lower3 ? 1 : 0, nt = TWO ? 2 : 0;
        if constexpr (i < K) {
            w.c1[i] = lds(s + c1o + i * 256);
        } else if constexpr (i < 2 * K) {
            if constexpr (wn) w.n1[i - K] = ldb(adv(ya, (i - K) * 256));
        } else if constexpr (i < (2 + nb) * K) {
            w.bx[i - 2 * K] = lds(s + rx_of(K) * 8 + l8 + (i - 2 * K) * 256);
        } else if constexpr (i < (2 + nb + nt) * K) {
            constexpr int j = i - (2 + nb) * K;
            if constexpr (j < K)
                w.c2[j] = lds(s + o_u3(K) * 8 + l8 + j * 256);
            else if constexpr (wn)
                w.n2[j - K] = ldg(y2q + (j - K) * 32);
        } else if constexpr (i < (3 + nb + nt) * K) {
            constexpr int j = i - (2 + nb + nt) * K;
            o.cp[j] = lds(s + cpo + j * 256);
        } else if constexpr (i < (4 + nb + nt) * K) {
            constexpr int j = i - (3 + nb + nt) * K;
            const double2 v = lds2(s + l16 + o_efb(K) * 8 + j * 512);
            o.eF[j] = v.x;
            o.eB[j] = v.y;
        } else {
            constexpr int j = i - (4 + nb + nt) * K;
            const double2 v = lds2(s + l16 + o_prep(K) * 8 + j * 512);
            o.pr[2 * j] = v.x;
            o.pr[2 * j + 1] = v.y;
        }
    };
    auto item_U = [&](auto I, auto WN, Ops<K> &o, double (&y)[K], double (&xo)[K], unsigned s, BA ya) {
        constexpr int i = decltype(I)::value;
        constexpr bool wn = decltype(WN)::value;
        constexpr int nx_ = lower3 ? 0 : 1;
        if constexpr (i < K) {
            o.cp[i] = lds(s + cpU + i * 256);
        } else if constexpr (i < 2 * K) {
            if constexpr (wn) y[i - K] = ldb(adv(ya, (i - K) * 256));
        } else if constexpr (i < (2 + nx_) * K) {
            xo[i - 2 * K] = lds(s + rx_of(K) * 8 + l8 + (i - 2 * K) * 256);
        } else if constexpr (i < (3 + nx_) * K) {
            constexpr int j = i - (2 + nx_) * K;
            const double2 v = lds2(s + l16 + o_efb(K) * 8 + j * 512);
            o.eF[j] = v.x;
            o.eB[j] = v.y;
        } else {
            constexpr int j = i - (3 + nx_) * K;
            const double2 v = lds2(s + l16 + o_prep(K) * 8 + j * 512);
            o.pr[2 * j] = v.x;
            o.pr[2 * j + 1] = v.y;
        }
    };
    const std::integral_constant<bool, true> WITH_N{};
    auto load_L = [&](auto J, auto WN, Ops<K> &o, Raw<K> &w, unsigned s, BA ya, const double *y2q, unsigned cpo) {
        constexpr int j = decltype(J)::value;
        constexpr int a = j < 0 ? 0 : j * NL_L / NHOOK, b = j < 0 ? NL_L : (j + 1) * NL_L / NHOOK;
        static_for<a, b>([&](auto I) { item_L(I, WN, o, w, s, ya, y2q, cpo); });
    };
    auto load_U = [&](auto J, auto WN, Ops<K> &o, double (&y)[K], double (&xo)[K], unsigned s, BA ya) {
        constexpr int j = decltype(J)::value;
        constexpr int a = j < 0 ? 0 : j * NL_U / NHOOK, b = j < 0 ? NL_U : (j + 1) * NL_U / NHOOK;
        static_for<a, b>([&](auto I) { item_U(I, WN, o, y, xo, s, ya); });
    };
    auto nbr_L = [&](Raw<K> &w, BA ya, const double *y2q) {
        ld_buf(w.n1, ya);
        if (TWO) {
#pragma unroll
            for (int k = 0; k < K; k++) w.n2[k] = ldg(y2q + k * 32);
        }
    };
    const std::integral_constant<int, -1> ALL{};
    auto fin_L = [&](Ops<K> &o, const Raw<K> &w) {
#pragma unroll
        for (int k = 0; k < K; k++) {
            double v = lower3 ? fma(-w.c1[k], w.n1[k], w.bx[k]) : w.c1[k] * w.n1[k];
            if (TWO) v = fma(-w.c2[k], w.n2[k], v);
            o.pt[k] = v;
        }
    };
    // PIPE (narrow lines): step r solves record r while the operands of record r+1 are loaded behind
    // its shuffle rounds, in five equal shares.  Wide lines (K > 5) do not have the registers for two
    // whole operand sets; their loads follow the registers as the line solve frees them: the rhs part
    // and cp of record r die with rho, eF / eB with the lane maps, so record r+1's couplings, then its
    // rhs part, then its eF / eB are loaded behind rounds 0..4, while its scan coefficients (and xo)
    // are read in its own step behind round 0, after which the stage is released.  Neighbour-plane
    // values, which come from global memory, are requested two lines ahead (wn).
    constexpr bool PIPE = K <= 5;
    const unsigned cpT = (unsigned)o_l2(K) * 8 + l8;  // the twist record is read with L2' as cp
    Ops<K> cur;
    Raw<K> wn;  // wide lines: couplings of the next lower-type record, neighbour values of the one after
    bool okn = true;
    auto ld_pr = [&](Ops<K> &o, unsigned s) {
#pragma unroll
        for (int j = 0; j < NPREP / 2; j++) {
            const double2 v = lds2(s + l16 + o_prep(K) * 8 + j * 512);
            o.pr[2 * j] = v.x;
            o.pr[2 * j + 1] = v.y;
        }
    };
    auto ld_efb = [&](auto A, auto B, Ops<K> &o, unsigned s) {
        static_for<decltype(A)::value, decltype(B)::value>([&](auto J) {
            constexpr int j = decltype(J)::value;
            const double2 v = lds2(s + l16 + o_efb(K) * 8 + j * 512);
            o.eF[j] = v.x;
            o.eB[j] = v.y;
        });
    };
    const std::integral_constant<int, 0> I0{};
    const std::integral_constant<int, (K + 1) / 2> IH{};
    const std::integral_constant<int, K> IK{};
    // ---------------- prologue: the plane's first record (a lower line, or the twist line when cnt == 0)
    {
        Raw<K> w;
        mbar_wait_a(full(rec), par(rec));
        load_L(ALL, WITH_N, cur, w, sa(rec), yn, y2p, cpL);
        if constexpr (PIPE) mbar_arrive_if(empty(rec), lane == 0 && cnt > 0);  // the twist record releases itself
        okn = mbar_test_a(full(rec + 1), par(rec + 1));
        fin_L(cur, w);
        if constexpr (!PIPE) nbr_L(wn, cnt > 0 ? adv(yn, dqB) : yn, cnt > 0 ? y2p + dq * LR : y2p);
    }
    // ---------------- level-2 lower sweep (ntd_solve.py:147-171)
    double xprev[K];
#pragma unroll
    for (int k = 0; k < K; k++) xprev[k] = 0.0;
#pragma unroll 1
    for (int i = 0; i < cnt; i++, rec++) {
        Ops<K> nxt;
        Raw<K> w;
        const bool last = i == cnt - 1;  // the next record is the twist line (an L-type record as well)
        // (checked here, at a block boundary: a branch inside the line solve splits its straight-line
        // code and costs ~65 cycles per step)
        if (!okn) mbar_wait_a(full(rec + 1), par(rec + 1));
        // wide lines: neighbour values two lines ahead (the twist line is the last lower-type record)
        const BA yn2 = last ? yn : adv(yn, 2 * dqB);
        const double *y2q2 = last ? y2p : y2p + 2 * dq * LR;
        const unsigned sn = sa(rec + 1), cpn = last ? cpT : cpL;
        double rho[K], x[K];
#pragma unroll
        for (int k = 0; k < K; k++) rho[k] = fma(-cur.cp[k], xprev[k], cur.pt[k]);  // line 0: xprev = 0
        solve_line<K, false>(cur, lane, rho, x, [&](auto J) {
            constexpr int j = decltype(J)::value;
            if constexpr (!PIPE) {
                if constexpr (j == 0) {
                    ld_pr(cur, sa(rec));
                    mbar_arrive_if(empty(rec), lane == 0);
                    ld_row(wn.c1, sn + c1o);
                } else if constexpr (j == 1) {
                    if constexpr (lower3) ld_row(wn.bx, sn + rx_of(K) * 8 + l8);
                    if constexpr (TWO) ld_row(wn.c2, sn + o_u3(K) * 8 + l8);
                } else if constexpr (j == 2) {
                    fin_L(nxt, wn);
                    nbr_L(wn, yn2, y2q2);
                    ld_row(nxt.cp, sn + cpn);
                } else if constexpr (j == 3) {
                    ld_efb(I0, IH, nxt, sn);
                } else if constexpr (j == 4) {
                    ld_efb(IH, IK, nxt, sn);
                } else {
                    okn = mbar_test_a(full(rec + 2), par(rec + 2));
                }
            } else if constexpr (j < NHOOK) {
                load_L(J, WITH_N, nxt, w, sa(rec + 1), adv(yn, dqB), y2p + dq * LR, last ? cpT : cpL);
            } else {
                mbar_arrive_if(empty(rec + 1), lane == 0 && !last);
                okn = mbar_test_a(full(rec + 2), par(rec + 2));
            }
        });
        st_buf(xl, x);
#pragma unroll
        for (int k = 0; k < K; k++) xprev[k] = x[k];
        if constexpr (PIPE) fin_L(nxt, w);
        cur = nxt;
        xl = adv(xl, dqB);
        yn = adv(yn, dqB);
        y2p += dq * LR;
    }
    // ---------------- exchange the lines next to the twist
    const unsigned mine = ex_a + (unsigned)((parity * 2 + w2) * LB) + l8;
    const unsigned other = ex_a + (unsigned)((parity * 2 + (1 - w2)) * LB) + l8;
#pragma unroll
    for (int k = 0; k < K; k++) sts(mine + k * 256, xprev[k]);
    named_bar(bar_id, 64);
    parity ^= 1;
    double xo_[K];
    ld_row(xo_, other);
    // ---------------- twist line (ntd_solve.py:172-177); xl / yn are at line t2
    double xn[K];
    Ops<K> nxt;
    double ycur[K], xocur[K];
    {
        double u2c[K], xo[K];
        if constexpr (!PIPE) ld_pr(cur, sa(rec));
        ld_row(u2c, sa(rec) + o_u2(K) * 8 + l8);
        if (!lower3) ld_row(xo, sa(rec) + rx_of(K) * 8 + l8);
        mbar_arrive_if(empty(rec), lane == 0);
        if (cnt > 0 && !okn) mbar_wait_a(full(rec + 1), par(rec + 1));
        double rho[K];
#pragma unroll
        for (int k = 0; k < K; k++) {
            const double xa = w2 == 0 ? xprev[k] : xo_[k], xd = w2 == 0 ? xo_[k] : xprev[k];
            double v = cur.pt[k];
            if (t2 > 0) v = fma(-cur.cp[k], xa, v);
            if (t2 < ny - 1) v = fma(-u2c[k], xd, v);
            rho[k] = v;
        }
        solve_line<K, false>(cur, lane, rho, xn, [&](auto J) {
            constexpr int j = decltype(J)::value;
            if (cnt > 0) {
                if constexpr (!PIPE) {
                    if constexpr (j == 0) ld_row(nxt.cp, sa(rec + 1) + cpU);
                    if constexpr (j == 1) ld_buf(ycur, adv(xl, -dqB));
                    if constexpr (j == 3) ld_efb(I0, IH, nxt, sa(rec + 1));
                    if constexpr (j == 4) ld_efb(IH, IK, nxt, sa(rec + 1));
                    if constexpr (j == NHOOK) okn = mbar_test_a(full(rec + 2), par(rec + 2));
                } else if constexpr (j < NHOOK) {
                    load_U(J, WITH_N, nxt, ycur, xocur, sa(rec + 1), adv(xl, -dqB));
                } else {
                    mbar_arrive_if(empty(rec + 1), lane == 0);
                    okn = mbar_test_a(full(rec + 2), par(rec + 2));
                }
            }
        });
        double nv[K];
#pragma unroll
        for (int k = 0; k < K; k++) nv[k] = lower3 ? xn[k] : xo[k] - xn[k];  // UPPER3: final = xo - value
        rec++;
        if (w2 == 0) {
#pragma unroll
            for (int k = 0; k < K; k++) stg(xpl + (i64)t2 * LR + k * 32, nv[k]);
        }
        if constexpr (SMB) st_buf(xl, nv);  // both warps keep the twist line
    }
    // ---------------- level-2 upper sweep (ntd_solve.py:178-185)
    //   value_q = y_q - T_q^{-1}(cp' value_prev);  LOWER3: x_q = value_q;  UPPER3: x_q = xo_q - value_q
    cur = nxt;
    BA xu = adv(xl, -dqB);
    double *xg = xpl + (i64)(t2 - dq) * LR;
#pragma unroll 1
    for (int i = 0; i < cnt; i++, rec++) {
        const bool more = i + 1 < cnt;
        double ynx[K], xonx[K];
        if (more && !okn) mbar_wait_a(full(rec + 1), par(rec + 1));
        double rho[K];
#pragma unroll
        for (int k = 0; k < K; k++) rho[k] = cur.cp[k] * xn[k];
#pragma unroll
        for (int k = 0; k < K; k++) xn[k] = ycur[k];
        // past the sweep's last line the loads read stale ring / buffer data that is never used
        solve_line<K, true>(cur, lane, rho, xn, [&](auto J) {
            constexpr int j = decltype(J)::value;
            if constexpr (!PIPE) {
                if constexpr (j == 0) {
                    ld_pr(cur, sa(rec));
                    if constexpr (!lower3) ld_row(xocur, sa(rec) + rx_of(K) * 8 + l8);
                    mbar_arrive_if(empty(rec), lane == 0);
                    ld_row(nxt.cp, sa(rec + 1) + cpU);
                } else if constexpr (j == 1) {
                    ld_buf(ynx, adv(xu, -dqB));
                } else if constexpr (j == 3) {
                    ld_efb(I0, IH, nxt, sa(rec + 1));
                } else if constexpr (j == 4) {
                    ld_efb(IH, IK, nxt, sa(rec + 1));
                } else if constexpr (j == NHOOK) {
                    okn = mbar_test_a(full(rec + 2), par(rec + 2));
                }
            } else if constexpr (j < NHOOK) {
                load_U(J, WITH_N, nxt, ynx, xonx, sa(rec + 1), adv(xu, -dqB));
            } else {
                mbar_arrive_if(empty(rec + 1), lane == 0 && more);
                okn = mbar_test_a(full(rec + 2), par(rec + 2));
            }
        });
        double nv[K];
#pragma unroll
        for (int k = 0; k < K; k++) nv[k] = lower3 ? xn[k] : xocur[k] - xn[k];
#pragma unroll
        for (int k = 0; k < K; k++) stg(xg + k * 32, nv[k]);
        if constexpr (SMB) st_buf(xu, nv);
#pragma unroll
        for (int k = 0; k < K; k++) ycur[k] = ynx[k];
        cur = nxt;
        if constexpr (PIPE) {
#pragma unroll
            for (int k = 0; k < K; k++) xocur[k] = xonx[k];
        }
        xu = adv(xu, -dqB);
        xg -= dq * LR;
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
    // (warp index through a shuffle: provably warp-uniform, so every branch on the warp's role,
    // half and trip counts is a uniform branch and the shuffles need no divergence checks)
    const int lane = threadIdx.x & 31, warp = __shfl_sync(FULL_MASK, (int)(threadIdx.x >> 5), 0);
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
            mbar_init(&R.empty[st], 1);  // released by lane 0 of the solver warp
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
    const unsigned ex_a = smem_u32(ex[NP == 2 ? pair : 0]);
    const unsigned ring_a = smem_u32(R.base), bars_a = smem_u32(bars[sw]), pbuf_a = smem_u32(pbuf);
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
            P.c1 = o_l3(K);  // (and U3 as the second coupling)
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
    if (producer) {
        produce_range<K, D>(S, desc, 0, nlow, Q, ring_a, bars_a, rec);
    } else {
        for (int i = 0; i < nlow; i++)
            solve_plane<K, D, M_LOWER3, false, SMB>(S, desc(i), Q, bar, ex_a, parity, ring_a, bars_a, rec, pbuf_a);
    }
    phase_sync();
    if (pair == 0) {
        if (producer) {
            fence_proxy_async();
            produce_range<K, D>(S, desc, nlow, nlow + 1, Q, ring_a, bars_a, rec);
        } else {
            solve_plane<K, D, M_LOWER3, true, SMB>(S, desc(nlow), Q, bar, ex_a, parity, ring_a, bars_a, rec, pbuf_a);
        }
    }
    phase_sync();
    if (producer) {
        fence_proxy_async();  // x (read as xo) was written by generic stores
        produce_range<K, D>(S, desc, nlow + ntw, nplanes, Q, ring_a, bars_a, rec);
    } else {
        for (int i = nlow + ntw; i < nplanes; i++)
            solve_plane<K, D, M_UPPER3, false, SMB>(S, desc(i), Q, bar, ex_a, parity, ring_a, bars_a, rec, pbuf_a);
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
    // (+ one pad line: the last upper-sweep step requests a line past its buffer)
    const size_t smem = (size_t)2 * D * ts::stage_of(K) * 8 + (SMB ? (size_t)(2 * bl + 1) * ts::lr_of(K) * 8 : 0);
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
