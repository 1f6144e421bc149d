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
// padded slots are zero maps that need no branches.  The factor is converted
// to solve records once at setup (ntd_solve_bands); b is converted (and
// scaled by m) on entry and x converted back on exit.
//
// Per line step the solver waits on an mbarrier, reads its slots from a
// D-deep ring of line records streamed by 1-D bulk TMA (issued by the
// producer warp), forms the scan constants, runs the radix-4 16-lane scans
// of the twisted line solve (ntd_line4.cuh) and stores x.  x-dependent
// operands (neighbour plane, lower-sweep values of this plane) are loaded by
// the solver one line ahead.
#pragma once
#include "ntd_kernels.cuh"
#include "ntd_line4.cuh"

namespace sl {


// Solve record of one line (record-major, [system][line][RECD]):
//   [ NL | NU | PREP (NPREP x 32) | L2' | U2' | L3' | U3' ]
// NL = -(l1 m), NU = -(u1 m) are the chain coefficients, PREP the line's
// factor-only scan coefficients, and the couplings are pre-multiplied by the
// level-1 pivot reciprocal m (c' = c m), as is b on entry (b' = b m), so the
// solver forms the scan constants cr = b' - sum c' y directly and m itself is
// never streamed.  A phase copies only the block [NL|NU|PREP] plus the
// couplings it reads.
constexpr int NPREP = 11;  // stored LinePrep coefficients per lane ([coef][lane]); p1, e0, q1, f0 are rebuilt
__host__ __device__ constexpr int lr_of(int K) { return 32 * K + 2; }
__host__ __device__ constexpr int o_nl(int K) { return 0; }
__host__ __device__ constexpr int o_nu(int K) { return lr_of(K); }
__host__ __device__ constexpr int o_prep(int K) { return 2 * lr_of(K); }
__host__ __device__ constexpr int blk_of(int K) { return 2 * lr_of(K) + NPREP * 32; }  // [NL|NU|PREP]
__host__ __device__ constexpr int o_l2(int K) { return blk_of(K); }
__host__ __device__ constexpr int o_u2(int K) { return blk_of(K) + lr_of(K); }
__host__ __device__ constexpr int o_l3(int K) { return blk_of(K) + 2 * lr_of(K); }
__host__ __device__ constexpr int o_u3(int K) { return blk_of(K) + 3 * lr_of(K); }
__host__ __device__ constexpr int recd_of(int K) { return blk_of(K) + 4 * lr_of(K); }
// ring stage: [block | S0: in-plane coupling | S1: C1 | S2: C2 | X: b' or xo]
__host__ __device__ constexpr int rs0_of(int K) { return blk_of(K); }
__host__ __device__ constexpr int rs1_of(int K) { return blk_of(K) + lr_of(K); }
__host__ __device__ constexpr int rs2_of(int K) { return blk_of(K) + 2 * lr_of(K); }
__host__ __device__ constexpr int rx_of(int K) { return blk_of(K) + 3 * lr_of(K); }
__host__ __device__ constexpr int stage_of(int K) { return blk_of(K) + 4 * lr_of(K); }
// ring depth: as many stages as fit beside the static shared memory (<= 8)
__host__ __device__ constexpr int static_smem_of(int K) { return 2 * 2 * 2 * (32 * K + 1) * 8 + 4 * 2 * 8 * 8; }
__host__ __device__ constexpr int depth_of(int K)
{
    return (232448 - 1024 - static_smem_of(K)) / (4 * stage_of(K) * 8) > 8
               ? 8
               : (232448 - 1024 - static_smem_of(K)) / (4 * stage_of(K) * 8);
}

// split kernel (one level-3 half per CTA, 2 solver warps): its own depth
__host__ __device__ constexpr int static_smem2_of(int K) { return 2 * 2 * (32 * K + 1) * 8 + 2 * 2 * 8 * 8; }
__host__ __device__ constexpr int depth2_of(int K)
{
    return (232448 - 1024 - static_smem2_of(K)) / (2 * stage_of(K) * 8) > 8
               ? 8
               : (232448 - 1024 - static_smem2_of(K)) / (2 * stage_of(K) * 8);
}

// SMB split kernel: ring depth left beside the two plane buffers, sized for
// ny <= 32K+1 (a half-plane of 16K+1 lines per solver warp); < 2: no SMB
__host__ __device__ constexpr int depth_smb_of(int K)
{
    return (232448 - 1024 - static_smem2_of(K) - 2 * (16 * K + 1) * lr_of(K) * 8) / (2 * stage_of(K) * 8) > 8
               ? 8
               : (232448 - 1024 - static_smem2_of(K) - 2 * (16 * K + 1) * lr_of(K) * 8) / (2 * stage_of(K) * 8);
}

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

// cell of SL element r of a line (-1: padding)
__device__ __forceinline__ int sl_cell(int r, int nx, int K)
{
    const int t = (nx - 1) / 2;
    const int P0 = 16 * K - t, P1 = 16 * K - (nx - 1 - t);
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
    return c;
}

// b (B, N) -> b' = b m in SL (B, N_SL).  One thread per SL element.
static __global__ void k_to_sl(const double *__restrict__ src, const double *__restrict__ pre,
                               double *__restrict__ dst, int nx, i64 lines, int K, i64 batch)
{
    const int LR = lr_of(K);
    const i64 total = lines * LR * batch, n = lines * nx;
    for (i64 e = blockIdx.x * (i64)blockDim.x + threadIdx.x; e < total; e += (i64)gridDim.x * blockDim.x) {
        const i64 line = e / LR;  // global line over batch
        const int r = (int)(e - line * LR);
        const int c = sl_cell(r, nx, K);
        const i64 s = line / lines, g = line * nx + c;
        dst[e] = c >= 0 ? src[g] * pre[s * 6 * n + 6 * n + g] : 0.0;  // pre[s][6][cell]: m
    }
}

// x in SL -> natural; systems masked off by `active` get x = 0
static __global__ void k_from_sl(const double *__restrict__ src, double *__restrict__ dst, int nx, i64 lines, int K,
                                 i64 batch, const int32_t *__restrict__ active)
{
    const int LR = lr_of(K);
    const i64 total = lines * nx * batch;
    for (i64 e = blockIdx.x * (i64)blockDim.x + threadIdx.x; e < total; e += (i64)gridDim.x * blockDim.x) {
        const i64 line = e / nx;
        const int c = (int)(e - line * nx);
        const bool on = !active || active[line / lines];
        dst[e] = on ? src[line * LR + sl_index(c, nx, K)] : 0.0;
    }
}

// solve records from a factor (B,7,N): NL, NU, (PREP by k_prep_sl), m l2, m u2, m l3, m u3
static __global__ void k_solve_sl(const double *__restrict__ pre, double *__restrict__ solve, int nx, i64 lines, int K,
                                  i64 batch)
{
    const int LR = lr_of(K), RECD = recd_of(K);
    const i64 nsl = lines * LR, n = lines * nx;
    const i64 total = nsl * batch;
    for (i64 e = blockIdx.x * (i64)blockDim.x + threadIdx.x; e < total; e += (i64)gridDim.x * blockDim.x) {
        const i64 s = e / nsl, el = e - s * nsl;
        const i64 line = el / LR;
        const int r = (int)(el - line * LR);
        const int c = sl_cell(r, nx, K);
        const double *p = pre + s * 7 * n;
        double *o = solve + (s * lines + line) * (i64)RECD + r;
        const i64 g = line * nx + c;
        const bool on = c >= 0;
        const double m = on ? p[6 * n + g] : 0.0;
        o[o_nl(K)] = on ? -(p[g] * m) : 0.0;
        o[o_nu(K)] = on ? -(p[n + g] * m) : 0.0;
        o[o_l2(K)] = on ? p[2 * n + g] * m : 0.0;
        o[o_u2(K)] = on ? p[3 * n + g] * m : 0.0;
        o[o_l3(K)] = on ? p[4 * n + g] * m : 0.0;
        o[o_u3(K)] = on ? p[5 * n + g] * m : 0.0;
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
    const double *b;      // b' = b m
    double *x, *xs;
    const double *zero;   // one plane of zero records: the missing level-3 neighbour
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
__device__ __forceinline__ void st_rec(double *rec, const LaneSl<K> &L, const double (&v)[K], double vt)
{
#pragma unroll
    for (int k = 0; k < K; k++) rec[L.base + k] = v[k];
    rec[L.tw] = vt;  // every lane holds the same twist value: branch-free
}

// ring of D stages per solver warp
template <int K, int D>
struct Ring {
    double *base;
    unsigned long long *full, *empty;
    __device__ __forceinline__ double *stage(int st) const { return base + (size_t)st * stage_of(K); }
};

struct PlaneDesc {
    bool nbuf;     // SMB: the level-3 neighbour y1 is the plane this warp processed last (in its smem buffer)
    i64 prec;      // record index of the plane's first line (plane * ny)
    int mode;      // M_LOWER3 / M_UPPER3
    int c1;        // record offset of the level-3 coupling C1 (two: L3 then U3 = C2)
    bool two;      // both level-3 neighbours (twist plane)
    bool hasM, hasP, nbrUp;
    bool up;       // lower sweep: the level-3 neighbour is plane p+1 (descending half)
};

struct Seq {
    int cnt, t2, ny, w2;
    __device__ __forceinline__ int qlow(int i) const { return w2 == 0 ? i : ny - 1 - i; }
    __device__ __forceinline__ int qup(int i) const { return w2 == 0 ? t2 - 1 - i : t2 + 1 + i; }
};

// stored scan coefficients + the four rebuilt ones (same expressions as line_prep)
template <int K>
__device__ __forceinline__ LinePrep read_prep(const double *pp, int lane, const double (&aL)[K],
                                              const double (&aU)[K])
{
    const int s = lane & 15;
    LinePrep P;
    double A0 = 1.0, B0 = 1.0;
#pragma unroll
    for (int k = 0; k < K; k++) {
        A0 *= aL[k];
        B0 *= aU[k];
    }
    P.p1 = s >= 1 ? A0 : 0.0;
    P.e0 = s >= 1 ? 1.0 : 0.0;
    P.q1 = s <= 14 ? B0 : 0.0;
    P.f0 = s <= 14 ? 1.0 : 0.0;
    P.p2 = pp[0 * 32 + lane];
    P.p3 = pp[1 * 32 + lane];
    P.e1 = pp[2 * 32 + lane];
    P.e2 = pp[3 * 32 + lane];
    P.e3 = pp[4 * 32 + lane];
    P.q2 = pp[5 * 32 + lane];
    P.q3 = pp[6 * 32 + lane];
    P.f1 = pp[7 * 32 + lane];
    P.f2 = pp[8 * 32 + lane];
    P.f3 = pp[9 * 32 + lane];
    P.bex = pp[10 * 32 + lane];
    return P;
}

// scan coefficients of every line (setup): one warp per line
template <int K>
__global__ void k_prep_sl(double *__restrict__ solve, i64 lines_total)
{
    const int lane = threadIdx.x & 31;
    const i64 line = (blockIdx.x * (i64)blockDim.x + threadIdx.x) >> 5;
    if (line >= lines_total) return;
    double *rec = solve + line * (i64)recd_of(K);
    const LaneSl<K> L(lane);
    double aL[K], aU[K];
    ld_rec(rec + (L.desc ? o_nu(K) : o_nl(K)), L, aL);
    ld_rec(rec + (L.desc ? o_nl(K) : o_nu(K)), L, aU);
    const LinePrep P = line_prep<K>(lane & 15, aL, aU);
    double *pp = rec + o_prep(K);
    const double v[NPREP] = {P.p2, P.p3, P.e1, P.e2, P.e3, P.q2, P.q3, P.f1, P.f2, P.f3, P.bex};
#pragma unroll
    for (int c = 0; c < NPREP; c++) pp[c * 32 + lane] = v[c];
}

// ---------------- producer: bulk copies of what each line step reads
//   lower sweep:  block, in-plane coupling (L2' / U2' by half), C1 (+C2), b' (LOWER3)
//   upper sweep:  block, in-plane coupling (U2' / L2'), xo (UPPER3)
// Record k of a plane (k < cnt: lower sweep, else upper sweep) is copied
// into a ring stage (dst) or, with dst == nullptr, prefetched into L2.
#ifndef NTD_L2_PF
#define NTD_L2_PF 0
#endif
constexpr int L2_PF = NTD_L2_PF;
#ifndef NTD_PRODUCER_FENCE
#define NTD_PRODUCER_FENCE 1
#endif
constexpr bool PRODUCER_FENCE = NTD_PRODUCER_FENCE;
#ifndef NTD_WAIT_AHEAD
#define NTD_WAIT_AHEAD 1
#endif
constexpr bool WAIT_AHEAD = NTD_WAIT_AHEAD;  // test the barrier of record i+2, consume after the solve
  // L2 prefetch distance in records (ahead of the ring copies)

__device__ __forceinline__ void prefetch_bulk_l2(const double *p, unsigned bytes)
{
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// Producer-side wait.  try_wait suspends the warp in hardware until the phase
// completes (or the hint expires), so a waiting producer takes no issue slots
// from the solver warp of its SM sub-partition.
#ifndef NTD_PRODUCER_TRYWAIT
#define NTD_PRODUCER_TRYWAIT 1
#endif
__device__ __forceinline__ void mbar_wait_producer(void *bar, unsigned parity)
{
    if constexpr (NTD_PRODUCER_TRYWAIT) {
        unsigned ok = 0;
        const unsigned a = smem_u32(bar);
        while (!ok) {
            asm volatile(
                "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3; selp.u32 %0, 1, 0, p; }"
                : "=r"(ok)
                : "r"(a), "r"(parity), "r"(1000000u)
                : "memory");
        }
    } else {
        mbar_wait_lazy(bar, parity);
    }
}

template <int K>
__device__ __forceinline__ void rec_copy(const SlArrays &S, const PlaneDesc &P, const Seq &Q, int k, double *dst,
                                         unsigned long long *bar)
{
    constexpr int LR = lr_of(K);
    constexpr unsigned lb = LR * 8u, bb = blk_of(K) * 8u;
    const bool lower3 = P.mode == M_LOWER3;
    const int ph = k < Q.cnt ? 0 : 1, i = ph ? k - Q.cnt : k;
    const int cpl = (ph == 0) == (Q.w2 == 0) ? o_l2(K) : o_u2(K);
    const unsigned nc = ph == 0 ? (P.two ? 2u : 1u) : 0u;
    const bool extra = ph == 0 ? lower3 : !lower3;
    const i64 line = P.prec + (ph == 0 ? Q.qlow(i) : Q.qup(i));
    const double *src = S.solve + line * (i64)recd_of(K);
    const double *xsrc = (ph == 0 ? S.b : S.x) + line * (i64)LR;
    if (dst) {
        mbar_expect_tx(bar, bb + lb + nc * lb + (extra ? lb : 0u));
        tma_load_1d(dst, src, bb, bar);
        tma_load_1d(dst + rs0_of(K), src + cpl, lb, bar);
        if (nc) tma_load_1d(dst + rs1_of(K), src + P.c1, nc * lb, bar);
        if (extra) tma_load_1d(dst + rx_of(K), xsrc, lb, bar);
    } else {
        prefetch_bulk_l2(src, bb);
        prefetch_bulk_l2(src + cpl, lb);
        if (nc) prefetch_bulk_l2(src + P.c1, nc * lb);
        if (extra) prefetch_bulk_l2(xsrc, lb);
    }
}

// Pn: the warp's next plane (L2 prefetch runs across the boundary), or nullptr
template <int K, int D>
__device__ void produce_plane(const SlArrays &S, const PlaneDesc &P, const PlaneDesc *Pn, const Seq &Q,
                              const Ring<K, D> &R, unsigned &rec)
{
    const int lane = threadIdx.x & 31;
    const int n = 2 * Q.cnt;
    if (lane == 0) {
        for (int k = 0; k < n; k++, rec++) {
            if constexpr (L2_PF > 0) {
                const int j = k + L2_PF;
                if (j < n)
                    rec_copy<K>(S, P, Q, j, nullptr, nullptr);
                else if (Pn && j - n < n)
                    rec_copy<K>(S, *Pn, Q, j - n, nullptr, nullptr);
            }
            const int st = rec % D;
            if (rec >= (unsigned)D) mbar_wait_producer(&R.empty[st], ((rec / D) + 1) & 1);
            if (PRODUCER_FENCE) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            rec_copy<K>(S, P, Q, k, R.stage(st), &R.full[st]);
        }
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

template <int K>
__device__ __forceinline__ void sub_mul(double (&r)[K], double &rt, const double *c, const LaneSl<K> &L,
                                        const double (&y)[K], double yt)
{
    double cv[K], ct;
    ld_rec(c, L, cv, ct);
#pragma unroll
    for (int k = 0; k < K; k++) r[k] -= cv[k] * y[k];
    rt -= ct * yt;
}

// Ring operands of one line step, loaded one step ahead (software pipeline):
// ld_* only issues the shared-memory loads; fin_* (placed after the current
// line's solve) forms the x-independent constants from them.
template <int K>
struct LineOps {
    double aL[K], aU[K], cp[K], pt[K], c1[K], c2[K];  // chain coefs, in-plane coupling, constants, C1', C2'
    double cpt, ptt, c1t, c2t, nlt, nut;
    LinePrep P;
};

template <int K>
__device__ __forceinline__ void ld_common(LineOps<K> &o, const double *sg, const LaneSl<K> &L, int lane)
{
    ld_rec(sg + (L.desc ? o_nu(K) : o_nl(K)), L, o.aL);
    ld_rec(sg + (L.desc ? o_nl(K) : o_nu(K)), L, o.aU);
    o.nlt = sg[o_nl(K) + L.tw];
    o.nut = sg[o_nu(K) + L.tw];
    ld_rec(sg + rs0_of(K), L, o.cp, o.cpt);
    const double *pp = sg + o_prep(K);
    o.P.p2 = pp[0 * 32 + lane];
    o.P.p3 = pp[1 * 32 + lane];
    o.P.e1 = pp[2 * 32 + lane];
    o.P.e2 = pp[3 * 32 + lane];
    o.P.e3 = pp[4 * 32 + lane];
    o.P.q2 = pp[5 * 32 + lane];
    o.P.q3 = pp[6 * 32 + lane];
    o.P.f1 = pp[7 * 32 + lane];
    o.P.f2 = pp[8 * 32 + lane];
    o.P.f3 = pp[9 * 32 + lane];
    o.P.bex = pp[10 * 32 + lane];
}

// p1, e0, q1, f0 (same expressions as line_prep)
template <int K>
__device__ __forceinline__ void fin_prep(LineOps<K> &o, int lane)
{
    const int s = lane & 15;
    double A0 = 1.0, B0 = 1.0;
#pragma unroll
    for (int k = 0; k < K; k++) {
        A0 *= o.aL[k];
        B0 *= o.aU[k];
    }
    o.P.p1 = s >= 1 ? A0 : 0.0;
    o.P.e0 = s >= 1 ? 1.0 : 0.0;
    o.P.q1 = s <= 14 ? B0 : 0.0;
    o.P.f0 = s <= 14 ? 1.0 : 0.0;
}

// lower sweep: pt = b' - C1' y1 (- C2' y2)   (LOWER3)   or   C1' y1   (UPPER3)
template <int K, bool LOWER3, bool TWO>
__device__ __forceinline__ void ld_lower(LineOps<K> &o, const double *sg, const LaneSl<K> &L, int lane)
{
    ld_common(o, sg, L, lane);
    if (LOWER3) ld_rec(sg + rx_of(K), L, o.pt, o.ptt);
    ld_rec(sg + rs1_of(K), L, o.c1, o.c1t);
    if (TWO) ld_rec(sg + rs2_of(K), L, o.c2, o.c2t);
}
template <int K, bool LOWER3, bool TWO>
__device__ __forceinline__ void fin_lower(LineOps<K> &o, int lane, const double (&v1)[K], double v1t,
                                          const double (&v2)[K], double v2t)
{
    fin_prep(o, lane);
    if (LOWER3) {
#pragma unroll
        for (int k = 0; k < K; k++) o.pt[k] -= o.c1[k] * v1[k];
        o.ptt -= o.c1t * v1t;
        if (TWO) {
#pragma unroll
            for (int k = 0; k < K; k++) o.pt[k] -= o.c2[k] * v2[k];
            o.ptt -= o.c2t * v2t;
        }
    } else {
#pragma unroll
        for (int k = 0; k < K; k++) o.pt[k] = o.c1[k] * v1[k];
        o.ptt = o.c1t * v1t;
    }
}

// upper sweep: pt = xo (UPPER3)
template <int K, bool LOWER3>
__device__ __forceinline__ void ld_upper(LineOps<K> &o, const double *sg, const LaneSl<K> &L, int lane)
{
    ld_common(o, sg, L, lane);
    if (!LOWER3) ld_rec(sg + rx_of(K), L, o.pt, o.ptt);
}

#ifndef NTD_L1PF
#define NTD_L1PF 0
#endif
constexpr int L1PF = NTD_L1PF;
__device__ __forceinline__ void prefetch_l1(const double *p)
{
    asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}

// ---------------- solver: one plane
// SMB: the warp keeps its half of the plane it processed last in shared
// memory (pbuf, lines lo_line.. of the half incl. the twist line): each line
// slot holds the neighbour plane's final x until this plane's lower sweep
// replaces it with the lower-sweep value, which the upper sweep replaces with
// this plane's final x.  The solver then issues no global loads per line.
template <int K, int D, int MODE, bool TWO, bool SMB = false>
__device__ void solve_plane(const SlArrays &S, const PlaneDesc &P, const Seq &Q, int nx, int bar_id, double *ex,
                            int &parity, const Ring<K, D> &R, const LaneSl<K> &L, unsigned &rec,
                            double *pbuf = nullptr)
{
    constexpr int LR = lr_of(K);
    const int lane = threadIdx.x & 31, w2 = Q.w2;
    const int ny = Q.ny, t2 = Q.t2, cnt = Q.cnt, t = (nx - 1) / 2;
    const i64 plr = (i64)ny * LR;  // plane stride in SL
    constexpr bool lower3 = MODE == M_LOWER3;
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
        // line q of this half lives at pbuf + (q - lo_line) * LR
        double *bq = pbuf - (i64)(Q.w2 == 0 ? 0 : Q.t2) * LR;
        xlow = bq;
        if (P.nbuf) y1 = bq;
    }
    const int gL = L.desc ? o_nu(K) : o_nl(K), gU = L.desc ? o_nl(K) : o_nu(K);
    auto srec = [&](int off, int q) { return S.solve + (P.prec + q) * (i64)recd_of(K) + off; };
    double xprev[K], xprevt = 0.0;
#pragma unroll
    for (int k = 0; k < K; k++) xprev[k] = 0.0;
    // ---------------- level-2 lower sweep (ntd_solve.py:147-171)
    // Software-pipelined (PIPE): the ring operands of line i+1 and the
    // x-independent part of its scan constants are loaded while line i
    // solves, so the serial chain per line is cr = pt - cp' xprev and the
    // scans.  The full barrier of record i+2 is tested at the top of step i
    // and its result consumed after the solve (an mbarrier test queues behind
    // the warp's outstanding memory traffic: never block on it per step).
    constexpr bool PIPE = K <= 5;
    double n1[K], n1t = 0.0, n2[K], n2t = 0.0;  // neighbour-plane values, loaded ahead
#pragma unroll
    for (int k = 0; k < K; k++) n1[k] = n2[k] = 0.0;
    auto ld_nbr = [&](int j) {
        ld_rec(y1 + Q.qlow(j) * LR, L, n1, n1t);
        if (TWO) ld_rec(y2 + Q.qlow(j) * LR, L, n2, n2t);
    };
    // L1 prefetch of the x-dependent lines NTD_L1PF steps ahead of their load
    // (these operands are final long before use; an L1 hit keeps the copy of
    // the in-flight load at the top of a step from stalling on L2 latency)
    auto pf_nbr = [&](int j) {
        if constexpr (L1PF > 0) {
            if (j < cnt) {
                prefetch_l1(y1 + Q.qlow(j) * LR + L.base);
                if (TWO) prefetch_l1(y2 + Q.qlow(j) * LR + L.base);
            }
        }
    };
    auto full = [&](unsigned r) { return &R.full[r % D]; };
    auto par = [&](unsigned r) { return (r / D) & 1u; };
    LineOps<K> cur;
    if (cnt > 0) {
        ld_nbr(0);
        if (PIPE) {
            double v1[K], v1t = n1t, v2[K], v2t = n2t;
#pragma unroll
            for (int k = 0; k < K; k++) {
                v1[k] = n1[k];
                v2[k] = n2[k];
            }
            ld_nbr(cnt > 1 ? 1 : 0);
            mbar_wait(full(rec), par(rec));
            ld_lower<K, lower3, TWO>(cur, R.stage(rec % D), L, lane);
            fin_lower<K, lower3, TWO>(cur, lane, v1, v1t, v2, v2t);
            if (WAIT_AHEAD && cnt > 1) mbar_wait(full(rec + 1), par(rec + 1));
        }
    }
#pragma unroll 2  // ping-pong registers: no copies of in-flight loads
    for (int i = 0; i < cnt; i++, rec++) {
        const int st = rec % D;
        TSTAMP(q1);
        double v1[K], v1t = n1t, v2[K], v2t = n2t;
#pragma unroll
        for (int k = 0; k < K; k++) {
            v1[k] = n1[k];
            v2[k] = n2[k];
        }
        LineOps<K> nxo;
        bool ok2 = true;
        if (PIPE) {
            pf_nbr(i + 2 + L1PF);
            ld_nbr(i + 2 < cnt ? i + 2 : cnt - 1);
            if (WAIT_AHEAD)
                ok2 = mbar_test(full(rec + 2), par(rec + 2));
            else if (i + 1 < cnt)
                mbar_wait(full(rec + 1), par(rec + 1));
            ld_lower<K, lower3, TWO>(nxo, R.stage((rec + 1) % D), L, lane);  // unused past the sweep
        } else {
            ld_nbr(i + 1 < cnt ? i + 1 : cnt - 1);
            mbar_wait(full(rec), par(rec));
            ld_lower<K, lower3, TWO>(cur, R.stage(st), L, lane);
            fin_lower<K, lower3, TWO>(cur, lane, v1, v1t, v2, v2t);
        }
        TSTAMP(q2);
        TACC(0, q1, q2);
        double rhs[K], rhst = cur.ptt - cur.cpt * xprevt;  // line 0: xprev = 0
#pragma unroll
        for (int k = 0; k < K; k++) rhs[k] = cur.pt[k] - cur.cp[k] * xprev[k];
        TSTAMP(q3);
        TACC(1, q2, q3);
        double x[K], xt;
        line_solve4<K>(cur.P, nx, t, cur.aL, rhs, cur.aU, rhst, cur.nlt, cur.nut, x, xt);
        TSTAMP(q4);
        TACC(2, q3, q4);
        mbar_arrive(&R.empty[st]);  // every operand of stage st has been consumed
        st_rec(xlow + Q.qlow(i) * LR, L, x, xt);
#pragma unroll
        for (int k = 0; k < K; k++) xprev[k] = x[k];
        xprevt = xt;
        if (PIPE) {
            fin_lower<K, lower3, TWO>(nxo, lane, v1, v1t, v2, v2t);
            if (WAIT_AHEAD && i + 2 < cnt && !ok2) mbar_wait(full(rec + 2), par(rec + 2));
            cur = nxo;
        }
        TSTAMP(q5);
        TACC(3, q4, q5);
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
    // lower-sweep value of the next upper-sweep line, one line ahead: line 0's
    // is the last lower-sweep x
    double ya[K], yat = xprevt;
#pragma unroll
    for (int k = 0; k < K; k++) ya[k] = xprev[k];
    if (PIPE && cnt > 0) {  // first upper-sweep records: loads overlap the twist line
        mbar_wait(full(rec), par(rec));
        ld_upper<K, lower3>(cur, R.stage(rec % D), L, lane);
        fin_prep(cur, lane);
        if (WAIT_AHEAD && cnt > 1) mbar_wait(full(rec + 1), par(rec + 1));
    }
    {
        const int q = t2;
        double aL[K], aU[K], rhs[K], rhst;
        ld_rec(srec(gL, q), L, aL);
        ld_rec(srec(gU, q), L, aU);
        const double nlt = srec(o_nl(K), q)[L.tw], nut = srec(o_nu(K), q)[L.tw];
        if (lower3) {
            ld_rec(S.b + (P.prec + q) * LR, L, rhs, rhst);
            // the neighbours' twist lines: y1 (buffer or global) is plane p-1
            // unless only the upper neighbour exists (descending half)
            const double *ym = SMB && P.nbuf && !P.up ? y1 : xpl - plr;
            const double *yp = SMB && P.nbuf && P.up ? y1 : xpl + plr;
            if (P.hasM) {
                double y[K], yt;
                ld_rec(ym + q * LR, L, y, yt);
                sub_mul(rhs, rhst, srec(o_l3(K), q), L, y, yt);
            }
            if (P.hasP) {
                double y[K], yt;
                ld_rec(yp + q * LR, L, y, yt);
                sub_mul(rhs, rhst, srec(o_u3(K), q), L, y, yt);
            }
        } else {
            double c[K], ct, y[K], yt;
            ld_rec(srec(P.c1, q), L, c, ct);
            ld_rec(y1 + q * LR, L, y, yt);
#pragma unroll
            for (int k = 0; k < K; k++) rhs[k] = c[k] * y[k];
            rhst = ct * yt;
        }
        if (t2 > 0) sub_mul(rhs, rhst, srec(o_l2(K), q), L, xa, xat);
        if (t2 < ny - 1) sub_mul(rhs, rhst, srec(o_u2(K), q), L, xd, xdt);
        const LinePrep PP = line_prep<K>(lane & 15, aL, aU);
        line_solve4<K>(PP, nx, t, aL, rhs, aU, rhst, nlt, nut, xn, xnt);
        if constexpr (SMB) {
            // both warps keep the twist line's final value in their buffers
            double nv[K], nvt = xnt;
#pragma unroll
            for (int k = 0; k < K; k++) nv[k] = xn[k];
            if (!lower3) {
                double xo[K], xot;
                ld_rec(xpl + q * LR, L, xo, xot);
#pragma unroll
                for (int k = 0; k < K; k++) nv[k] = xo[k] - xn[k];
                nvt = xot - xnt;
            }
            if (w2 == 0) st_rec(xpl + q * LR, L, nv, nvt);
            __syncwarp();  // every lane has read the old twist slot (twist element is shared)
            st_rec(xlow + q * LR, L, nv, nvt);
        } else if (w2 == 0) {
            if (lower3) {
                st_rec(xpl + q * LR, L, xn, xnt);
            } else {
                double xo[K], xot, nv[K];
                ld_rec(xpl + q * LR, L, xo, xot);
#pragma unroll
                for (int k = 0; k < K; k++) nv[k] = xo[k] - xn[k];
                st_rec(xpl + q * LR, L, nv, xot - xnt);
            }
        }
    }
    // ---------------- level-2 upper sweep (ntd_solve.py:178-185)
    auto ustep = [&](int i, double (&yb_)[K], double &ybt_) {
        const int st = rec % D;
        double y[K], yt = ybt_;
#pragma unroll
        for (int k = 0; k < K; k++) y[k] = yb_[k];
        if constexpr (L1PF > 0) {
            if (i + 1 + L1PF < cnt) prefetch_l1(xlow + Q.qup(i + 1 + L1PF) * LR + L.base);
        }
        ld_rec(xlow + Q.qup(i + 1 < cnt ? i + 1 : i) * LR, L, yb_, ybt_);  // line i+1 (unconditional)
        LineOps<K> nxo;
        bool ok2 = true;
        if (PIPE) {
            if (WAIT_AHEAD)
                ok2 = mbar_test(full(rec + 2), par(rec + 2));
            else if (i + 1 < cnt)
                mbar_wait(full(rec + 1), par(rec + 1));
            ld_upper<K, lower3>(nxo, R.stage((rec + 1) % D), L, lane);  // unused past the sweep
        } else {
            mbar_wait(full(rec), par(rec));
            ld_upper<K, lower3>(cur, R.stage(st), L, lane);
            fin_prep(cur, lane);
        }
        double bs[K];
#pragma unroll
        for (int k = 0; k < K; k++) bs[k] = cur.cp[k] * xn[k];
        double xs[K], xst;
        line_solve4<K>(cur.P, nx, t, cur.aL, bs, cur.aU, cur.cpt * xnt, cur.nlt, cur.nut, xs, xst);
#pragma unroll
        for (int k = 0; k < K; k++) xn[k] = y[k] - xs[k];
        xnt = yt - xst;
        double nv[K], nvt = xnt;
#pragma unroll
        for (int k = 0; k < K; k++) nv[k] = xn[k];
        if (!lower3) {
#pragma unroll
            for (int k = 0; k < K; k++) nv[k] = cur.pt[k] - xn[k];
            nvt = cur.ptt - xnt;
        }
        mbar_arrive(&R.empty[st]);
        st_rec(xpl + Q.qup(i) * LR, L, nv, nvt);
        if constexpr (SMB) st_rec(xlow + Q.qup(i) * LR, L, nv, nvt);  // (xlow is the buffer)
        if (PIPE) {
            fin_prep(nxo, lane);
            if (WAIT_AHEAD && i + 2 < cnt && !ok2) mbar_wait(full(rec + 2), par(rec + 2));
            cur = nxo;
        }
        rec++;
    };
#pragma unroll 2  // ping-pong registers: no copies of in-flight loads
    for (int i = 0; i < cnt; i++) ustep(i, ya, yat);
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
    extern __shared__ __align__(128) double sl_ring[];
    __shared__ double ex[NP][2 * 2 * (32 * K + 1)];
    __shared__ __align__(8) unsigned long long bars[2 * NP][2 * D];
    constexpr int LR = lr_of(K);
    const i64 sys = NP == 2 ? blockIdx.x : blockIdx.x >> 1;
    if (active && !active[sys]) return;  // both CTAs of a cluster leave together
    const i64 nsl = (i64)nz * ny * LR;
    SlArrays S;
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
    R.base = sl_ring + (size_t)sw * D * stage_of(K);
    // SMB plane buffer of this solver warp: max(t2+1, ny-t2) lines
    const int bl = (ny - 1) / 2 + 1 > ny - (ny - 1) / 2 ? (ny - 1) / 2 + 1 : ny - (ny - 1) / 2;
    double *pbuf = sl_ring + (size_t)2 * NP * D * stage_of(K) + (size_t)sw * bl * LR;
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
    const LaneSl<K> L(lane);
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
    auto produce = [&](int idx) {
        const PlaneDesc P = desc(idx), Pn = desc(idx + 1);
        produce_plane<K, D>(S, P, idx + 1 < nplanes ? &Pn : nullptr, Q, R, rec);
    };
    for (int i = 0; i < nlow; i++) {
        if (producer)
            produce(i);
        else
            solve_plane<K, D, M_LOWER3, false, SMB>(S, desc(i), Q, nx, bar, myex, parity, R, L, rec, pbuf);
    }
    phase_sync();
    if (pair == 0) {
        if (producer) {
            fence_proxy_async();
            produce(nlow);
        } else {
            solve_plane<K, D, M_LOWER3, true, SMB>(S, desc(nlow), Q, nx, bar, myex, parity, R, L, rec, pbuf);
        }
    }
    phase_sync();
    if (producer) fence_proxy_async();  // x (read as xo) was written by generic stores
    for (int i = nlow + ntw; i < nplanes; i++) {
        if (producer)
            produce(i);
        else
            solve_plane<K, D, M_UPPER3, false, SMB>(S, desc(i), Q, nx, bar, myex, parity, R, L, rec, pbuf);
    }
}

}  // namespace sl

template <int K>
int launch_prep_sl_k(double *solve, i64 lines_total, cudaStream_t st);
template <int K>
int launch_apply_sl_k(const double *solve, const double *bsl, double *xsl, double *xssl, const double *zpl, int nx,
                      int ny, int nz, i64 batch, const int32_t *active, cudaStream_t st, int ctas_per_system = 1);

template <int K>
int launch_apply_smb(const double *solve, const double *bsl, double *xsl, double *xssl, const double *zpl, int nx,
                     int ny, int nz, i64 batch, const int32_t *active, cudaStream_t st, int bl)
{
    constexpr int Ds = sl::depth_smb_of(K) >= 2 ? sl::depth_smb_of(K) : 2;
    const size_t smem = (size_t)2 * Ds * sl::stage_of(K) * 8 + (size_t)2 * bl * sl::lr_of(K) * 8;
    cudaError_t e = cudaFuncSetAttribute(sl::k_apply<K, Ds, 1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
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
    e = cudaLaunchKernelEx(&cfg, sl::k_apply<K, Ds, 1, true>, solve, bsl, xsl, xssl, zpl, nx, ny, nz, active);
    if (e != cudaSuccess) {
        ntd::set_error("ntd_apply (cluster)", e);
        return NTD_ELAUNCH;
    }
    return ntd::check_launch("ntd_apply");
}

#define NTD_INSTANTIATE_SL(K)                                                                                     \
    template <>                                                                                                    \
    int launch_prep_sl_k<K>(double *solve, i64 lines_total, cudaStream_t st)                                      \
    {                                                                                                              \
        const i64 threads = lines_total * 32;                                                                      \
        sl::k_prep_sl<K><<<(unsigned)((threads + 255) / 256), 256, 0, st>>>(solve, lines_total);                  \
        return ntd::check_launch("ntd_solve_bands prep");                                                          \
    }                                                                                                              \
    template <>                                                                                                    \
    int launch_apply_sl_k<K>(const double *solve, const double *bsl, double *xsl, double *xssl, const double *zpl,   \
                             int nx, int ny, int nz, i64 batch, const int32_t *active, cudaStream_t st,            \
                             int ctas_per_system)                                                                  \
    {                                                                                                              \
        const int bl_ = (ny - 1) / 2 + 1 > ny - (ny - 1) / 2 ? (ny - 1) / 2 + 1 : ny - (ny - 1) / 2;             \
        if constexpr (sl::depth_smb_of(K) >= 2) {                                                                  \
            if (ctas_per_system == 2 && bl_ <= 16 * K + 1)                                                            \
                return launch_apply_smb<K>(solve, bsl, xsl, xssl, zpl, nx, ny, nz, batch, active, st, bl_);        \
        }                                                                                                          \
        if (ctas_per_system == 2) {                                                                                \
            constexpr int D2 = sl::depth2_of(K);                                                                   \
            const size_t smem2 = (size_t)2 * D2 * sl::stage_of(K) * 8;                                             \
            cudaError_t e2 = cudaFuncSetAttribute(sl::k_apply<K, D2, 1>,                                          \
                                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2);        \
            if (e2 != cudaSuccess) {                                                                               \
                ntd::set_error("ntd_apply smem", e2);                                                              \
                return NTD_ELAUNCH;                                                                                \
            }                                                                                                      \
            cudaLaunchConfig_t cfg = {};                                                                           \
            cfg.gridDim = dim3((unsigned)(2 * batch));                                                             \
            cfg.blockDim = dim3(128);                                                                              \
            cfg.dynamicSmemBytes = smem2;                                                                          \
            cfg.stream = st;                                                                                       \
            cudaLaunchAttribute attr[1];                                                                           \
            attr[0].id = cudaLaunchAttributeClusterDimension;                                                      \
            attr[0].val.clusterDim.x = 2;                                                                          \
            attr[0].val.clusterDim.y = 1;                                                                          \
            attr[0].val.clusterDim.z = 1;                                                                          \
            cfg.attrs = attr;                                                                                      \
            cfg.numAttrs = 1;                                                                                      \
            e2 = cudaLaunchKernelEx(&cfg, sl::k_apply<K, D2, 1>, solve, bsl, xsl, xssl, zpl, nx, ny, nz, active);  \
            if (e2 != cudaSuccess) {                                                                               \
                ntd::set_error("ntd_apply (cluster)", e2);                                                         \
                return NTD_ELAUNCH;                                                                                \
            }                                                                                                      \
            return ntd::check_launch("ntd_apply");                                                                 \
        }                                                                                                          \
        constexpr int D = sl::depth_of(K);                                                                         \
        const size_t smem = (size_t)4 * D * sl::stage_of(K) * 8;                                                   \
        cudaError_t e = cudaFuncSetAttribute(sl::k_apply<K, D, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,    \
                                             (int)smem);                                                           \
        if (e != cudaSuccess) {                                                                                    \
            ntd::set_error("ntd_apply smem", e);                                                                   \
            return NTD_ELAUNCH;                                                                                    \
        }                                                                                                          \
        sl::k_apply<K, D, 2><<<(unsigned)batch, 256, smem, st>>>(solve, bsl, xsl, xssl, zpl, nx, ny, nz, active);  \
        return ntd::check_launch("ntd_apply");                                                                     \
    }
