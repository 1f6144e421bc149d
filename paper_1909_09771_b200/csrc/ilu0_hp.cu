// ilu0_hp.cu -- block ILU0 triangular solves as a hyperplane-synchronous
// wavefront (bitwise the reference's _ilu0_apply_half, ilu0.py:95-114).
//
// Same skewed unit layout as ilu0_skew.cu (a unit = 32 lines of one plane;
// at its local step tau lane L handles cell i = tau - L; coefficient records
// [u][tau][c][lane] from ntd_ilu0_skew_build, guards folded in as zeros), but
// a different schedule.  Unit (plane kk, group h) of a half starts at global
// step s = 32 h + kk; every operand a unit reads at global step T was produced
// at step T - 1:
//     z(i-1)          the lane's own previous value         (register)
//     z(i -/+ nx)     lane L-1 / L+1 of the same unit       (warp shuffle)
//                     lane 31 / 0 of the neighbour group    (shared memory)
//     z(i -/+ nxy)    the same lane of the previous plane   (shared memory)
// so the whole half advances one step per barrier, with every unit's row of
// the previous step double-buffered in shared memory.  A half is one CTA, or a
// thread-block cluster of NC CTAs that split its planes; the row of a CTA's
// last plane is also stored into the next CTA's halo rows (distributed shared
// memory) and the step barrier is the cluster barrier.  The critical path is
// the wavefront length, 32 (G - 1) + planes + nx + 31 steps, instead of the
// progress-word chains of ilu0_skew.cu, whose L2 / DSMEM round trips set the
// step time of small systems (0.24 ms per 32^3 apply) and whose 48 warps per
// half serialise a 350^3 half (30 ms per apply).
//
// Per unit and step a warp loads its next operands one step ahead (one
// register set, reloaded right after use: no copies), so the loads of all its
// units are in flight across the barrier.  Warp w owns units w, w + W, ... of
// its CTA; in the backward sweep the same physical units (so each lane reads
// back the forward result it wrote itself).
#include "common.cuh"

namespace hp {

#ifdef HP_TIMING
#ifndef HP_TIMING_BLOCK
#define HP_TIMING_BLOCK 0
#endif
// per-warp cycle accounting of one CTA (experiments): [warp][0 work, 1 loads, 2 barrier, 3 steps]
__device__ unsigned long long g_hp_timing[32][4];
#define HPT_NOW(v) const long long v = clock64()
#define HPT_ADD(k, val) \
    if (blockIdx.x == HP_TIMING_BLOCK && (threadIdx.x & 31) == 0) g_hp_timing[threadIdx.x >> 5][k] += (unsigned long long)(val)
#else
#define HPT_NOW(v)
#define HPT_ADD(k, val)
#endif

struct Sweep {
    int G, T, nk, kb;   // groups per plane, steps per unit, planes in the half, first plane (absolute)
    int nx, ny;
    i64 nxy;
    int pc0, pc1;       // this CTA's planes [pc0, pc1) (relative to the half, ascending)
    int U;              // units of this CTA
    int rows;           // rows of each step buffer: the largest CTA share + halo + zero row (same in every CTA)
    int S;              // global steps of a sweep
};

__device__ __forceinline__ void cluster_arrive() { asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory"); }
__device__ __forceinline__ void cluster_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }

// store v to the same shared-memory location in CTA `rank` of the cluster
__device__ __forceinline__ void st_remote(double *local_addr, int rank, double v)
{
    unsigned la = (unsigned)__cvta_generic_to_shared(local_addr), ra;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(la), "r"(rank));
    asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(ra), "d"(v) : "memory");
}

// Global-memory link between the CTAs of a half that do not form a cluster
// (more than 16 CTAs, one lone large system).  The boundary plane's row goes
// through a ring of RING slots in global memory whose empty state is a
// sentinel NaN (all bits set; the host fills the rings with it): the value
// is its own signal, so a consumer lane spins on its 8-byte slot until it is
// not the sentinel, uses it and resets the slot -- no fences or flags on the
// critical path.  The only flag is the consumer's progress (published with
// release every few steps), which the producer checks before it reuses a
// slot (RING steps of slack).  The next step's halo is loaded speculatively
// with the operands and re-polled only if it was still empty.  All CTAs of
// the launch are co-resident (a cooperative launch), so the waits resolve.
constexpr int RING = 16;
constexpr int PUBLISH = 4;  // consumer progress published every PUBLISH steps
struct Link {
    double *halo_in;          // ring this CTA reads (RING x G x 32), nullptr: no predecessor
    double *halo_out;         // ring this CTA writes, nullptr: no successor
    unsigned *flag_self;      // this CTA's progress (read by its predecessor)
    const unsigned *flag_succ;
};

__device__ __forceinline__ unsigned ld_acquire(const unsigned *p)
{
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(unsigned *p, unsigned v)
{
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ double ld_relaxed(const double *p)
{
    double v;
    asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed(double *p, double v)
{
    asm volatile("st.relaxed.gpu.global.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}
__device__ __forceinline__ bool is_empty_slot(double v) { return __double_as_longlong(v) == -1ll; }

// One sweep of one half.  buf: [2][rows][32] (rows 0..G-1: halo = the
// previous plane in sweep order, owned by the neighbour CTA; row rows-1:
// zeros; rows is the same in every CTA of the cluster, so a row has the same
// offset in every CTA's buffer).
template <bool FWD, int UPW, int OUT, int PF, bool GL>
__device__ __forceinline__ void sweep(const Sweep &w, const double *__restrict__ coef, const double *__restrict__ in,
                                      double *zf, double *zout, double *accio, double *buf, int nc, int crank,
                                      const Link &lk)
{
    const int lane = threadIdx.x & 31, warp = __shfl_sync(FULL_MASK, (int)(threadIdx.x >> 5), 0), W = blockDim.x >> 5;  // (provably warp-uniform)
    constexpr int NCF = FWD ? 3 : 4;
    constexpr int NOP = FWD ? 4 : ((OUT & 2) ? 6 : 5);  // operands per unit and step
    constexpr int NO = NOP;
    const int G = w.G, Tu = w.T, U = w.U;
    const int rows = w.rows, zrow = w.rows - 1;
    // sweep-order index of this CTA's first plane; the CTA that receives our
    // last plane as its halo (-1: none)
    const int koff = FWD ? w.pc0 : w.nk - w.pc1;
    const int next = FWD ? (crank + 1 < nc ? crank + 1 : -1) : (crank > 0 ? crank - 1 : -1);
    constexpr bool has_zo = !FWD && (OUT & 1), has_ao = !FWD && (OUT & 2);

    int sm[UPW], mm[UPW], rb[UPW], uu[UPW];
    bool own[UPW], jv[UPW];
    // operand sets: step tau uses (and then reloads, for tau + PF) set tau % PF,
    // so a set is never copied while its loads are in flight
    double zprev[UPW], o[PF][UPW][NO];
#pragma unroll
    for (int j = 0; j < UPW; j++) {
        const int mw = warp + j * W;
        own[j] = mw < U;
        const int m = FWD ? mw : U - 1 - mw;  // local unit in sweep order
        mm[j] = m;
        const int kk = koff + m / G, h = m % G;
        sm[j] = 32 * h + kk;
        const int krel = FWD ? kk : w.nk - 1 - kk, g = FWD ? h : G - 1 - h;
        uu[j] = (w.kb + krel) * G + g;  // unit index in the system
        const int line = 32 * g + lane;
        jv[j] = own[j] && line < w.ny;
        rb[j] = (int)(w.nxy * (w.kb + krel) + (i64)w.nx * line - lane);  // natural row of skew row t: rb + t
        zprev[j] = 0.0;
#pragma unroll
        for (int p = 0; p < PF; p++)
#pragma unroll
            for (int c = 0; c < NO; c++) o[p][j][c] = 0.0;
    }
    // operands of skew row t (FWD: t = tau; BWD: t = Tu-1-tau) into d
    auto load = [&](int j, int tau, double *d) {
        const int t = FWD ? tau : Tu - 1 - tau;
        const bool ok = jv[j] && (unsigned)(t - lane) < (unsigned)w.nx;
        const double *c = coef + (uu[j] * Tu + t) * (32 * NCF) + lane;
        d[0] = __ldg(c);
        d[1] = __ldg(c + 32);
        d[2] = __ldg(c + 64);
        if (FWD) {
            d[3] = ok ? __ldg(in + rb[j] + t) : 0.0;  // rhs, gathered from the natural layout
        } else {
            d[3] = __ldg(c + 96);                                     // pivot f3 (1 on empty slots)
            d[4] = __ldcg(zf + (uu[j] * Tu + t) * 32 + lane);         // forward result
            if constexpr (has_ao) d[5] = ok ? accio[rb[j] + t] : 0.0;
        }
    };
    // global-link mode: the halo value of a unit's NEXT step, requested one step ahead (not PF steps
    // like the other operands: every step of look-ahead on the halo is a step of lag between
    // consecutive CTAs of the wavefront, 47 times per sweep at 96^3)
    double hnext[UPW];
#pragma unroll
    for (int j = 0; j < UPW; j++) hnext[j] = __longlong_as_double(-1ll);
    unsigned seen_succ = 0;  // (thread 0) last observed successor progress
    for (int T = -PF; T < w.S; T++) {
        const int cur = T & 1, prv = cur ^ 1;
        double *bc = buf + (size_t)cur * rows * 32, *bp = buf + (size_t)prv * rows * 32;
        // step tau of unit j with operand set op, then the loads of step tau + PF into op
        auto unit_step = [&](int j, int tau, double *op) {
            if (tau >= 0) {
                const int m = mm[j], h = m % G;
                const int t = FWD ? tau : Tu - 1 - tau;
                // neighbour line: lane L-1 (FWD) / L+1 (BWD) of this unit, or the
                // edge lane of the neighbour group's row of the previous step
                const double zn = FWD ? __shfl_up_sync(FULL_MASK, zprev[j], 1) : __shfl_down_sync(FULL_MASK, zprev[j], 1);
                const double ze = bp[(h > 0 ? m + G - 1 : zrow) * 32 + (FWD ? 31 : 0)];
                const double zy = (FWD ? lane == 0 : lane == 31) ? ze : zn;
                // previous plane: row m (the halo rows 0..G-1, or unit m - G); in the
                // global-link mode the halo comes from the predecessor's ring
                double zz;
                if (GL && m < G) {
                    zz = 0.0;
                    if constexpr (GL) {
                        if (lk.halo_in) {
                            double *slot = lk.halo_in + ((T - 1) % RING) * G * 32 + h * 32 + lane;
                            zz = hnext[j];
                            long long spins = 0;
                            while (is_empty_slot(zz)) {
                                zz = ld_relaxed(slot);
                                if (++spins > (1ll << 28)) __trap();
                            }
                            st_relaxed(slot, __longlong_as_double(-1ll));  // empty again
                            // the next step's halo (slot T % RING), speculatively
                            hnext[j] = tau + 1 < Tu ? ld_relaxed(lk.halo_in + (T % RING) * G * 32 + h * 32 + lane)
                                                    : __longlong_as_double(-1ll);
                        }
                    }
                } else {
                    zz = bp[m * 32 + lane];
                }
                double acc = FWD ? op[3] : op[4];
                acc = sub_rn(acc, mul_rn(op[0], zprev[j]));
                acc = sub_rn(acc, mul_rn(op[1], zy));
                acc = sub_rn(acc, mul_rn(op[2], zz));
                double zv;
                if (FWD) {
                    zv = acc;
#ifndef HP_NO_ZF_STORE
                    __stcg(zf + (uu[j] * Tu + t) * 32 + lane, zv);
#endif
                } else {
                    const bool ok = jv[j] && (unsigned)(t - lane) < (unsigned)w.nx;
                    zv = ok ? acc / op[3] : 0.0;
#ifndef HP_NO_OUT_STORE
                    if (ok) {
                        if constexpr (has_zo) zout[rb[j] + t] = zv;
                        if constexpr (has_ao) accio[rb[j] + t] = add_rn(op[5], zv);
                    }
#endif
                }
                zprev[j] = zv;
                bc[(m + G) * 32 + lane] = zv;
                if (GL) {
                    if (lk.halo_out && m >= U - G)
                        st_relaxed(lk.halo_out + (T % RING) * G * 32 + (m - (U - G)) * 32 + lane, zv);
                } else if (next >= 0 && m >= U - G) {
                    st_remote(&bc[(m - (U - G)) * 32 + lane], next, zv);
                }
            }
            if (tau + PF < Tu) load(j, tau + PF, op);
        };
        HPT_NOW(t_w0);
#pragma unroll
        for (int j = 0; j < UPW; j++) {
            const int tau = T - sm[j];
            if (!own[j] || tau < -PF || tau >= Tu) continue;
            // warp-uniform choice of the operand set (registers, not an indexed array)
            const int ph = (tau + PF) % PF;
            if constexpr (PF == 1) {
                unit_step(j, tau, o[0][j]);
            } else if constexpr (PF == 2) {
                if (ph == 0) unit_step(j, tau, o[0][j]);
                else unit_step(j, tau, o[1][j]);
            } else {
                if (ph == 0) unit_step(j, tau, o[0][j]);
                else if (ph == 1) unit_step(j, tau, o[1][j]);
                else unit_step(j, tau, o[2][j]);
            }
        }
        HPT_NOW(t_w1);
        HPT_ADD(0, t_w1 - t_w0);
        if (GL || nc == 1) {
            if (GL && lk.halo_out && T + 1 >= 0) {
                // before slot (T + 1) % RING is reused by the next step: the successor has completed
                // the last step that read it (T + 1 - RING + 1).  Checked by thread 0 ahead of this
                // step's barrier, which then also holds the other warps back: one barrier per step.
                const int need = T + 1 - RING + 2;
                if (threadIdx.x == 0 && need > 0 && seen_succ < (unsigned)need) {
                    long long spins = 0;  // (a protocol error must not hang the GPU: fail the launch)
                    while ((seen_succ = ~ld_acquire(lk.flag_succ)) < (unsigned)need)
                        if (++spins > (1ll << 28)) __trap();
                }
            }
            __syncthreads();
#ifdef HP_TIMING
            { HPT_NOW(t_w2); HPT_ADD(2, t_w2 - t_w1); HPT_ADD(3, 1); }
#endif
            // progress for the predecessor's slot reuse (our slot resets are
            // ordered before it: CTA barrier, then a release by thread 0)
            if (GL && lk.halo_in && threadIdx.x == 0 && T >= 0 && (T % PUBLISH == PUBLISH - 1 || T == w.S - 1))
                st_release(lk.flag_self, ~((unsigned)T + 1));
        } else {
            cluster_arrive();
            cluster_wait();
        }
    }
}

// One sweep (FWD: forward into zf; else backward from zf into z and/or
// acc += z).  grid: 2 * batch * nc CTAs (a cluster of nc CTAs per half).
template <int UPW>
struct HpTraits {
    static constexpr int PF = UPW == 1 ? 3 : (UPW == 2 ? 2 : 1);  // operand sets (steps of look-ahead)
    static constexpr int MAXT = UPW <= 1 ? 768 : 512;     // threads per CTA (register budget)
};

template <bool FWD, int UPW, int OUT, bool GL>
__global__ void __launch_bounds__(HpTraits<UPW>::MAXT, 1)
    k_sweep(const double *__restrict__ coef, const double *__restrict__ r, double *zf, double *z, double *acc,
            i64 split, int nx, int ny, int nz, const int32_t *__restrict__ active, int nc, double *glbuf)
{
    extern __shared__ __align__(16) double hp_buf[];
    const int hb = blockIdx.x / nc, crank = blockIdx.x % nc;
    const i64 sys = hb >> 1;
    const int half = hb & 1;
    if (active && !active[sys]) return;  // every CTA of a cluster leaves together
    Sweep w;
    w.G = (ny + 31) / 32;
    w.T = nx + 31;
    w.nx = nx;
    w.ny = ny;
    w.nxy = (i64)nx * ny;
    const int ks = (int)(split / w.nxy);
    w.kb = half ? ks : 0;
    w.nk = half ? nz - ks : ks;
    if (w.nk <= 0) return;
    w.pc0 = (int)((i64)w.nk * crank / nc);
    w.pc1 = (int)((i64)w.nk * (crank + 1) / nc);
    w.U = (w.pc1 - w.pc0) * w.G;
    w.rows = (w.nk + nc - 1) / nc * w.G + w.G + 1;
    w.S = 32 * (w.G - 1) + w.nk - 1 + w.T;
    const i64 n = w.nxy * nz, per = (i64)nz * w.G * w.T * 32;
    for (int e = threadIdx.x; e < 2 * w.rows * 32; e += blockDim.x) hp_buf[e] = 0.0;
    Link lk = {nullptr, nullptr, nullptr, nullptr};
    if (GL) {
        // glbuf: [batch][2 halves][nc boundaries][RING][G][32] rings, then two sets (forward sweep,
        // backward sweep) of [batch][2][nc] progress words; the host fills all of it with 0xff
        const size_t ring = (size_t)RING * w.G * 32;
        const i64 hs = sys * 2 + half;  // this system half
        double *rings = glbuf + (size_t)hs * nc * ring;
        // progress words are stored complemented (all-ones = no step done), one set per sweep, so a
        // single 0xff fill before the forward sweep prepares the rings (empty sentinel) and both sets;
        // every ring slot is consumed and reset by its reader, so the backward sweep finds them empty
        unsigned *flags = (unsigned *)(glbuf + (size_t)gridDim.x / nc * nc * ring) + (FWD ? 0 : gridDim.x) + hs * nc;
        const int pred = FWD ? crank - 1 : crank + 1, succ = FWD ? crank + 1 : crank - 1;
        // boundary b lies between CTAs b and b + 1
        if (pred >= 0 && pred < nc) lk.halo_in = rings + (size_t)(FWD ? pred : crank) * ring;
        if (succ >= 0 && succ < nc) lk.halo_out = rings + (size_t)(FWD ? crank : succ) * ring;
        lk.flag_self = flags + crank;
        lk.flag_succ = flags + (succ >= 0 && succ < nc ? succ : crank);
    }
    if (GL || nc == 1) {
        __syncthreads();
    } else {
        cluster_arrive();
        cluster_wait();
    }
    sweep<FWD, UPW, OUT, HpTraits<UPW>::PF, GL>(w, coef + sys * per * (FWD ? 3 : 4), FWD ? r + sys * n : nullptr,
                                               zf + sys * per, (OUT & 1) ? z + sys * n : nullptr,
                                               (OUT & 2) ? acc + sys * n : nullptr, hp_buf, nc, crank, lk);
}

}  // namespace hp

// Largest CTA share of a half's units: rows of the step buffers in shared
// memory (2 x (U + G + 1) x 256 B <= 200 KB).
static constexpr int HP_MAX_UNITS = 380;

extern "C" int64_t ntd_ilu0_hp_units(int64_t nx, int64_t ny, int64_t nz, int64_t split)
{
    const i64 nxy = nx * ny;
    if (nx < 1 || ny < 1 || nz < 1 || split % nxy != 0) return 0;
    const i64 ks = split / nxy, G = (ny + 31) / 32;
    const i64 nk = ks > nz - ks ? ks : nz - ks;
    return nk * G;  // units of the larger half
}

extern "C" int ntd_ilu0_hp_apply_ex(const double *coef, int64_t split, const double *r, double *z, double *acc,
                                    double *work, int64_t nx, int64_t ny, int64_t nz, int64_t batch,
                                    const int32_t *active, int64_t ctas_per_half, int64_t warps_per_cta,
                                    int64_t links, void *stream);

extern "C" int ntd_ilu0_hp_apply(const double *coef, int64_t split, const double *r, double *z, double *acc,
                                 double *work, int64_t nx, int64_t ny, int64_t nz, int64_t batch,
                                 const int32_t *active, int64_t ctas_per_half, int64_t warps_per_cta, void *stream)
{
    return ntd_ilu0_hp_apply_ex(coef, split, r, z, acc, work, nx, ny, nz, batch, active, ctas_per_half,
                                warps_per_cta, 0, stream);
}

// links: how the CTAs of a half exchange their boundary planes.  1: a thread-block cluster (<= 16 CTAs,
// DSMEM stores, cluster barrier per step); 2: global-memory rings (cooperative launch, every CTA
// resident: 2 * batch * CTAs <= 148); 0: 2 above 16 CTAs per half, else 1.
extern "C" int ntd_ilu0_hp_apply_ex(const double *coef, int64_t split, const double *r, double *z, double *acc,
                                    double *work, int64_t nx, int64_t ny, int64_t nz, int64_t batch,
                                    const int32_t *active, int64_t ctas_per_half, int64_t warps_per_cta,
                                    int64_t links, void *stream)
{
    if (!coef || !r || !work || (!z && !acc) || nx < 1 || ny < 1 || nz < 1 || batch < 1) return NTD_EINVAL;
    const int nc = (int)ctas_per_half, W = (int)warps_per_cta;
    if (nc < 1 || nc > 74 || W < 1 || W > 24 || links < 0 || links > 2) return NTD_EINVAL;
    if (links == 1 && nc > 16) return NTD_EINVAL;
    const bool gl = nc > 1 && (links == 2 || (links == 0 && nc > 16));
    if (gl && nc > 16 && 2 * batch * nc > 148) return NTD_EINVAL;
    const i64 nxy = nx * ny, G = (ny + 31) / 32, T = nx + 31;
    if (split % nxy != 0) return NTD_ENOTSUP;
    const i64 ks = split / nxy, nk = ks > nz - ks ? ks : nz - ks;
    if (nc > nk) return NTD_EINVAL;
    const i64 umax = (nk + nc - 1) / nc * G;  // largest CTA share
    if (umax > HP_MAX_UNITS) return NTD_ENOTSUP;
    if (nz * G * T * 32 * 4 >= (1ll << 31) || nxy * nz >= (1ll << 31)) return NTD_ENOTSUP;  // 32-bit offsets
    const int upw = (int)((umax + W - 1) / W);
    const size_t smem = (size_t)2 * (umax + G + 1) * 32 * 8;
    const i64 per = nz * G * T * 32;
    // global-link scratch (rings + progress words) in the second half of the
    // work buffer (the skewed kernel's backward array, unused here)
    double *glbuf = work + per * batch;
    const size_t ring_doubles = (size_t)2 * batch * nc * hp::RING * G * 32;
    const int out = (z ? 1 : 0) | (acc ? 2 : 0);
    typedef void (*Kern)(const double *, const double *, double *, double *, double *, i64, int, int, int,
                         const int32_t *, int, double *);
    Kern kf = nullptr, kb = nullptr;
    int maxt = 0;
#define HP_CASE2(U_, GL_)                                                                                  \
    kf = hp::k_sweep<true, U_, 0, GL_>;                                                                    \
    kb = out == 1 ? hp::k_sweep<false, U_, 1, GL_>                                                         \
                  : (out == 2 ? hp::k_sweep<false, U_, 2, GL_> : hp::k_sweep<false, U_, 3, GL_>);          \
    maxt = hp::HpTraits<U_>::MAXT;
#define HP_CASE(U_)                  \
    case U_:                         \
        if (gl) {                    \
            HP_CASE2(U_, true)       \
        } else {                     \
            HP_CASE2(U_, false)      \
        }                            \
        break;
    switch (upw) {
        HP_CASE(1)
        HP_CASE(2)
        HP_CASE(3)
        HP_CASE(4)
        HP_CASE(5)
        HP_CASE(6)
        HP_CASE(7)
        HP_CASE(8)
    default: return NTD_ENOTSUP;
    }
#undef HP_CASE
#undef HP_CASE2
    if (W * 32 > maxt) return NTD_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    for (int pass = 0; pass < 2; pass++) {
        Kern k = pass == 0 ? kf : kb;
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        // global links need every CTA of a half resident at once: up to 16 CTAs a thread-block cluster
        // guarantees that (a plain cluster launch costs less than a cooperative one), above that a
        // cooperative launch
        const bool coop = gl && nc > 16;
        if (e == cudaSuccess && !coop && nc > 8)
            e = cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (e == cudaSuccess && gl && pass == 0)
            e = cudaMemsetAsync(glbuf, 0xff, sizeof(double) * ring_doubles + sizeof(unsigned) * 2 * (2 * batch * nc),
                                st);
        if (e != cudaSuccess) {
            ntd::set_error("ilu0 hp apply attributes", e);
            return NTD_ELAUNCH;
        }
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)(2 * batch * nc));
        cfg.blockDim = dim3(W * 32);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        if (coop) {
            attr[0].id = cudaLaunchAttributeCooperative;
            attr[0].val.cooperative = 1;
        } else {
            attr[0].id = cudaLaunchAttributeClusterDimension;
            attr[0].val.clusterDim.x = nc;
            attr[0].val.clusterDim.y = 1;
            attr[0].val.clusterDim.z = 1;
        }
        cfg.attrs = attr;
        cfg.numAttrs = (gl || nc > 1) ? 1 : 0;
        const double *cf = pass == 0 ? coef : coef + per * batch * 3;
        e = cudaLaunchKernelEx(&cfg, k, cf, r, work, z, acc, (i64)split, (int)nx, (int)ny, (int)nz, active, nc,
                               glbuf);
        if (e != cudaSuccess) {
            ntd::set_error("ilu0 hp apply", e);
            return NTD_ELAUNCH;
        }
        int rc = ntd::check_launch("ilu0 hp apply");
        if (rc) return rc;
    }
    return NTD_OK;
}

#ifdef HP_TIMING
extern "C" int ntd_hp_timing(unsigned long long *out, int reset)
{
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(out, hp::g_hp_timing, sizeof(unsigned long long) * 32 * 4);
    if (reset) {
        static unsigned long long z[32 * 4] = {};
        cudaMemcpyToSymbol(hp::g_hp_timing, z, sizeof(z));
    }
    return 0;
}
#endif
