// ilu0_skew.cu -- block ILU0 triangular solves in the skewed unit layout.
//
// Same arithmetic, in the same order, as ilu0.cu / the reference
// (_ilu0_apply_half, /root/reference/pkg/src/ntdprecon/ilu0.py:95-114), so the
// result is bitwise identical.  What changes is the data layout: a "unit" is
// 32 consecutive grid lines of one plane, processed by one warp as a skewed
// wavefront (lane L handles cell i = tau - L of line 32g + L at step tau), and
// every array the sweep touches is stored per unit as
//     [tau = 0 .. nx+30][lane 0..31]
// so each step reads / writes one contiguous 256-byte row (coalesced; the
// reference-layout version touches 32 different lines per instruction).  The
// index guards of the reference (i-1 >= lo, ...) are folded into the stored
// coefficients (0 where the reference skips the term), so the step is
// branch-free: acc - 0*z == acc for the finite z the sweep produces.
//
// Mapping: one CTA of 24 warps per system half; warps take units round-robin
// in sweep order and follow their neighbour units through progress words in
// shared memory.  Coefficient and input rows are staged by cp.async into a
// per-warp ring 4 steps ahead; the neighbour-unit z values are loaded 2 steps
// ahead into registers.  (Measured on B200, 96^3, one system: 16 warps with
// 4-step register look-ahead 1.42 ms per fwd+bwd apply, this mapping 1.29 ms;
// the sweep is bound by warps in flight, 144 units x 127 steps / 24 warps.)
//
// Applies when the half split is a plane boundary (split % (nx*ny) == 0, true
// for every BASELINE config); ntd_ilu0_apply falls back to ilu0.cu otherwise.
#include <stdio.h>

#include "common.cuh"

namespace skew {

#ifndef SKEW_WARPS
#define SKEW_WARPS 24
#endif
constexpr int WARPS = SKEW_WARPS;
#ifndef SKEW_PF
#define SKEW_PF 2
#endif
constexpr int PF = SKEW_PF;  // steps of look-ahead of the x-dependent operands (registers)

struct Geom {
    int nx, ny, nz, G, T;  // groups per plane, steps per unit (nx + 31)
    i64 nxy, n;
    i64 units;             // nz * G
    __device__ __host__ Geom(int nx_, int ny_, int nz_)
    {
        nx = nx_;
        ny = ny_;
        nz = nz_;
        G = (ny + 31) / 32;
        T = nx + 31;
        nxy = (i64)nx * ny;
        n = nxy * nz;
        units = (i64)nz * G;
    }
    __device__ __host__ i64 skew_size() const { return units * T * 32; }  // per system, per array
};

// unit-local (tau, lane) -> natural row, or -1 when the slot holds no cell
__device__ __forceinline__ i64 slot_row(const Geom &g, i64 u, int tau, int lane)
{
    const i64 k = u / g.G;
    const int grp = (int)(u - k * g.G);
    const int i = tau - lane, j = grp * 32 + lane;
    if (i < 0 || i >= g.nx || j >= g.ny) return -1;
    return i + (i64)g.nx * j + g.nxy * k;
}

// factor -> skewed coefficient records (setup).  Per system:
//   fw[u][tau][3][32] = c2, c1, c0  (forward, guards folded in)
//   bw[u][tau][4][32] = c4, c5, c6, f3  (backward; f3 = 1 on empty slots)
__global__ void k_build(const double *__restrict__ f, double *__restrict__ fw, double *__restrict__ bw, i64 split,
                        int nx, int ny, int nz, i64 batch)
{
    const Geom g(nx, ny, nz);
    const i64 per = g.units * g.T * 32;
    for (i64 e = blockIdx.x * (i64)blockDim.x + threadIdx.x; e < per * batch; e += (i64)gridDim.x * blockDim.x) {
        const i64 s = e / per, el = e - s * per;
        const i64 u = el / (g.T * 32);
        const int rem = (int)(el - u * g.T * 32), tau = rem >> 5, lane = rem & 31;
        const i64 row = slot_row(g, u, tau, lane);
        double c2 = 0.0, c1 = 0.0, c0 = 0.0, c4 = 0.0, c5 = 0.0, c6 = 0.0, f3 = 1.0;
        if (row >= 0) {
            const double *fs = f + s * 7 * g.n;
            const i64 lo = row < split ? 0 : split, hi = row < split ? split : g.n;
            const int i = tau - lane, j = (int)((u % g.G) * 32 + lane);
            if (i >= 1 && row - 1 >= lo) c2 = fs[2 * g.n + row];
            if (j >= 1 && row - nx >= lo) c1 = fs[1 * g.n + row];
            if (row - g.nxy >= lo) c0 = fs[row];
            if (i + 1 < nx && row + 1 < hi) c4 = fs[4 * g.n + row];
            if (j + 1 < ny && row + nx < hi) c5 = fs[5 * g.n + row];
            if (row + g.nxy < hi) c6 = fs[6 * g.n + row];
            f3 = fs[3 * g.n + row];
        }
        double *w = fw + s * per * 3 + (u * g.T + tau) * 96;
        w[lane] = c2;
        w[32 + lane] = c1;
        w[64 + lane] = c0;
        double *b = bw + s * per * 4 + (u * g.T + tau) * 128;
        b[lane] = c4;
        b[32 + lane] = c5;
        b[64 + lane] = c6;
        b[96 + lane] = f3;
    }
}

// natural row of slot (tau, lane) of a unit: base + tau when valid
struct UnitRow {
    i64 base;  // nxy*k + nx*(32*grp + lane) - lane
    bool jv;   // the lane's line exists (32*grp + lane < ny)
};
__device__ __forceinline__ UnitRow unit_row(const Geom &g, i64 u, int lane)
{
    const i64 k = u / g.G;
    const int grp = (int)(u - k * g.G);
    const int j = grp * 32 + lane;
    return UnitRow{g.nxy * k + (i64)g.nx * j - lane, j < g.ny};
}
__device__ __forceinline__ bool slot_valid(const Geom &g, const UnitRow &ur, int tau, int lane)
{
    return ur.jv && tau >= lane && tau - lane < g.nx;
}

#ifdef SKEW_TIMING
__device__ unsigned long long g_skew_timing[4];  // cycles waiting, cycles total, steps, units (block 0 only)
#define SKT_NOW(v) long long v = clock64()
#define SKT_ADD(slot, val) \
    if ((threadIdx.x & 31) == 0 && blockIdx.x == 0) atomicAdd(&g_skew_timing[slot], (unsigned long long)(val))
#else
#define SKT_NOW(v)
#define SKT_ADD(slot, val)
#endif

#ifdef SKEW_CHECK
// first out-of-bounds access: what (1 coef, 2 in_nat, 3 in_skew, 4 acc_in, 5 zp, 6 zop, 7 aop, 8 zz, 9 zy),
// block, warp, lane, offset, count; the access itself is then redirected to the base
__device__ long long g_skc[6];
__device__ __forceinline__ bool skc_bad(const double *p, const double *base, long long count, int what)
{
    if (p >= base && p < base + count) return false;
    if (atomicCAS((unsigned long long *)&g_skc[0], 0ull, (unsigned long long)what) == 0ull) {
        g_skc[1] = blockIdx.x;
        g_skc[2] = threadIdx.x >> 5;
        g_skc[3] = threadIdx.x & 31;
        g_skc[4] = p - base;
        g_skc[5] = count;
    }
    return true;
}
#define SKC(ptr, base, count, what) skc_bad((ptr), (base), (count), what)
#else
#define SKC(ptr, base, count, what)
#endif

// Progress words.  The units of a system half are shared by the warps of
// NC CTAs (a thread-block cluster when NC > 1, so all are co-resident): unit
// position v belongs to cluster-wide warp v % (NC*WARPS), whose CTA holds
// its progress word = v * (T+1) + steps completed (32-bit: units per half *
// (T+1) < 2^32 for every grid the kernels take).  Words are published with
// release and polled with acquire semantics at cluster scope (the z rows they
// guard are global memory, read with L2-coherent loads).
struct Prog {
    volatile unsigned *local;  // this CTA's words (nw)
    int nc, crank, nw;         // CTAs per half, this CTA's rank in the cluster, warps per CTA
};

__device__ __forceinline__ unsigned prog_read(const Prog &P, int gw)
{
    const int cta = gw / P.nw, idx = gw - cta * P.nw;
    if (P.nc == 1) return P.local[idx];
    unsigned la = (unsigned)__cvta_generic_to_shared((const void *)(P.local + idx)), ra, w;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(la), "r"(cta));
    asm volatile("ld.acquire.cluster.shared::cluster.u32 %0, [%1];" : "=r"(w) : "r"(ra) : "memory");
    return w;
}

__device__ __forceinline__ void wait_unit(const Prog &P, int WT, int unit, int steps, int T, unsigned &cw, int &cu)
{
    if (unit < 0) return;
    const unsigned need = (unsigned)unit * (unsigned)(T + 1) + (unsigned)(steps < T ? steps : T);
    if (cu == unit && cw >= need) return;
    unsigned w = 0;
    if ((threadIdx.x & 31) == 0) {
        long long spins = 0;
        do {
            w = prog_read(P, unit % WT);
            // a protocol error must not hang the GPU: fail the launch instead
            if (++spins > (1ll << 26)) __trap();
        } while (w < need);
        if (P.nc == 1)
            __threadfence_block();
        else
            asm volatile("fence.acq_rel.cluster;" ::: "memory");
    }
    w = __shfl_sync(FULL_MASK, w, 0);
    cw = w;
    cu = unit;
}

__device__ __forceinline__ void publish(const Prog &P, int warp, unsigned word)
{
    __syncwarp();
    if ((threadIdx.x & 31) == 0) {
        if (P.nc == 1) {
            __threadfence_block();
            P.local[warp] = word;
        } else {
            asm volatile("fence.acq_rel.cluster;" ::: "memory");
            asm volatile("st.relaxed.cluster.shared::cta.u32 [%0], %1;" ::"r"(
                             (unsigned)__cvta_generic_to_shared((const void *)(P.local + warp))),
                         "r"(word)
                         : "memory");
        }
    }
}

__device__ __forceinline__ void cluster_sync()
{
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// Static operands (coefficient rows, the input row -- gathered from the
// natural layout in the forward sweep, so no separate conversion pass -- and
// the accumulator being updated) are staged into a per-warp shared-memory
// ring by cp.async, PS steps ahead, continuously across the warp's units;
// only the x-dependent operands (z of the neighbour units, gated by their
// progress words) use a register look-ahead of PF steps.  Every address
// walks by a constant stride per step and is recomputed once per unit (the
// sweep is issue-bound: 24 warps share an SM, so instructions per step, not
// latency, set its speed).
#ifndef SKEW_PS
#define SKEW_PS 4
#endif
constexpr int PS = SKEW_PS;  // cp.async ring depth (steps), a power of two
constexpr int ROWS = 6;     // rows per stage: up to 4 coefficient rows, the input row, acc
__host__ __device__ constexpr int ring_doubles() { return WARPS * PS * ROWS * 32; }

__device__ __forceinline__ void cp_async8(double *dst, const double *src)
{
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((unsigned)__cvta_generic_to_shared(dst)),
                 "l"(src)
                 : "memory");
}
// the same with zero fill: nothing is read when !ok (the slot holds no cell)
__device__ __forceinline__ void cp_async8_zf(double *dst, const double *src, bool ok)
{
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"((unsigned)__cvta_generic_to_shared(dst)),
                 "l"(src), "r"(ok ? 8 : 0)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// One half-system sweep.  FWD: units ascending, tau ascending; BWD: mirror.
// FWD: in = rhs in the NATURAL layout (gathered by the stager, 0 on empty
//      slots), z = forward result, skewed.
// BWD: in = forward result, skewed; z = result, skewed (read back by the
//      neighbour units) and also written to the natural-layout outputs:
//      zout[row] = value and/or acc_out[row] += value (precond_pcg.py:64).
template <bool FWD>
__device__ void sweep(const Geom &g, int u_lo, int u_hi, const double *__restrict__ coef, const double *in,
                      double *z, const Prog &prog, double *ring, double *zout, double *acc_out)
{
    const int lane = threadIdx.x & 31, lwarp = __shfl_sync(FULL_MASK, (int)(threadIdx.x >> 5), 0);  // provably warp-uniform
    const int WT = prog.nw * prog.nc, warp = prog.crank * prog.nw + lwarp;  // cluster-wide warp
    const int T = g.T, G = g.G, nx = g.nx;
    constexpr int NC = FWD ? 3 : 4;
    constexpr int dt = FWD ? 1 : -1;  // tau step
    const int nunits = u_hi - u_lo;
    const int nmine = nunits > warp ? (nunits - warp + WT - 1) / WT : 0;  // units of this warp
    auto unit_of = [&](int v) { return FWD ? u_lo + v : u_hi - 1 - v; };
    const int tau0 = FWD ? 0 : T - 1;
    const bool has_zo = zout != nullptr, has_ao = acc_out != nullptr;
    // natural row of (unit u, lane, tau) is rowbase(u) + tau; the lane's slot
    // holds a cell when its line exists and 0 <= tau - lane < nx
    auto rowbase = [&](int u) {
        const int k = u / G, grp = u - k * G;
        return g.nxy * k + (i64)nx * (grp * 32 + lane) - lane;
    };
    auto jvalid = [&](int u) { return (u % G) * 32 + lane < g.ny; };
    // ---- stager: unit round sr, step sq, running pointers
    int sr = 0, sq = 0, stau = tau0;
    unsigned sslot = 0;
    bool sjv = false;
    const double *scs = coef, *sin = in;
    double *sacc = acc_out;
    auto stage_unit = [&]() {
        const int u = unit_of(warp + sr * WT);
        const i64 rb = rowbase(u);
        sjv = jvalid(u);
        stau = tau0;
        scs = coef + ((i64)u * T + tau0) * (32 * NC) + lane;
        sin = FWD ? in + rb + tau0 : in + ((i64)u * T + tau0) * 32 + lane;
        if (!FWD && has_ao) sacc = acc_out + rb + tau0;
    };
    if (nmine > 0) stage_unit();
    auto stage = [&]() {
        if (sr < nmine) {
            double *dst = ring + sslot * (ROWS * 32) + lane;
            const bool ok = sjv && (unsigned)(stau - lane) < (unsigned)nx;
            // empty slots: zero-filled, not read (their coefficients are 0;
            // the backward solve masks its division there)
#pragma unroll
            for (int c = 0; c < NC; c++) {
                const double *pc = scs + c * 32;
#ifdef SKEW_CHECK
                if (SKC(pc, coef, g.skew_size() * NC, 1)) pc = coef;
#endif
                cp_async8_zf(dst + c * 32, pc, ok);
            }
            if (FWD) {
                if (ok) {
                    const double *pi = sin;
#ifdef SKEW_CHECK
                    if (SKC(pi, in, g.n, 2)) pi = in;
#endif
                    cp_async8(dst + 4 * 32, pi);
                }
                else
                    dst[4 * 32] = 0.0;
            } else {
                const double *pi = sin;
#ifdef SKEW_CHECK
                if (SKC(pi, in, g.skew_size(), 3)) pi = in;
#endif
                cp_async8_zf(dst + 4 * 32, pi, ok);
                if (has_ao) {
                    const double *pa = ok ? sacc : acc_out;  // (empty slots: any valid address)
#ifdef SKEW_CHECK
                    if (SKC(pa, acc_out, g.n, 4)) pa = acc_out;
#endif
                    cp_async8_zf(dst + 5 * 32, pa, ok);
                }
            }
            scs += dt * 32 * NC;
            sin += FWD ? 1 : -32;
            sacc += dt;
            stau += dt;
            if (++sq == T) {
                sq = 0;
                if (++sr < nmine) stage_unit();
            }
        }
        sslot = (sslot + 1) & (PS - 1);
        cp_async_commit();  // one group per step, empty past the end
    };
    for (int k = 0; k < PS; k++) stage();
    SKT_NOW(tsw0);
    unsigned cw1 = 0, cw2 = 0;
    int cu1 = -1, cu2 = -1;
    unsigned slot = 0;  // ring slot of the solver's step
    unsigned jsteps = 0;
    for (int v = warp; v < nunits; v += WT) {  // v: position in sweep order
        const int u = unit_of(v);
        const bool has_y = FWD ? (u % G) > 0 : (u % G) < G - 1;  // neighbour unit in the same plane
        const bool has_z = FWD ? (u - G) >= u_lo : (u + G) < u_hi;  // previous plane inside the half
        const int uy = FWD ? u - 1 : u + 1, uz = FWD ? u - G : u + G;
        const int vy = v - 1, vz = v - G;  // their sweep positions
        const bool jv = jvalid(u);
        const bool edge = FWD ? lane == 0 : lane == 31;
        // running pointers at step q = 0 (tau = tau0)
        double *zp = z + ((i64)u * T + tau0) * 32 + lane;
        const double *zzp = z + ((i64)uz * T + tau0) * 32 + lane;
        // neighbour unit's edge lane at tau + 31 (FWD) / tau - 31 (BWD)
        const double *zyp = z + ((i64)uy * T + tau0 + dt * 31) * 32 + (FWD ? 31 : 0);
        const i64 rb = rowbase(u);
        // (pointer arithmetic only; dereferenced only through has_zo / has_ao)
        double *zop = zout + rb + tau0;
        double *aop = acc_out + rb + tau0;
        // register ring of the x-dependent operands for steps q .. q+PF-1
        double rzz[PF], rzy[PF];
        auto load = [&](int slot_, int q) {
            const double *pz = zzp + (i64)q * dt * 32;
#ifdef SKEW_CHECK
            if (has_z && SKC(pz, z, g.skew_size(), 8)) pz = z;
#endif
            rzz[slot_] = has_z ? __ldcg(pz) : 0.0;
            const int ty = FWD ? q + 31 : T - 1 - q - 31;  // neighbour's tau
            const double *py = zyp + (i64)q * dt * 32;
#ifdef SKEW_CHECK
            if (has_y && edge && ty >= 0 && ty < T && SKC(py, z, g.skew_size(), 9)) py = z;
#endif
            rzy[slot_] = (has_y && edge && ty >= 0 && ty < T) ? __ldcg(py) : 0.0;
        };
        // dependencies for the first PF steps
        SKT_NOW(tw0);
        if (has_y) wait_unit(prog, WT, vy, PF + 32, T, cw1, cu1);
        if (has_z) wait_unit(prog, WT, vz, PF, T, cw2, cu2);
        SKT_NOW(tw1);
        SKT_ADD(0, tw1 - tw0);
        SKT_ADD(3, 1);
#pragma unroll
        for (int q = 0; q < PF; q++) load(q, q);
        double zprev = 0.0;
        int tau = tau0;
        for (int q0 = 0; q0 < T; q0 += PF) {
            // operands of steps q0+PF .. q0+2PF-1 become loadable once the
            // neighbours are that far ahead
            if (q0 + PF < T) {
                SKT_NOW(tw2);
                if (has_y) wait_unit(prog, WT, vy, q0 + 2 * PF + 32, T, cw1, cu1);
                if (has_z) wait_unit(prog, WT, vz, q0 + 2 * PF, T, cw2, cu2);
                SKT_NOW(tw3);
                SKT_ADD(0, tw3 - tw2);
            }
#pragma unroll
            for (int d = 0; d < PF; d++) {
                const int q = q0 + d;
                if (q >= T) break;
                cp_async_wait<PS - 1>();  // this lane's copies of this step have landed
                const double *sg = ring + slot * (ROWS * 32) + lane;
                slot = (slot + 1) & (PS - 1);
                const double rin = sg[4 * 32];
                const double zn = FWD ? __shfl_up_sync(FULL_MASK, zprev, 1) : __shfl_down_sync(FULL_MASK, zprev, 1);
                const double zy = edge ? rzy[d] : zn;
                double acc = rin;
                acc = sub_rn(acc, mul_rn(sg[0], zprev));
                acc = sub_rn(acc, mul_rn(sg[32], zy));
                acc = sub_rn(acc, mul_rn(sg[64], rzz[d]));
                const bool valid = jv && (unsigned)(tau - lane) < (unsigned)nx;
                const double zv = FWD ? acc : (valid ? acc / sg[96] : 0.0);
#ifdef SKEW_CHECK
                if (!SKC(zp, z, g.skew_size(), 5))
#endif
                    *zp = zv;
                if (!FWD && valid) {
                    if (has_zo) {
#ifdef SKEW_CHECK
                        if (!SKC(zop, zout, g.n, 6))
#endif
                            *zop = zv;
                    }
                    if (has_ao) {
#ifdef SKEW_CHECK
                        if (!SKC(aop, acc_out, g.n, 7))
#endif
                            *aop = add_rn(sg[5 * 32], zv);
                    }
                }
                zprev = zv;
                zp += dt * 32;
                if (!FWD) {
                    zop += dt;
                    aop += dt;
                }
                tau += dt;
                if (q + PF < T) load(d, q + PF);
                stage();  // refill the ring (each lane reads only its own copies)
                jsteps++;
            }
            if (((q0 / PF) & 1) == 1 || q0 + PF >= T)
                publish(prog, lwarp, (unsigned)v * (T + 1) + (q0 + PF < T ? q0 + PF : T));
        }
        publish(prog, lwarp, (unsigned)v * (T + 1) + T);
    }
    cp_async_wait<0>();
    SKT_NOW(tsw1);
    SKT_ADD(1, tsw1 - tsw0);
    SKT_ADD(2, jsteps);
}

// grid: 2 * batch * nc CTAs; CTA b works on system (b / nc) / 2, half
// (b / nc) % 2, as rank b % nc of its cluster of nc CTAs (nc = 1: no cluster)
__global__ void __launch_bounds__(WARPS * 32) k_apply(const double *__restrict__ fw, const double *__restrict__ bw,
                                                      const double *__restrict__ r, double *zf, double *zb,
                                                      double *z, double *acc, i64 split, int nx, int ny, int nz,
                                                      const int32_t *__restrict__ active, int nc)
{
    extern __shared__ __align__(16) double skew_ring[];
    __shared__ unsigned prog_s[WARPS];
    const Geom g(nx, ny, nz);
    const int hb = blockIdx.x / nc;
    const i64 sys = hb >> 1;
    const int half = hb & 1;
    // every CTA of a cluster takes the same early exits (same system / half)
    if (active && !active[sys]) return;
    const i64 ksplit = split / g.nxy;
    const i64 u_lo = half ? ksplit * g.G : 0, u_hi = half ? g.units : ksplit * g.G;
    if (u_lo >= u_hi) return;
    const i64 per = g.skew_size();
    const double *fws = fw + sys * per * 3, *bws = bw + sys * per * 4;
    const double *rn = r + sys * g.n;
    double *zn = z ? z + sys * g.n : nullptr, *an = acc ? acc + sys * g.n : nullptr;
    double *zfs = zf + sys * per, *zbs = zb + sys * per;
    double *ring = skew_ring + (size_t)__shfl_sync(FULL_MASK, (int)(threadIdx.x >> 5), 0) * PS * ROWS * 32;
    const int nw = blockDim.x >> 5;
    const Prog P{prog_s, nc, (int)(blockIdx.x % nc), nw};
    if (threadIdx.x < nw) prog_s[threadIdx.x] = 0u;
    if (nc > 1) cluster_sync(); else __syncthreads();
    sweep<true>(g, (int)u_lo, (int)u_hi, fws, rn, zfs, P, ring, nullptr, nullptr);
    // the backward sweep reads every unit's forward result
    if (nc > 1) cluster_sync(); else __syncthreads();
    if (threadIdx.x < nw) prog_s[threadIdx.x] = 0u;
    if (nc > 1) cluster_sync(); else __syncthreads();
    sweep<false>(g, (int)u_lo, (int)u_hi, bws, zfs, zbs, P, ring, zn, an);
    // no CTA leaves while another may still poll its progress words
    if (nc > 1) cluster_sync();
}

}  // namespace skew

static unsigned grid_n(i64 total)
{
    i64 b = (total + 255) / 256;
    if (b > 148 * 16) b = 148 * 16;
    return (unsigned)(b > 0 ? b : 1);
}

extern "C" int64_t ntd_ilu0_skew_doubles(int64_t nx, int64_t ny, int64_t nz, int64_t batch, int64_t split)
{
    const skew::Geom g((int)nx, (int)ny, (int)nz);
    if (split % g.nxy != 0) return 0;  // plane-boundary split only
    return g.skew_size() * batch * 7;  // coefficient records (3 + 4 per slot)
}

extern "C" int ntd_ilu0_skew_build(const double *f, double *coef, int64_t split, int64_t nx, int64_t ny, int64_t nz,
                                   int64_t batch, void *stream)
{
    if (!f || !coef || nx < 1 || ny < 1 || nz < 1 || batch < 1) return NTD_EINVAL;
    const skew::Geom g((int)nx, (int)ny, (int)nz);
    if (split % g.nxy != 0) return NTD_ENOTSUP;
    const i64 per = g.skew_size();
    skew::k_build<<<grid_n(per * batch), 256, 0, (cudaStream_t)stream>>>(f, coef, coef + per * batch * 3, split,
                                                                         (int)nx, (int)ny, (int)nz, batch);
    NTD_CHECK_LAUNCH("ntd_ilu0_skew_build");
}

extern "C" int64_t ntd_ilu0_skew_work_doubles(int64_t nx, int64_t ny, int64_t nz, int64_t batch)
{
    const skew::Geom g((int)nx, (int)ny, (int)nz);
    return g.skew_size() * batch * 2;  // forward, backward (skewed)
}

extern "C" int ntd_ilu0_skew_apply_ex(const double *coef, int64_t split, const double *r, double *z, double *acc,
                                      double *work, int64_t nx, int64_t ny, int64_t nz, int64_t batch,
                                      const int32_t *active, int64_t ctas_per_half, int64_t warps_per_cta,
                                      void *stream);

extern "C" int ntd_ilu0_skew_apply(const double *coef, int64_t split, const double *r, double *z, double *acc,
                                   double *work, int64_t nx, int64_t ny, int64_t nz, int64_t batch,
                                   const int32_t *active, void *stream)
{
    return ntd_ilu0_skew_apply_ex(coef, split, r, z, acc, work, nx, ny, nz, batch, active, 1, skew::WARPS, stream);
}

extern "C" int ntd_ilu0_skew_apply_ex(const double *coef, int64_t split, const double *r, double *z, double *acc,
                                      double *work, int64_t nx, int64_t ny, int64_t nz, int64_t batch,
                                      const int32_t *active, int64_t ctas_per_half, int64_t warps_per_cta,
                                      void *stream)
{
    if (ctas_per_half < 1 || ctas_per_half > 8 || warps_per_cta < 1 || warps_per_cta > skew::WARPS)
        return NTD_EINVAL;
    if (!coef || !r || !work || (!z && !acc) || nx < 1 || ny < 1 || nz < 1 || batch < 1) return NTD_EINVAL;
    const skew::Geom g((int)nx, (int)ny, (int)nz);
    if (split % g.nxy != 0) return NTD_ENOTSUP;
    cudaStream_t st = (cudaStream_t)stream;
    const i64 per = g.skew_size();
    double *zf = work, *zb = work + per * batch;
    const int smem = skew::ring_doubles() * 8;
    // the attribute is per function and per device: set it on every call (a
    // host-side driver call, cheap next to the sweep), as the NTD launchers do
    {
        cudaError_t e = cudaFuncSetAttribute(skew::k_apply, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             smem > 120 * 1024 ? smem : 120 * 1024);
        if (e != cudaSuccess) {
            ntd::set_error("ilu0 skew apply smem", e);
            return NTD_ELAUNCH;
        }
    }
    const int nc = (int)ctas_per_half, nw = (int)warps_per_cta;
    if (nc == 1) {
        skew::k_apply<<<(unsigned)(2 * batch), nw * 32, smem, st>>>(coef, coef + per * batch * 3, r, zf, zb, z, acc,
                                                                    split, (int)nx, (int)ny, (int)nz, active, 1);
        NTD_CHECK_LAUNCH("ilu0 skew apply");
    }
    // a cluster spreads its CTAs over SMs only if two cannot share one: ask
    // for more than half of an SM's shared memory
    const int smem_c = smem > 120 * 1024 ? smem : 120 * 1024;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(2 * batch * nc));
    cfg.blockDim = dim3(nw * 32);
    cfg.dynamicSmemBytes = smem_c;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = nc;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, skew::k_apply, coef, (const double *)(coef + per * batch * 3), r, zf,
                                       zb, z, acc, (i64)split, (int)nx, (int)ny, (int)nz, active, nc);
    if (e != cudaSuccess) {
        ntd::set_error("ilu0 skew apply (cluster)", e);
        return NTD_ELAUNCH;
    }
    NTD_CHECK_LAUNCH("ilu0 skew apply");
}

#ifdef SKEW_TIMING
extern "C" int ntd_skew_timing(unsigned long long *out, int reset)
{
    cudaMemcpyFromSymbol(out, skew::g_skew_timing, sizeof(unsigned long long) * 4);
    if (reset) {
        unsigned long long z[4] = {0, 0, 0, 0};
        cudaMemcpyToSymbol(skew::g_skew_timing, z, sizeof(z));
    }
    return 0;
}
#endif

#ifdef SKEW_CHECK
extern "C" int ntd_skew_check(long long *out)
{
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(out, skew::g_skc, sizeof(long long) * 6);
    return 0;
}
#endif
