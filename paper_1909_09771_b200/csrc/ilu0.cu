// ilu0.cu -- block ILU0 factor and triangular solves, bitwise equal to the
// reference (/root/reference/pkg/src/ntdprecon/ilu0.py).
//
// Each half [lo,hi) of a system is one CTA.  Natural-order substitution is
// exactly reproduced by a skewed wavefront: a "unit" is 32 consecutive grid
// lines of one plane, one lane per line; at step tau lane L handles cell
// i = tau - L of its line.  The x-dependency (i-1) stays in the lane's
// register, the y-dependency (same i, line j-1) comes from lane L-1 by shuffle
// (lane 0: from the previous unit through memory), the z-dependency (previous
// plane) from memory.  Units are distributed round-robin over the CTA's warps
// and ordered by per-warp progress words in shared memory, so every cell sees
// exactly the operands, in exactly the order, of the reference's row loop.
// Requires the BandedMatrix zero pattern (no coupling across line / plane
// boundaries, banded_core.py:39-42), which the Python layer validates.
#include "common.cuh"

static constexpr int ILU_WARPS = 16;
static constexpr int PUB = 4;  // publish progress every PUB steps

struct SweepGeom {
    i64 n, lo, hi, nxy;
    int nx, ny, G, S;  // groups per plane, steps per unit
    i64 klo, khi;
    int units;
};

__device__ __forceinline__ SweepGeom make_geom(i64 n, i64 lo, i64 hi, int nx, int ny)
{
    SweepGeom g;
    g.n = n;
    g.lo = lo;
    g.hi = hi;
    g.nx = nx;
    g.ny = ny;
    g.nxy = (i64)nx * ny;
    g.G = (ny + 31) / 32;
    g.S = nx + 31;
    g.klo = lo / g.nxy;
    g.khi = (hi - 1) / g.nxy;
    g.units = (int)(g.khi - g.klo + 1) * g.G;
    return g;
}

// progress word: unit * (S+1) + steps completed
__device__ __forceinline__ void wait_progress(volatile unsigned long long *prog, int W, int unit, int steps,
                                              int S, unsigned long long &cache_word, int &cache_unit)
{
    if (unit < 0) return;
    unsigned long long need = (unsigned long long)unit * (S + 1) + (unsigned long long)(steps < S ? steps : S);
    if (cache_unit == unit && cache_word >= need) return;
    int lane = threadIdx.x & 31;
    unsigned long long w = 0;
    if (lane == 0) {
        do {
            w = prog[unit % W];
        } while (w < need);
        __threadfence_block();
    }
    w = __shfl_sync(FULL_MASK, w, 0);
    __syncwarp();
    cache_word = w;
    cache_unit = unit;
}

__device__ __forceinline__ void publish(volatile unsigned long long *prog, int warp, unsigned long long word)
{
    __syncwarp();
    if ((threadIdx.x & 31) == 0) {
        __threadfence_block();
        prog[warp] = word;
    }
}

// ------------------------------------------------------------ sweeps
// FWD: z_i = ((r_i - f2 z_{i-1}) - f1 z_{i-nx}) - f0 z_{i-nxy}   (ilu0.py:97-105)
// BWD: z_i = (((z_i - f4 z_{i+1}) - f5 z_{i+nx}) - f6 z_{i+nxy}) / f3   (ilu0.py:106-114)
template <bool FWD>
__device__ void ilu_sweep(const SweepGeom &g, const double *__restrict__ f, const double *__restrict__ rin,
                          double *z, double *acc_out, volatile unsigned long long *prog, unsigned long long base_word)
{
    const int lane = threadIdx.x & 31, warp = __shfl_sync(FULL_MASK, (int)(threadIdx.x >> 5), 0), W = blockDim.x >> 5;
    const i64 n = g.n, nxy = g.nxy;
    const int nx = g.nx, ny = g.ny, S = g.S, G = g.G;
    const double *fa = FWD ? f + 2 * n : f + 4 * n;  // x coupling (f2 | f4)
    const double *fb = FWD ? f + n : f + 5 * n;      // y coupling (f1 | f5)
    const double *fc = FWD ? f : f + 6 * n;          // z coupling (f0 | f6)
    const double *f3 = f + 3 * n;
    unsigned long long cw1 = 0, cw2 = 0;
    int cu1 = -1, cu2 = -1;
    for (int u = warp; u < g.units; u += W) {
        int pi = u / G, grp = u % G;
        i64 k = FWD ? g.klo + pi : g.khi - pi;
        int jl = grp * 32 + lane;  // line within the sweep order
        int j = FWD ? jl : ny - 1 - jl;
        double zprev = 0.0;
        for (int tau = 0; tau < S; tau++) {
            if ((tau % PUB) == 0) {
                // unit u-1 (same plane, lines before): lane 31 must be past cell
                // tau+PUB-1 -> its step tau+PUB-1+31 done; unit u-G: step tau+PUB done.
                if (grp > 0) wait_progress(prog, W, u - 1, tau + PUB + 31, S, cw1, cu1);
                if (pi > 0) wait_progress(prog, W, u - G, tau + PUB, S, cw2, cu2);
                if (tau > 0) publish(prog, warp, (unsigned long long)u * (S + 1) + tau);
            }
            int il = tau - lane;  // cell index in sweep order
            int i = FWD ? il : nx - 1 - il;
            bool cell_ok = (il >= 0) && (il < nx) && (jl < ny);
            i64 row = cell_ok ? (i + (i64)nx * j + nxy * k) : 0;
            bool in_half = cell_ok && row >= g.lo && row < g.hi;
            double zy = __shfl_up_sync(FULL_MASK, zprev, 1);
            double zval = 0.0;
            if (in_half) {
                double acc = FWD ? rin[row] : z[row];
                if (FWD) {
                    if (i >= 1 && row - 1 >= g.lo) acc = sub_rn(acc, mul_rn(fa[row], zprev));
                    if (j >= 1 && row - nx >= g.lo) {
                        double v = (lane == 0) ? z[row - nx] : zy;
                        acc = sub_rn(acc, mul_rn(fb[row], v));
                    }
                    if (row - nxy >= g.lo) acc = sub_rn(acc, mul_rn(fc[row], z[row - nxy]));
                    zval = acc;
                } else {
                    if (i + 1 < nx && row + 1 < g.hi) acc = sub_rn(acc, mul_rn(fa[row], zprev));
                    if (j + 1 < ny && row + nx < g.hi) {
                        double v = (lane == 0) ? z[row + nx] : zy;
                        acc = sub_rn(acc, mul_rn(fb[row], v));
                    }
                    if (row + nxy < g.hi) acc = sub_rn(acc, mul_rn(fc[row], z[row + nxy]));
                    zval = acc / f3[row];
                    if (acc_out) acc_out[row] = add_rn(acc_out[row], zval);
                }
                z[row] = zval;
            }
            zprev = zval;
        }
        publish(prog, warp, (unsigned long long)u * (S + 1) + S);
    }
}

__global__ void __launch_bounds__(ILU_WARPS * 32) k_ilu0_apply(const double *__restrict__ f, i64 split,
                                                              const double *__restrict__ r, double *z,
                                                              double *acc_out, int nx, int ny, int nz,
                                                              const int32_t *__restrict__ active)
{
    __shared__ unsigned long long prog[ILU_WARPS];
    i64 sys = blockIdx.x >> 1;
    int half = blockIdx.x & 1;
    if (active && !active[sys]) return;
    i64 n = (i64)nx * ny * nz;
    i64 lo = half ? split : 0, hi = half ? n : split;
    if (lo >= hi) return;
    SweepGeom g = make_geom(n, lo, hi, nx, ny);
    const double *fs = f + sys * 7 * n;
    const double *rs = r + sys * n;
    double *zs = z + sys * n;
    double *as = acc_out ? acc_out + sys * n : nullptr;
    if (threadIdx.x < ILU_WARPS) prog[threadIdx.x] = 0ull;
    __syncthreads();
    ilu_sweep<true>(g, fs, rs, zs, nullptr, prog, 0);
    __syncthreads();
    __threadfence_block();
    if (threadIdx.x < ILU_WARPS) prog[threadIdx.x] = 0ull;
    __syncthreads();
    ilu_sweep<false>(g, fs, rs, zs, as, prog, 0);
}

extern "C" int ntd_ilu0_apply(const double *f, int64_t split, const double *r, double *z, double *acc,
                              int64_t nx, int64_t ny, int64_t nz, int64_t batch, const int32_t *active,
                              void *stream)
{
    i64 n = nx * ny * nz;
    if (!f || !r || !z || nx < 1 || ny < 1 || nz < 1 || batch < 1 || split < 0 || split > n) return NTD_EINVAL;
    k_ilu0_apply<<<(unsigned)(2 * batch), ILU_WARPS * 32, 0, (cudaStream_t)stream>>>(f, split, r, z, acc, (int)nx,
                                                                                      (int)ny, (int)nz, active);
    NTD_CHECK_LAUNCH("ntd_ilu0_apply");
}

// ------------------------------------------------------------ factor
// IKJ elimination of one row on the original band pattern (ilu0.py:38-83).
// fr[0..6]: the row's current entries (in/out).  Neighbour rows k=i-d for
// d = nxy, nx, 1 supply their final U entries uk[d][0..3] = f3,f4,f5,f6.
__device__ __forceinline__ void ikj_row(double (&fr)[7], const double (&orig)[7], i64 i, i64 lo, i64 hi, i64 nx,
                                        i64 nxy, const double (&u_z)[4], const double (&u_y)[4],
                                        const double (&u_x)[4])
{
#pragma unroll
    for (int t = 0; t < 3; t++) {
        i64 d = t == 0 ? nxy : (t == 1 ? nx : 1);
        i64 k = i - d;
        if (k < lo || orig[t] == 0.0) continue;
        const double(&uk)[4] = t == 0 ? u_z : (t == 1 ? u_y : u_x);
        double fac = fr[t] / uk[0];
        fr[t] = fac;
#pragma unroll
        for (int s = 0; s < 3; s++) {
            i64 du = s == 0 ? 1 : (s == 1 ? nx : nxy);
            double uv = uk[1 + s];
            if (uv == 0.0) continue;
            i64 jj = k + du;
            if (jj >= hi) continue;
            i64 dj = jj - i;
            double upd = mul_rn(fac, uv);
            if (dj == 0) fr[3] = sub_rn(fr[3], upd);
            else if (dj == 1 && orig[4] != 0.0) fr[4] = sub_rn(fr[4], upd);
            else if (dj == nx && orig[5] != 0.0) fr[5] = sub_rn(fr[5], upd);
            else if (dj == nxy && orig[6] != 0.0) fr[6] = sub_rn(fr[6], upd);
            else if (dj == -1 && orig[2] != 0.0) fr[2] = sub_rn(fr[2], upd);
            else if (dj == -nx && orig[1] != 0.0) fr[1] = sub_rn(fr[1], upd);
            else if (dj == -nxy && orig[0] != 0.0) fr[0] = sub_rn(fr[0], upd);
        }
    }
}

__global__ void __launch_bounds__(ILU_WARPS * 32) k_ilu0_factor(const double *__restrict__ a, double *f, i64 split,
                                                               int64_t *status, int nx, int ny, int nz)
{
    __shared__ unsigned long long prog[ILU_WARPS];
    i64 sys = blockIdx.x >> 1;
    int half = blockIdx.x & 1;
    i64 n = (i64)nx * ny * nz;
    i64 lo = half ? split : 0, hi = half ? n : split;
    if (lo >= hi) return;
    SweepGeom g = make_geom(n, lo, hi, nx, ny);
    const double *as = a + sys * 7 * n;
    double *fs = f + sys * 7 * n;
    const i64 nxy = g.nxy;
    if (threadIdx.x < ILU_WARPS) prog[threadIdx.x] = 0ull;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = __shfl_sync(FULL_MASK, (int)(threadIdx.x >> 5), 0), W = blockDim.x >> 5;
    const int S = g.S, G = g.G;
    unsigned long long cw1 = 0, cw2 = 0;
    int cu1 = -1, cu2 = -1;
    i64 bad = -1;
    for (int u = warp; u < g.units; u += W) {
        int pi = u / G, grp = u % G;
        i64 k = g.klo + pi;
        int j = grp * 32 + lane;
        double ux[4] = {0, 0, 0, 0};
        for (int tau = 0; tau < S; tau++) {
            if ((tau % PUB) == 0) {
                if (grp > 0) wait_progress(prog, W, u - 1, tau + PUB + 31, S, cw1, cu1);
                if (pi > 0) wait_progress(prog, W, u - G, tau + PUB, S, cw2, cu2);
                if (tau > 0) publish(prog, warp, (unsigned long long)u * (S + 1) + tau);
            }
            int i = tau - lane;
            bool cell_ok = (i >= 0) && (i < nx) && (j < ny);
            i64 row = cell_ok ? (i + (i64)nx * j + nxy * k) : 0;
            bool in_half = cell_ok && row >= lo && row < hi;
            double uy[4];
#pragma unroll
            for (int q = 0; q < 4; q++) uy[q] = __shfl_up_sync(FULL_MASK, ux[q], 1);
            double nu[4] = {0, 0, 0, 0};
            if (in_half) {
                double fr[7], orig[7];
#pragma unroll
                for (int b = 0; b < 7; b++) {
                    orig[b] = as[b * n + row];
                    fr[b] = fs[b * n + row];
                }
                double uz[4] = {1, 0, 0, 0}, uyy[4] = {1, 0, 0, 0}, uxx[4] = {1, 0, 0, 0};
                if (row - nxy >= lo) {
#pragma unroll
                    for (int q = 0; q < 4; q++) uz[q] = fs[(3 + q) * n + row - nxy];
                }
                if (j >= 1 && row - nx >= lo) {
                    if (lane == 0) {
#pragma unroll
                        for (int q = 0; q < 4; q++) uyy[q] = fs[(3 + q) * n + row - nx];
                    } else {
#pragma unroll
                        for (int q = 0; q < 4; q++) uyy[q] = uy[q];
                    }
                }
                if (i >= 1 && row - 1 >= lo) {
#pragma unroll
                    for (int q = 0; q < 4; q++) uxx[q] = ux[q];
                }
                ikj_row(fr, orig, row, lo, hi, nx, nxy, uz, uyy, uxx);
#pragma unroll
                for (int b = 0; b < 7; b++) fs[b * n + row] = fr[b];
                double piv = fr[3];
                if ((piv == 0.0 || !isfinite(piv)) && (bad < 0 || row < bad)) bad = row;
#pragma unroll
                for (int q = 0; q < 4; q++) nu[q] = fr[3 + q];
            }
#pragma unroll
            for (int q = 0; q < 4; q++) ux[q] = nu[q];
        }
        publish(prog, warp, (unsigned long long)u * (S + 1) + S);
    }
    if (bad >= 0) {
        atomicMin((unsigned long long *)&status[sys * 3 + 2], (unsigned long long)bad);
        status[sys * 3 + 0] = 1;
    }
}

// split-crossing couplings dropped in the copy (ilu0.py:126-131,148-149)
__global__ void k_ilu0_init(const double *__restrict__ a, double *__restrict__ f, i64 split, int64_t *status,
                            int nx, int ny, int nz)
{
    i64 sys = blockIdx.y;
    i64 n = (i64)nx * ny * nz, nxy = (i64)nx * ny;
    const i64 offs[7] = {-nxy, -(i64)nx, -1, 0, 1, nx, nxy};
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        status[sys * 3 + 0] = 0;
        status[sys * 3 + 1] = -1;
        status[sys * 3 + 2] = (int64_t)0x7fffffffffffffffLL;
    }
    for (i64 r = blockIdx.x * (i64)blockDim.x + threadIdx.x; r < n; r += (i64)gridDim.x * blockDim.x) {
#pragma unroll
        for (int b = 0; b < 7; b++) {
            i64 d = offs[b];
            double v = a[sys * 7 * n + b * n + r];
            bool drop = (d > 0 && r >= split - d && r < split) || (d < 0 && r >= split && r < split - d);
            f[sys * 7 * n + b * n + r] = drop ? 0.0 : v;
        }
    }
}

extern "C" int ntd_ilu0_factor(const double *a, double *f, int64_t split, int64_t *status, int64_t nx, int64_t ny,
                               int64_t nz, int64_t batch, void *stream)
{
    i64 n = nx * ny * nz;
    if (!a || !f || !status || nx < 1 || ny < 1 || nz < 1 || batch < 1 || split < 1 || split > n)
        return NTD_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    i64 blocks = (n + 255) / 256;
    if (blocks > 1184) blocks = 1184;
    k_ilu0_init<<<dim3((unsigned)blocks, (unsigned)batch), 256, 0, st>>>(a, f, split, status, (int)nx, (int)ny,
                                                                       (int)nz);
    int rc = ntd::check_launch("ilu0_init");
    if (rc) return rc;
    k_ilu0_factor<<<(unsigned)(2 * batch), ILU_WARPS * 32, 0, st>>>(a, f, split, status, (int)nx, (int)ny,
                                                                     (int)nz);
    NTD_CHECK_LAUNCH("ntd_ilu0_factor");
}
