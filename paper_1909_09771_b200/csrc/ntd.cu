// ntd.cu -- C-ABI entry points of the NTD setup / apply kernels
// (ntd_kernels.cuh); per-K instantiations live in ntd_k<K>.cu so they
// compile in parallel.  K = ceil(nx/32) cells per lane per chain.
#include <algorithm>

#include "ntd_kernels.cuh"
#include "ntd_apply_ts.cuh"
#include "stencil.cuh"

// instantiated K values (ntd_k<K>.cu); a line of nx cells uses the
// smallest instantiated K >= ceil(nx/32).
static const int KS[] = {1, 2, 3, 4, 5, 6, 8, 11, 12, 16};
static constexpr int MAX_K = 16;

static int pick_k(i64 nx)
{
    int need = (int)((nx + 31) / 32);
    for (int k : KS)
        if (k >= need) return k;
    return -1;
}

#define NTD_DISPATCH(FN, ...)            \
    switch (K) {                         \
    case 1: return FN<1>(__VA_ARGS__);   \
    case 2: return FN<2>(__VA_ARGS__);   \
    case 3: return FN<3>(__VA_ARGS__);   \
    case 4: return FN<4>(__VA_ARGS__);   \
    case 5: return FN<5>(__VA_ARGS__);   \
    case 6: return FN<6>(__VA_ARGS__);   \
    case 8: return FN<8>(__VA_ARGS__);   \
    case 11: return FN<11>(__VA_ARGS__); \
    case 12: return FN<12>(__VA_ARGS__); \
    case 16: return FN<16>(__VA_ARGS__); \
    default: return NTD_ENOTSUP;         \
    }

extern "C" int64_t ntd_max_nx(void) { return 32 * MAX_K; }

// Lane-layout (TS) path: K values with an instantiated ring kernel and a ring
// that fits in shared memory.
static int sl_depth(int K)
{
    if (K > 11) return 0;
    return ts::depth_of(K) >= 2 ? ts::depth_of(K) : 0;
}

static i64 sl_doubles(i64 nx, i64 ny, i64 nz)
{
    const int K = pick_k(nx);
    return K > 0 ? ny * nz * (i64)ts::lr_of(K) : 0;
}

extern "C" int64_t ntd_solve_doubles(int64_t nx, int64_t ny, int64_t nz, int64_t batch)
{
    const int K = pick_k(nx);
    if (K <= 0 || !sl_depth(K)) return 0;
    return (int64_t)(ts::recd_of(K) + ts::lr_of(K)) * ny * nz * batch;  // records, then mu of every cell
}

extern "C" int64_t ntd_apply_work_doubles(int64_t nx, int64_t ny, int64_t nz, int64_t batch)
{
    const i64 n = nx * ny * nz * batch;
    const i64 s = sl_doubles(nx, ny, nz) * batch;
    const int K = pick_k(nx);
    // b, x, xs in SL, a zero plane (+ solve records when the caller has none)
    const i64 w = K > 0 ? 3 * s + ny * (i64)ts::lr_of(K) + (i64)(ts::recd_of(K) + ts::lr_of(K)) * ny * nz * batch : 0;
    return w > n ? w : n;
}

extern "C" int ntd_solve_bands(const double *pre, double *solve, int64_t nx, int64_t ny, int64_t nz, int64_t batch,
                               void *stream)
{
    if (!pre || !solve || nx < 1 || ny < 1 || nz < 1 || batch < 1) return NTD_EINVAL;
    const int K = pick_k(nx);
    if (K <= 0 || !sl_depth(K)) return NTD_ENOTSUP;
    const i64 lines = ny * nz;
    cudaStream_t st_ = (cudaStream_t)stream;
    double *mu = solve + (i64)ts::recd_of(K) * lines * batch;
    // padding elements of every record array are exact zeros
    if (cudaMemsetAsync(solve, 0, sizeof(double) * (size_t)ntd_solve_doubles(nx, ny, nz, batch), st_) != cudaSuccess)
        return ntd::check_launch("memset");
    ts::k_solve_ts<<<(unsigned)((lines * batch + 127) / 128), 128, 0, st_>>>(pre, solve, mu, (int)nx, lines, K, batch);
    int rc = ntd::check_launch("ntd_solve_bands");
    if (rc) return rc;
    switch (K) {
#define PREPCASE(KK) \
    case KK: return launch_prep_ts_k<KK>(solve, lines * batch, (cudaStream_t)stream);
        PREPCASE(1) PREPCASE(2) PREPCASE(3) PREPCASE(4) PREPCASE(5) PREPCASE(6) PREPCASE(8) PREPCASE(11)
#undef PREPCASE
    default: return NTD_ENOTSUP;
    }
}

static unsigned grid_for(i64 total)
{
    i64 blocks = (total + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    return (unsigned)(blocks > 0 ? blocks : 1);
}

extern "C" int ntd_apply_ex(const double *pre, const double *solve, const double *b, double *x, double *work,
                            int64_t nx, int64_t ny, int64_t nz, int64_t batch, const int32_t *active,
                            int64_t ctas_per_system, void *stream);

extern "C" int ntd_apply(const double *pre, const double *solve, const double *b, double *x, double *work,
                         int64_t nx, int64_t ny, int64_t nz, int64_t batch, const int32_t *active, void *stream)
{
    return ntd_apply_ex(pre, solve, b, x, work, nx, ny, nz, batch, active, 1, stream);
}

static int apply_impl(const double *pre, const double *solve, const double *b, double *x, double *work, int64_t nx,
                      int64_t ny, int64_t nz, int64_t batch, const int32_t *active, int64_t ctas_per_system,
                      bool direct, void *stream)
{
    if (!pre || !b || !x || !work || nx < 1 || ny < 1 || nz < 1 || batch < 1) return NTD_EINVAL;
    if (ctas_per_system != 1 && ctas_per_system != 2) return NTD_EINVAL;
    const int K = pick_k(nx);
    const int depth = K > 0 ? sl_depth(K) : 0;
    const bool aligned = ((uintptr_t)work % 16 == 0) && (!solve || (uintptr_t)solve % 16 == 0);
    cudaStream_t st = (cudaStream_t)stream;
    if (depth && aligned && !direct) {
        const i64 lines = ny * nz, s = sl_doubles(nx, ny, nz) * batch;
        double *bsl = work, *xsl = work + s, *xssl = work + 2 * s, *zpl = work + 3 * s;
        const i64 zn = ny * (i64)ts::lr_of(K);
        if (!solve) {
            double *sv = zpl + zn;
            int rc = ntd_solve_bands(pre, sv, nx, ny, nz, batch, stream);
            if (rc) return rc;
            solve = sv;
        }
        // the missing level-3 neighbour of the first/last plane reads zeros
        if (cudaMemsetAsync(zpl, 0, sizeof(double) * zn, st) != cudaSuccess) return ntd::check_launch("memset");
        ts::k_to_ts<<<grid_for(s), 256, 0, st>>>(b, solve + (i64)ts::recd_of(K) * lines * batch, bsl, (int)nx, lines, K,
                                                 batch);
        int rc = ntd::check_launch("ntd_apply to_sl");
        if (rc) return rc;
        switch (K) {
#define SLCASE(KK)                                                                                                \
    case KK:                                                                                                       \
        rc = launch_apply_ts_k<KK>(solve, bsl, xsl, xssl, zpl, (int)nx, (int)ny, (int)nz, batch, active, st,     \
                                   (int)ctas_per_system);                                                          \
        break;
            SLCASE(1) SLCASE(2) SLCASE(3) SLCASE(4) SLCASE(5) SLCASE(6) SLCASE(8) SLCASE(11)
#undef SLCASE
        default: return NTD_ENOTSUP;
        }
        if (rc) return rc;
        ts::k_from_ts<<<grid_for(nx * lines * batch), 256, 0, st>>>(xsl, x, (int)nx, lines, K, batch, active);
        return ntd::check_launch("ntd_apply from_sl");
    }
    NTD_DISPATCH(launch_apply_k, pre, b, x, work, (int)nx, (int)ny, (int)nz, batch, active, st);
}

extern "C" int ntd_apply_ex(const double *pre, const double *solve, const double *b, double *x, double *work,
                            int64_t nx, int64_t ny, int64_t nz, int64_t batch, const int32_t *active,
                            int64_t ctas_per_system, void *stream)
{
    return apply_impl(pre, solve, b, x, work, nx, ny, nz, batch, active, ctas_per_system, false, stream);
}

extern "C" int ntd_apply_direct(const double *pre, const double *b, double *x, double *work, int64_t nx, int64_t ny,
                                int64_t nz, int64_t batch, const int32_t *active, void *stream)
{
    return apply_impl(pre, nullptr, b, x, work, nx, ny, nz, batch, active, 1, true, stream);
}

// ------------------------------------------------------------------ fused
// The combined preconditioner's two residuals (precond_pcg.py:58-63) read /
// write the NTD apply's slot-layout buffers directly, so the apply needs no
// layout conversion passes:
//   t' = (r - A w) m  -> b' of the apply (k_to_sl's b m, same rounding)
//   z = x + w, t = r - A z with x read from the apply's slot-layout result
// Both keep the reference summation order (bitwise equal to ntd_residual on
// the natural-layout vectors).
template <int NB>
__global__ void __launch_bounds__(256) k_residual_to_sl(const double *__restrict__ a, const double *__restrict__ mu,
                                                        const double *__restrict__ r, const double *__restrict__ w,
                                                        double *__restrict__ bsl, i64 n, int nx, i64 nxy, int K,
                                                        const int32_t *__restrict__ active)
{
    const i64 s = blockIdx.y;
    if (active && !active[s]) return;
    const int LR = ts::lr_of(K);
    const i64 lines = n / nx;
    const double *__restrict__ as = a + s * NB * n, *__restrict__ ws = w + s * n, *__restrict__ rs = r + s * n;
    const double *__restrict__ ms = mu + s * lines * LR;
    double *__restrict__ bs = bsl + s * lines * LR;
    for (i64 r0 = blockIdx.x * (i64)blockDim.x + threadIdx.x; r0 < n; r0 += (i64)gridDim.x * blockDim.x) {
        const double t = sub_rn(rs[r0], row_of<NB>(as, ws, r0, n, nx, nxy));
        const unsigned line = (unsigned)r0 / (unsigned)nx;
        const int i = (int)(r0 - (i64)line * nx);
        const i64 e = (i64)line * LR + ts::ts_index(i, K);
        bs[e] = t * ms[e];
    }
}

template <int NB>
__global__ void __launch_bounds__(256) k_residual_from_sl(const double *__restrict__ a, const double *__restrict__ r,
                                                          const double *__restrict__ w, const double *__restrict__ xsl,
                                                          double *__restrict__ z_out, double *__restrict__ t, i64 n,
                                                          int nx, i64 nxy, int ny, int K,
                                                          const int32_t *__restrict__ active)
{
    const i64 s = blockIdx.y;
    if (active && !active[s]) return;
    const int LR = ts::lr_of(K);
    const i64 lines = n / nx, plr = (i64)ny * LR;
    const double *__restrict__ as = a + s * NB * n, *__restrict__ ws = w + s * n, *__restrict__ rs = r + s * n, *__restrict__ xs = xsl + s * lines * LR;
    double *__restrict__ zs = z_out + s * n, *__restrict__ ts = t + s * n;
    const double *d0 = as + (NB == 4 ? 0 : 3 * n);
    const double *lm1 = NB == 4 ? as + n - 1 : as + 2 * n, *lmx = NB == 4 ? as + 2 * n - nx : as + n;
    const double *lmz = NB == 4 ? as + 3 * n - nxy : as;
    const double *up1 = as + (NB == 4 ? n : 4 * n), *upx = as + (NB == 4 ? 2 * n : 5 * n);
    const double *upz = as + (NB == 4 ? 3 * n : 6 * n);
    for (i64 r0 = blockIdx.x * (i64)blockDim.x + threadIdx.x; r0 < n; r0 += (i64)gridDim.x * blockDim.x) {
        const unsigned line = (unsigned)r0 / (unsigned)nx;
        const int i = (int)(r0 - (i64)line * nx);
        const i64 lb = (i64)line * LR;
        const int sc = ts::ts_index(i, K);
        // x at the 7 taps (cell i-1 / i+1 wrap to the neighbouring line, where
        // the band value is an exact zero: same operands as the natural layout)
        const i64 pm1 = i > 0 ? lb + ts::ts_index(i - 1, K) : lb - LR + ts::ts_index(nx - 1, K);
        const i64 pp1 = i < nx - 1 ? lb + ts::ts_index(i + 1, K) : lb + LR + ts::ts_index(0, K);
#define ZV(idx, pos) add_rn(xs[pos], ws[idx])
        const double zc = ZV(r0, lb + sc);
        double sacc = mul_rn(d0[r0], zc);
        if (r0 >= 1) sacc = add_rn(sacc, mul_rn(lm1[r0], ZV(r0 - 1, pm1)));
        if (r0 >= nx) sacc = add_rn(sacc, mul_rn(lmx[r0], ZV(r0 - nx, lb - LR + sc)));
        if (r0 >= nxy) sacc = add_rn(sacc, mul_rn(lmz[r0], ZV(r0 - nxy, lb - plr + sc)));
        if (r0 + 1 < n) sacc = add_rn(sacc, mul_rn(up1[r0], ZV(r0 + 1, pp1)));
        if (r0 + nx < n) sacc = add_rn(sacc, mul_rn(upx[r0], ZV(r0 + nx, lb + LR + sc)));
        if (r0 + nxy < n) sacc = add_rn(sacc, mul_rn(upz[r0], ZV(r0 + nxy, lb + plr + sc)));
#undef ZV
        ts[r0] = sub_rn(rs[r0], sacc);
        zs[r0] = zc;
    }
}

static bool slot_path(i64 nx, const double *work, const double *solve, int *K_out)
{
    const int K = pick_k(nx);
    const bool aligned = ((uintptr_t)work % 16 == 0) && (!solve || (uintptr_t)solve % 16 == 0);
    *K_out = K;
    return K > 0 && sl_depth(K) && aligned && solve;
}

extern "C" int ntd_residual_to_slot(const double *a, int64_t bands, const double *solve, const double *r,
                                    const double *w, double *work, int64_t nx, int64_t ny, int64_t nz, int64_t batch,
                                    const int32_t *active, void *stream)
{
    if (!a || !solve || !r || !w || !work || nx < 1 || ny < 1 || nz < 1 || batch < 1) return NTD_EINVAL;
    if (bands != 4 && bands != 7) return NTD_EINVAL;
    const int K = pick_k(nx);
    if (K <= 0 || !sl_depth(K) || nx * ny * nz >= (1ll << 31)) return NTD_ENOTSUP;
    const i64 n = nx * ny * nz;
    const double *pre = solve + (i64)ts::recd_of(K) * ny * nz * batch;  // mu of every cell (lane layout)
    dim3 grid(bands == 4 ? ntd::fill_grid<k_residual_to_sl<4>>(n) : ntd::fill_grid<k_residual_to_sl<7>>(n),
              (unsigned)batch);
    if (bands == 4)
        k_residual_to_sl<4><<<grid, 256, 0, (cudaStream_t)stream>>>(a, pre, r, w, work, n, (int)nx, nx * ny, K, active);
    else
        k_residual_to_sl<7><<<grid, 256, 0, (cudaStream_t)stream>>>(a, pre, r, w, work, n, (int)nx, nx * ny, K, active);
    return ntd::check_launch("ntd_residual_to_slot");
}

extern "C" int ntd_apply_slot_ex(const double *solve, double *work, int64_t nx, int64_t ny, int64_t nz,
                                 int64_t batch, const int32_t *active, int64_t ctas_per_system, void *stream);

extern "C" int ntd_apply_slot(const double *solve, double *work, int64_t nx, int64_t ny, int64_t nz, int64_t batch,
                              const int32_t *active, void *stream)
{
    return ntd_apply_slot_ex(solve, work, nx, ny, nz, batch, active, 1, stream);
}

extern "C" int ntd_apply_slot_ex(const double *solve, double *work, int64_t nx, int64_t ny, int64_t nz,
                                 int64_t batch, const int32_t *active, int64_t ctas_per_system, void *stream)
{
    if (!solve || !work || nx < 1 || ny < 1 || nz < 1 || batch < 1) return NTD_EINVAL;
    if (ctas_per_system != 1 && ctas_per_system != 2) return NTD_EINVAL;
    int K;
    if (!slot_path(nx, work, solve, &K)) return NTD_ENOTSUP;
    cudaStream_t st = (cudaStream_t)stream;
    const i64 s = sl_doubles(nx, ny, nz) * batch;
    double *bsl = work, *xsl = work + s, *xssl = work + 2 * s, *zpl = work + 3 * s;
    const i64 zn = ny * (i64)ts::lr_of(K);
    if (cudaMemsetAsync(zpl, 0, sizeof(double) * zn, st) != cudaSuccess) return ntd::check_launch("memset");
    switch (K) {
#define SLCASE(KK) \
    case KK:                                                                                                       \
        return launch_apply_ts_k<KK>(solve, bsl, xsl, xssl, zpl, (int)nx, (int)ny, (int)nz, batch, active, st,    \
                                     (int)ctas_per_system);
        SLCASE(1) SLCASE(2) SLCASE(3) SLCASE(4) SLCASE(5) SLCASE(6) SLCASE(8) SLCASE(11)
#undef SLCASE
    default: return NTD_ENOTSUP;
    }
}

extern "C" int ntd_residual_from_slot(const double *a, int64_t bands, const double *work, const double *r,
                                      const double *w, double *z_out, double *t, int64_t nx, int64_t ny, int64_t nz,
                                      int64_t batch, const int32_t *active, void *stream)
{
    if (!a || !work || !r || !w || !z_out || !t || nx < 1 || ny < 1 || nz < 1 || batch < 1) return NTD_EINVAL;
    if (bands != 4 && bands != 7) return NTD_EINVAL;
    const int K = pick_k(nx);
    if (K <= 0 || !sl_depth(K) || nx * ny * nz >= (1ll << 31)) return NTD_ENOTSUP;
    const i64 n = nx * ny * nz, s = sl_doubles(nx, ny, nz) * batch;
    const double *xsl = work + s;
    dim3 grid(bands == 4 ? ntd::fill_grid<k_residual_from_sl<4>>(n) : ntd::fill_grid<k_residual_from_sl<7>>(n),
              (unsigned)batch);
    if (bands == 4)
        k_residual_from_sl<4><<<grid, 256, 0, (cudaStream_t)stream>>>(a, r, w, xsl, z_out, t, n, (int)nx, nx * ny,
                                                                      (int)ny, K, active);
    else
        k_residual_from_sl<7><<<grid, 256, 0, (cudaStream_t)stream>>>(a, r, w, xsl, z_out, t, n, (int)nx, nx * ny,
                                                                      (int)ny, K, active);
    return ntd::check_launch("ntd_residual_from_slot");
}

extern "C" int64_t ntd_factor_work_doubles(int64_t nx, int64_t ny, int64_t nz, int64_t batch)
{
    (void)nz;
    return batch * 2 * S_PER_PAIR * nx * ny;
}

extern "C" int ntd_factor(const double *a, double *pre, double *work, int64_t *status, int64_t nx, int64_t ny,
                          int64_t nz, int64_t batch, void *stream)
{
    if (!a || !pre || !work || !status || nx < 1 || ny < 1 || nz < 1 || batch < 1) return NTD_EINVAL;
    int K = pick_k(nx);
    NTD_DISPATCH(launch_factor_k, a, pre, work, status, (int)nx, (int)ny, (int)nz, batch, (cudaStream_t)stream);
}

