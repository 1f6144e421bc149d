// blas.cu -- 7-point stencil SpMV and the fused CG vector kernels.
//
// Replaces the reference's _spmv_kernel / spmv / dot / axpy / norm2
// (/root/reference/pkg/src/ntdprecon/banded_core.py:95-147) and the BLAS-1
// steps of pcg (precond_pcg.py:84-119).  The SpMV keeps the reference's
// summation order (dg,-1,-nx,-nxy,+1,+nx,+nxy; banded_core.py:105-117) with
// exactly-rounded multiplies/adds, so it is bitwise equal to the reference.
// Reductions are deterministic fixed-order trees (per-block partials in a
// fixed row assignment, then one block per system sums them in order).
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "common.cuh"
#include "stencil.cuh"

namespace ntd {
static thread_local char g_err[512];
void set_error(const char *where, cudaError_t e)
{
    snprintf(g_err, sizeof(g_err), "%s: %s", where, cudaGetErrorString(e));
}
int check_launch(const char *where)
{
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_error(where, e);
        return NTD_ELAUNCH;
    }
    return NTD_OK;
}

}  // namespace ntd

static constexpr int RED_THREADS = 256;
// Reductions (dot products, A p . p, ||b - A x||^2) keep one partial per warp
// (warp-shuffle tree, no block barriers that would idle the SM at the end of
// each block) over VB(n) virtual blocks per system, summed in fixed order by
// one block per system.  VB depends on n only -- not on the batch, the stream
// or the grid -- so the reduction tree, and every PCG iterate, is the same
// for a system solved alone or in any batch.  VB grows with n (about 8 rows
// per thread) up to 8 blocks per SM, so one large system keeps every SM's
// memory pipeline busy (a fixed 148 blocks per system held a single 350^3
// system at 13% of HBM); at least 8 rows per thread, so a mid-size system
// (128^3: 820 blocks) still fills the GPU.
// at most one wave of the heaviest reduction kernel (k_spmv_dot: 40 registers,
// 6 resident 256-thread blocks per SM), so a lone system's reduction never
// runs a partial second wave (148 * 8 virtual blocks: 52% warps active)
static constexpr int MAX_VB = 148 * 6;
static constexpr int MAX_PARTS = MAX_VB * (RED_THREADS / 32);
static constexpr int STN_UNROLL = 2;  // measured: 1 -> 68%, 2 -> 76%, 4 -> 56% of HBM for spmv+dot (64 systems)
__host__ __device__ __forceinline__ int red_vblocks(i64 n)
{
    const i64 v = (n + 8 * RED_THREADS - 1) / (8 * RED_THREADS);
    return (int)(v < 1 ? 1 : (v > MAX_VB ? MAX_VB : v));
}
// Launched blocks per system: every virtual block for a lone system (its
// rows need the whole GPU's memory pipelines), at most 148 per system in a
// batch (each block then walks several virtual blocks in order; the partials
// -- hence the result -- do not change).  Measured on the 64-system batch:
// 148 blocks per system walking 432 virtual blocks of 8 rows each 65% of
// HBM for spmv+dot, one block per 24-row virtual block 80%.
static unsigned red_grid(i64 n, i64 batch)
{
    const i64 v = red_vblocks(n);
    return (unsigned)(batch == 1 || v < 148 ? v : 148);
}

__device__ __forceinline__ double warp_sum(double v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = add_rn(v, __shfl_xor_sync(FULL_MASK, v, o));
    return v;
}

// Block-level fixed-order tree reduction (deterministic).
__device__ __forceinline__ double block_sum(double v, double *sh)
{
    int tid = threadIdx.x;
    sh[tid] = v;
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
        if (tid < s) sh[tid] = add_rn(sh[tid], sh[tid + s]);
        __syncthreads();
    }
    double r = sh[0];
    __syncthreads();
    return r;
}

// ---------------------------------------------------------------- spmv
__global__ void __launch_bounds__(256) k_spmv(const double *__restrict__ a, const double *__restrict__ x,
                                              double *__restrict__ y, i64 n, i64 nx, i64 nxy,
                                              const int32_t *__restrict__ active)
{
    i64 s = blockIdx.y;
    if (active && !active[s]) return;
    const double *__restrict__ as = a + s * 7 * n;
    const double *__restrict__ xs = x + s * n;
    double *__restrict__ ys = y + s * n;
    for (i64 r = blockIdx.x * (i64)blockDim.x + threadIdx.x; r < n; r += (i64)gridDim.x * blockDim.x)
        ys[r] = spmv_row(as, xs, r, n, nx, nxy);
}


extern "C" int ntd_spmv(const double *a, const double *x, double *y, int64_t nx, int64_t ny,
                        int64_t nz, int64_t batch, const int32_t *active, void *stream)
{
    if (!a || !x || !y || nx < 1 || ny < 1 || nz < 1 || batch < 1) return NTD_EINVAL;
    i64 n = nx * ny * nz;
    dim3 grid(ntd::fill_grid<k_spmv>(n), (unsigned)batch);
    k_spmv<<<grid, 256, 0, (cudaStream_t)stream>>>(a, x, y, n, nx, nx * ny, active);
    NTD_CHECK_LAUNCH("ntd_spmv");
}

// ------------------------------------------------------------ residual
// t = r - A(w [+ v]); optionally z_out = w + v.  numpy: `z = ntd(t); z += w`
// gives z = v + w (elementwise add, commutative in IEEE) and `r - spmv(a, z)`.
template <int NB>
__global__ void __launch_bounds__(256) k_residual(const double *__restrict__ a, const double *__restrict__ r,
                                                  const double *__restrict__ w, const double *__restrict__ v,
                                                  double *__restrict__ z_out, double *__restrict__ t, i64 n,
                                                  i64 nx, i64 nxy, const int32_t *__restrict__ active)
{
    i64 s = blockIdx.y;
    if (active && !active[s]) return;
    const double *__restrict__ as = a + s * NB * n;
    const double *__restrict__ ws = w + s * n;
    const double *__restrict__ rs = r + s * n;
    double *__restrict__ ts = t + s * n;
    if (!v) {
        for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x)
            ts[i] = sub_rn(rs[i], row_of<NB>(as, ws, i, n, nx, nxy));
        return;
    }
    const double *__restrict__ vs = v + s * n;
    double *__restrict__ zs = z_out + s * n;
    for (i64 r0 = blockIdx.x * (i64)blockDim.x + threadIdx.x; r0 < n; r0 += (i64)gridDim.x * blockDim.x) {
        // spmv of z = v + w, z formed on the fly at the 7 taps (bitwise).
#define ZV(idx) add_rn(vs[idx], ws[idx])
        // band values: 7-band layout, or the mirrored upper band (NB == 4)
        const double *d0 = as + (NB == 4 ? 0 : 3 * n);
        const double *lm1 = NB == 4 ? as + n - 1 : as + 2 * n, *lmx = NB == 4 ? as + 2 * n - nx : as + n;
        const double *lmz = NB == 4 ? as + 3 * n - nxy : as;
        const double *up1 = as + (NB == 4 ? n : 4 * n), *upx = as + (NB == 4 ? 2 * n : 5 * n);
        const double *upz = as + (NB == 4 ? 3 * n : 6 * n);
        double zc = ZV(r0);
        double sacc = mul_rn(d0[r0], zc);
        if (r0 >= 1) sacc = add_rn(sacc, mul_rn(lm1[r0], ZV(r0 - 1)));
        if (r0 >= nx) sacc = add_rn(sacc, mul_rn(lmx[r0], ZV(r0 - nx)));
        if (r0 >= nxy) sacc = add_rn(sacc, mul_rn(lmz[r0], ZV(r0 - nxy)));
        if (r0 + 1 < n) sacc = add_rn(sacc, mul_rn(up1[r0], ZV(r0 + 1)));
        if (r0 + nx < n) sacc = add_rn(sacc, mul_rn(upx[r0], ZV(r0 + nx)));
        if (r0 + nxy < n) sacc = add_rn(sacc, mul_rn(upz[r0], ZV(r0 + nxy)));
#undef ZV
        ts[r0] = sub_rn(rs[r0], sacc);
        zs[r0] = zc;
    }
}

template <int NB>
static int residual_nb(const double *a, const double *r, const double *w, const double *v, double *z_out,
                       double *t, int64_t nx, int64_t ny, int64_t nz, int64_t batch, const int32_t *active,
                       void *stream)
{
    if (!a || !r || !w || !t || nx < 1 || ny < 1 || nz < 1 || batch < 1) return NTD_EINVAL;
    if ((v == nullptr) != (z_out == nullptr)) return NTD_EINVAL;
    i64 n = nx * ny * nz;
    dim3 grid(ntd::fill_grid<k_residual<NB>>(n), (unsigned)batch);
    k_residual<NB><<<grid, 256, 0, (cudaStream_t)stream>>>(a, r, w, v, z_out, t, n, nx, nx * ny, active);
    NTD_CHECK_LAUNCH("ntd_residual");
}
extern "C" int ntd_residual(const double *a, const double *r, const double *w, const double *v,
                            double *z_out, double *t, int64_t nx, int64_t ny, int64_t nz, int64_t batch,
                            const int32_t *active, void *stream)
{
    return residual_nb<7>(a, r, w, v, z_out, t, nx, ny, nz, batch, active, stream);
}
extern "C" int ntd_residual_sym(const double *a4, const double *r, const double *w, const double *v,
                                double *z_out, double *t, int64_t nx, int64_t ny, int64_t nz, int64_t batch,
                                const int32_t *active, void *stream)
{
    return residual_nb<4>(a4, r, w, v, z_out, t, nx, ny, nz, batch, active, stream);
}

// ------------------------------------------------------------ symmetric pack
// a4[s] = (A_0, A_+1, A_+nx, A_+nxy); sym_ok[s] is cleared when any mirrored
// pair (A[r][r-d], A[r-d][r]) differs in its bits (signed zeros included), in
// which case the caller keeps the 7-band operator.
__global__ void k_sym_pack(const double *__restrict__ a, double *__restrict__ a4, int32_t *__restrict__ ok, i64 n,
                           i64 nx, i64 nxy)
{
    const i64 s = blockIdx.y;
    const double *__restrict__ as = a + s * 7 * n;
    double *__restrict__ o = a4 + s * 4 * n;
    bool good = true;
    for (i64 r = blockIdx.x * (i64)blockDim.x + threadIdx.x; r < n; r += (i64)gridDim.x * blockDim.x) {
        o[r] = as[3 * n + r];
        o[n + r] = as[4 * n + r];
        o[2 * n + r] = as[5 * n + r];
        o[3 * n + r] = as[6 * n + r];
        auto same = [](double p, double q) { return __double_as_longlong(p) == __double_as_longlong(q); };
        if (r >= 1 && !same(as[2 * n + r], as[4 * n + r - 1])) good = false;
        if (r >= nx && !same(as[n + r], as[5 * n + r - nx])) good = false;
        if (r >= nxy && !same(as[r], as[6 * n + r - nxy])) good = false;
    }
    if (!good) ok[s] = 0;
}

extern "C" int ntd_sym_pack(const double *a, double *a4, int32_t *sym_ok, int64_t nx, int64_t ny, int64_t nz,
                            int64_t batch, void *stream)
{
    if (!a || !a4 || !sym_ok || nx < 1 || ny < 1 || nz < 1 || batch < 1) return NTD_EINVAL;
    i64 n = nx * ny * nz;
    dim3 grid(ntd::fill_grid<k_sym_pack>(n), (unsigned)batch);
    k_sym_pack<<<grid, 256, 0, (cudaStream_t)stream>>>(a, a4, sym_ok, n, nx, nx * ny);
    NTD_CHECK_LAUNCH("ntd_sym_pack");
}

// ----------------------------------------------------------------- dot
// Stage 1: one partial per warp of every virtual block; thread t of virtual
// block vb sums rows vb*T + t, step VB*T (VB = red_vblocks(n)).
__global__ void __launch_bounds__(RED_THREADS) k_dot_partial(const double *__restrict__ x,
                                                             const double *__restrict__ y, double *__restrict__ part,
                                                             i64 n, const int32_t *__restrict__ active)
{
    i64 s = blockIdx.y;
    if (active && !active[s]) return;
    const int VB = red_vblocks(n);
    const double *__restrict__ xs = x + s * n, *__restrict__ ys = y + s * n;
    for (int vb = blockIdx.x; vb < VB; vb += gridDim.x) {
        double acc = 0.0;
#pragma unroll STN_UNROLL
        for (i64 i = vb * (i64)RED_THREADS + threadIdx.x; i < n; i += (i64)VB * RED_THREADS)
            acc = add_rn(acc, mul_rn(xs[i], ys[i]));
        const double wsum = warp_sum(acc);
        if ((threadIdx.x & 31) == 0) part[s * MAX_PARTS + vb * (RED_THREADS / 32) + (threadIdx.x >> 5)] = wsum;
    }
}

// partials of system s (n rows): part[s * MAX_PARTS + 0 .. parts), fixed-order sum
__device__ __forceinline__ double sum_partials(const double *part, i64 s, double *sh, i64 n)
{
    const int nparts = red_vblocks(n) * (RED_THREADS / 32);
    double v = 0.0;
    for (int k = threadIdx.x; k < nparts; k += blockDim.x) v = add_rn(v, part[s * MAX_PARTS + k]);
    return block_sum(v, sh);
}

__global__ void __launch_bounds__(RED_THREADS) k_dot_final(const double *__restrict__ part, double *__restrict__ out,
                                                           int sqrt_out, i64 n, const int32_t *__restrict__ active)
{
    __shared__ double sh[RED_THREADS];
    i64 s = blockIdx.x;
    if (active && !active[s]) return;
    double v = sum_partials(part, s, sh, n);
    if (threadIdx.x == 0) out[s] = sqrt_out ? sqrt(v) : v;
}

extern "C" int64_t ntd_dot_work_doubles(int64_t batch) { return batch * MAX_PARTS; }

static int launch_dot(const double *x, const double *y, double *work, i64 n, i64 batch, const int32_t *active,
                      cudaStream_t st)
{
    dim3 grid(red_grid(n, batch), (unsigned)batch);
    k_dot_partial<<<grid, RED_THREADS, 0, st>>>(x, y, work, n, active);
    return ntd::check_launch("dot_partial");
}

extern "C" int ntd_dot(const double *x, const double *y, double *out, int sqrt_out, int64_t n, int64_t batch,
                       double *work, const int32_t *active, void *stream)
{
    if (!x || !y || !out || !work || n < 0 || batch < 1) return NTD_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    int rc = launch_dot(x, y, work, n, batch, active, st);
    if (rc) return rc;
    k_dot_final<<<(unsigned)batch, RED_THREADS, 0, st>>>(work, out, sqrt_out, n, active);
    NTD_CHECK_LAUNCH("ntd_dot");
}

// ----------------------------------------------------------------- PCG
#define ST(s, k) state[(s) * NTD_ST_N + (k)]
#define FL(s, k) flags[(s) * NTD_FL_N + (k)]

// x = 0, r = b (precond_pcg.py:84,91)
__global__ void k_pcg_init_vec(const double *__restrict__ b, double *__restrict__ x, double *__restrict__ r, i64 n)
{
    i64 s = blockIdx.y;
    for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
        x[s * n + i] = 0.0;
        r[s * n + i] = b[s * n + i];
    }
}

// bnorm = sqrt(b.b); zero rhs short-circuits (precond_pcg.py:86-90)
__global__ void k_pcg_init_final(const double *__restrict__ part, double *__restrict__ state,
                                 int32_t *__restrict__ flags, int32_t *__restrict__ active, double tol, i64 n)
{
    __shared__ double sh[RED_THREADS];
    i64 s = blockIdx.x;
    double v = sum_partials(part, s, sh, n);
    if (threadIdx.x == 0) {
        double bn = sqrt(v);
        for (int k = 0; k < NTD_ST_N; k++) ST(s, k) = 0.0;
        ST(s, NTD_ST_BNORM) = bn;
        ST(s, NTD_ST_TOL) = tol;
        FL(s, NTD_FL_ITERS) = 0;
        if (bn == 0.0) {
            FL(s, NTD_FL_STATUS) = NTD_PCG_CONVERGED;
            FL(s, NTD_FL_ACTIVE) = 0;
        } else {
            FL(s, NTD_FL_STATUS) = NTD_PCG_RUNNING;
            FL(s, NTD_FL_ACTIVE) = 1;
        }
        active[s] = FL(s, NTD_FL_ACTIVE);
    }
}

extern "C" int ntd_pcg_init(const double *b, double *x, double *r, double *state, int32_t *flags,
                            int32_t *active, double tol, int64_t n, int64_t batch, double *work, void *stream)
{
    if (!b || !x || !r || !state || !flags || !active || !work || n < 1 || batch < 1) return NTD_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    dim3 grid(ntd::fill_grid<k_pcg_init_vec>(n), (unsigned)batch);
    k_pcg_init_vec<<<grid, 256, 0, st>>>(b, x, r, n);
    int rc = launch_dot(b, b, work, n, batch, nullptr, st);
    if (rc) return rc;
    k_pcg_init_final<<<(unsigned)batch, RED_THREADS, 0, st>>>(work, state, flags, active, tol, n);
    NTD_CHECK_LAUNCH("ntd_pcg_init");
}

// p = z; rz = r.z (precond_pcg.py:92-94)
__global__ void k_copy(const double *__restrict__ src, double *__restrict__ dst, i64 n,
                       const int32_t *__restrict__ active)
{
    i64 s = blockIdx.y;
    if (active && !active[s]) return;
    for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x)
        dst[s * n + i] = src[s * n + i];
}

__global__ void k_set_scalar(const double *__restrict__ part, double *__restrict__ state, int which, i64 n,
                             const int32_t *__restrict__ active)
{
    __shared__ double sh[RED_THREADS];
    i64 s = blockIdx.x;
    if (active && !active[s]) return;
    double v = sum_partials(part, s, sh, n);
    if (threadIdx.x == 0) ST(s, which) = v;
}

extern "C" int ntd_pcg_start(const double *r, const double *z, double *p, double *state, const int32_t *active,
                             int64_t n, int64_t batch, double *work, void *stream)
{
    if (!r || !z || !p || !state || !work || n < 1 || batch < 1) return NTD_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    dim3 grid(ntd::fill_grid<k_copy>(n), (unsigned)batch);
    k_copy<<<grid, 256, 0, st>>>(z, p, n, active);
    int rc = launch_dot(r, z, work, n, batch, active, st);
    if (rc) return rc;
    k_set_scalar<<<(unsigned)batch, RED_THREADS, 0, st>>>(work, state, NTD_ST_RZ, n, active);
    NTD_CHECK_LAUNCH("ntd_pcg_start");
}

// ap = A p and partial p.ap in one pass
template <int NB>
__global__ void __launch_bounds__(RED_THREADS) k_spmv_dot(const double *__restrict__ a, const double *__restrict__ p,
                                                          double *__restrict__ ap, double *__restrict__ part, i64 n,
                                                          i64 nx, i64 nxy, const int32_t *__restrict__ active)
{
    __shared__ double sh[RED_THREADS];
    i64 s = blockIdx.y;
    if (active && !active[s]) return;
    const double *__restrict__ as = a + s * NB * n, *__restrict__ ps = p + s * n;
    double *__restrict__ aps = ap + s * n;
    // virtual blocks vb = the partials' owners, so the reduction tree (and the
    // result) depends on n only, not on the launched grid
    const int VB = red_vblocks(n);
    for (int vb = blockIdx.x; vb < VB; vb += gridDim.x) {
        double acc = 0.0;
#pragma unroll STN_UNROLL
        for (i64 i = vb * (i64)RED_THREADS + threadIdx.x; i < n; i += (i64)VB * RED_THREADS) {
            double y = row_of<NB>(as, ps, i, n, nx, nxy);
            aps[i] = y;
            acc = add_rn(acc, mul_rn(ps[i], y));
        }
        const double wsum = warp_sum(acc);
        if ((threadIdx.x & 31) == 0) part[s * MAX_PARTS + vb * (RED_THREADS / 32) + (threadIdx.x >> 5)] = wsum;
    }
    (void)sh;
}

// pap, breakdown check, alpha (precond_pcg.py:99-102)
__global__ void k_alpha(const double *__restrict__ part, double *__restrict__ state, int32_t *__restrict__ flags,
                        int32_t *__restrict__ active, i64 n)
{
    __shared__ double sh[RED_THREADS];
    i64 s = blockIdx.x;
    if (!active[s]) return;
    double pap = sum_partials(part, s, sh, n);
    if (threadIdx.x == 0) {
        ST(s, NTD_ST_PAP) = pap;
        if (pap <= 0.0 || !isfinite(pap)) {
            FL(s, NTD_FL_STATUS) = NTD_PCG_BREAKDOWN;
            FL(s, NTD_FL_ACTIVE) = 0;
            active[s] = 0;
        } else {
            ST(s, NTD_ST_ALPHA) = ST(s, NTD_ST_RZ) / pap;
        }
    }
}

template <int NB>
static int spmv_alpha_nb(const double *a, const double *p, double *ap, double *state, int32_t *flags,
                         int32_t *active, int64_t nx, int64_t ny, int64_t nz, int64_t batch, double *work,
                         void *stream)
{
    if (!a || !p || !ap || !state || !flags || !active || !work || batch < 1) return NTD_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    i64 n = nx * ny * nz;
    dim3 grid(red_grid(n, batch), (unsigned)batch);
    k_spmv_dot<NB><<<grid, RED_THREADS, 0, st>>>(a, p, ap, work, n, nx, nx * ny, active);
    int rc = ntd::check_launch("spmv_dot");
    if (rc) return rc;
    k_alpha<<<(unsigned)batch, RED_THREADS, 0, st>>>(work, state, flags, active, n);
    NTD_CHECK_LAUNCH("ntd_pcg_spmv_alpha");
}
extern "C" int ntd_pcg_spmv_alpha(const double *a, const double *p, double *ap, double *state, int32_t *flags,
                                  int32_t *active, int64_t nx, int64_t ny, int64_t nz, int64_t batch, double *work,
                                  void *stream)
{
    return spmv_alpha_nb<7>(a, p, ap, state, flags, active, nx, ny, nz, batch, work, stream);
}
extern "C" int ntd_pcg_spmv_alpha_sym(const double *a4, const double *p, double *ap, double *state,
                                      int32_t *flags, int32_t *active, int64_t nx, int64_t ny, int64_t nz,
                                      int64_t batch, double *work, void *stream)
{
    return spmv_alpha_nb<4>(a4, p, ap, state, flags, active, nx, ny, nz, batch, work, stream);
}

// x = alpha*p + x ; r = (-alpha)*ap + r  (axpy, banded_core.py:139-143: two roundings)
__global__ void k_update_xr(double *__restrict__ x, double *__restrict__ r, const double *__restrict__ p,
                            const double *__restrict__ ap, const double *__restrict__ state, i64 n,
                            const int32_t *__restrict__ active)
{
    i64 s = blockIdx.y;
    if (!active[s]) return;
    double alpha = ST(s, NTD_ST_ALPHA);
    double nalpha = -alpha;
    for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
        i64 k = s * n + i;
        x[k] = add_rn(mul_rn(alpha, p[k]), x[k]);
        r[k] = add_rn(mul_rn(nalpha, ap[k]), r[k]);
    }
}

// ||(-1)*A x + b||^2 partials (precond_pcg.py:106: axpy(-1.0, spmv(a, x), b))
template <int NB>
__global__ void __launch_bounds__(RED_THREADS) k_true_res(const double *__restrict__ a, const double *__restrict__ b,
                                                          const double *__restrict__ x, double *__restrict__ part,
                                                          i64 n, i64 nx, i64 nxy, const int32_t *__restrict__ active)
{
    __shared__ double sh[RED_THREADS];
    i64 s = blockIdx.y;
    if (!active[s]) return;
    const double *__restrict__ as = a + s * NB * n, *__restrict__ xs = x + s * n, *__restrict__ bs = b + s * n;
    const int VB = red_vblocks(n);
    for (int vb = blockIdx.x; vb < VB; vb += gridDim.x) {  // virtual blocks, as in k_spmv_dot
        double acc = 0.0;
#pragma unroll STN_UNROLL
        for (i64 i = vb * (i64)RED_THREADS + threadIdx.x; i < n; i += (i64)VB * RED_THREADS) {
            double res = add_rn(-row_of<NB>(as, xs, i, n, nx, nxy), bs[i]);
            acc = add_rn(acc, mul_rn(res, res));
        }
        const double wsum = warp_sum(acc);
        if ((threadIdx.x & 31) == 0) part[s * MAX_PARTS + vb * (RED_THREADS / 32) + (threadIdx.x >> 5)] = wsum;
    }
    (void)sh;
}

// relres, history, convergence (precond_pcg.py:106-114)
__global__ void k_relres(const double *__restrict__ part, double *__restrict__ state, int32_t *__restrict__ flags,
                         int32_t *__restrict__ active, double *__restrict__ history, i64 max_iters, i64 n)
{
    __shared__ double sh[RED_THREADS];
    i64 s = blockIdx.x;
    if (!active[s]) return;
    double v = sum_partials(part, s, sh, n);
    if (threadIdx.x == 0) {
        double rel = sqrt(v) / ST(s, NTD_ST_BNORM);
        int it = FL(s, NTD_FL_ITERS);
        if (it < max_iters) history[s * max_iters + it] = rel;
        FL(s, NTD_FL_ITERS) = it + 1;
        ST(s, NTD_ST_RELRES) = rel;
        if (!isfinite(rel)) {
            FL(s, NTD_FL_STATUS) = NTD_PCG_NONFINITE;
            FL(s, NTD_FL_ACTIVE) = 0;
            active[s] = 0;
        } else if (rel < ST(s, NTD_ST_TOL)) {
            FL(s, NTD_FL_STATUS) = NTD_PCG_CONVERGED;
            FL(s, NTD_FL_ACTIVE) = 0;
            active[s] = 0;
        }
    }
}

template <int NB>
static int update_residual_nb(const double *a, const double *b, double *x, double *r, const double *p,
                              const double *ap, double *state, int32_t *flags, int32_t *active, double *history,
                              int64_t max_iters, int64_t nx, int64_t ny, int64_t nz, int64_t batch, double *work,
                              void *stream)
{
    if (!a || !b || !x || !r || !p || !ap || !state || !flags || !active || !history || !work) return NTD_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    i64 n = nx * ny * nz;
    dim3 grid(ntd::fill_grid<k_update_xr>(n), (unsigned)batch);
    k_update_xr<<<grid, 256, 0, st>>>(x, r, p, ap, state, n, active);
    int rc = ntd::check_launch("update_xr");
    if (rc) return rc;
    dim3 g2(red_grid(n, batch), (unsigned)batch);
    k_true_res<NB><<<g2, RED_THREADS, 0, st>>>(a, b, x, work, n, nx, nx * ny, active);
    rc = ntd::check_launch("true_res");
    if (rc) return rc;
    k_relres<<<(unsigned)batch, RED_THREADS, 0, st>>>(work, state, flags, active, history, max_iters, n);
    NTD_CHECK_LAUNCH("ntd_pcg_update_residual");
}
extern "C" int ntd_pcg_update_residual(const double *a, const double *b, double *x, double *r, const double *p,
                                       const double *ap, double *state, int32_t *flags, int32_t *active,
                                       double *history, int64_t max_iters, int64_t nx, int64_t ny, int64_t nz,
                                       int64_t batch, double *work, void *stream)
{
    return update_residual_nb<7>(a, b, x, r, p, ap, state, flags, active, history, max_iters, nx, ny, nz, batch,
                                 work, stream);
}
extern "C" int ntd_pcg_update_residual_sym(const double *a4, const double *b, double *x, double *r,
                                           const double *p, const double *ap, double *state, int32_t *flags,
                                           int32_t *active, double *history, int64_t max_iters, int64_t nx,
                                           int64_t ny, int64_t nz, int64_t batch, double *work, void *stream)
{
    return update_residual_nb<4>(a4, b, x, r, p, ap, state, flags, active, history, max_iters, nx, ny, nz, batch,
                                 work, stream);
}

// beta = rz_new / rz ; rz = rz_new  (precond_pcg.py:116-118)
__global__ void k_beta(const double *__restrict__ part, double *__restrict__ state, const int32_t *__restrict__ active,
                       i64 n)
{
    __shared__ double sh[RED_THREADS];
    i64 s = blockIdx.x;
    if (!active[s]) return;
    double rzn = sum_partials(part, s, sh, n);
    if (threadIdx.x == 0) {
        ST(s, NTD_ST_BETA) = rzn / ST(s, NTD_ST_RZ);
        ST(s, NTD_ST_RZ) = rzn;
    }
}

// p = beta*p + z  (axpy(beta, p, z), precond_pcg.py:119)
__global__ void k_update_p(double *__restrict__ p, const double *__restrict__ z, const double *__restrict__ state,
                           i64 n, const int32_t *__restrict__ active)
{
    i64 s = blockIdx.y;
    if (!active[s]) return;
    double beta = ST(s, NTD_ST_BETA);
    for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
        i64 k = s * n + i;
        p[k] = add_rn(mul_rn(beta, p[k]), z[k]);
    }
}

extern "C" int ntd_pcg_direction(const double *r, const double *z, double *p, double *state,
                                 const int32_t *active, int64_t n, int64_t batch, double *work, void *stream)
{
    if (!r || !z || !p || !state || !active || !work) return NTD_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    int rc = launch_dot(r, z, work, n, batch, active, st);
    if (rc) return rc;
    k_beta<<<(unsigned)batch, RED_THREADS, 0, st>>>(work, state, active, n);
    rc = ntd::check_launch("beta");
    if (rc) return rc;
    dim3 grid(ntd::fill_grid<k_update_p>(n), (unsigned)batch);
    k_update_p<<<grid, 256, 0, st>>>(p, z, state, n, active);
    NTD_CHECK_LAUNCH("ntd_pcg_direction");
}

extern "C" const char *ntd_version(void) { return "ntdgpu 0.1 sm_100a"; }
extern "C" const char *ntd_last_error(void) { return ntd::g_err; }
