// vec.cu -- the reference's public vector helpers that sit beside the PCG hot
// path: axpy (banded_core.py:139-143) and chain_bidiagonal_solve
// (ntd_solve.py:272-300 with the lane-composed recurrence _chain_scaled,
// ntd_solve.py:20-64).  Both are bitwise restatements (exactly rounded
// multiplies/adds in the reference's order).
#include "common.cuh"

// out = alpha*x + y: numpy's `alpha * x + y` rounds the product, then the sum.
__global__ void k_axpy(double alpha, const double *__restrict__ x, const double *__restrict__ y,
                       double *__restrict__ out, i64 n)
{
    for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x)
        out[i] = add_rn(mul_rn(alpha, x[i]), y[i]);
}

extern "C" int ntd_axpy(double alpha, const double *x, const double *y, double *out, int64_t n, void *stream)
{
    if (n < 0 || (n > 0 && (!x || !y || !out))) return NTD_EINVAL;
    if (n == 0) return NTD_OK;
    i64 blocks = (n + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    k_axpy<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(alpha, x, y, out, n);
    NTD_CHECK_LAUNCH("ntd_axpy");
}

// One chain per thread: x[p] = (rhs[p] - off[p]*x[p-step]) * dr[p] walked
// p = lo, lo+step, .. (m = n cells), lanes > 1 composing equal chunks as
// affine maps x_new = a*x_prev + c (aw/cw scratch of n doubles per chain),
// stitching the lane carries in order and walking the remainder
// sequentially -- _chain_scaled (ntd_solve.py:20-64) operation for operation.
__global__ void k_chain(const double *__restrict__ dr, const double *__restrict__ off,
                        const double *__restrict__ rhs, double *__restrict__ x, double *__restrict__ aw,
                        double *__restrict__ cw, i64 m, int backward, int lanes, i64 chains)
{
    const i64 c = blockIdx.x * (i64)blockDim.x + threadIdx.x;
    if (c >= chains) return;
    dr += c * m;
    off += c * m;
    rhs += c * m;
    x += c * m;
    aw += c * m;
    cw += c * m;
    const i64 lo = backward ? m - 1 : 0;
    const i64 step = backward ? -1 : 1;
    if (lanes <= 1 || m < 2 * (i64)lanes) {
        double xp = 0.0;
        i64 p = lo;
        for (i64 t = 0; t < m; t++, p += step) {
            xp = mul_rn(sub_rn(rhs[p], mul_rn(off[p], xp)), dr[p]);
            x[p] = xp;
        }
        return;
    }
    const i64 chunk = m / lanes;
    for (int l = 0; l < lanes; l++) {
        const i64 base = l * chunk;
        i64 p = lo + base * step;
        double a = mul_rn(-off[p], dr[p]);
        aw[base] = a;
        cw[base] = mul_rn(rhs[p], dr[p]);
        for (i64 t = 1; t < chunk; t++) {
            p += step;
            a = mul_rn(-off[p], dr[p]);
            aw[base + t] = mul_rn(a, aw[base + t - 1]);
            cw[base + t] = add_rn(mul_rn(a, cw[base + t - 1]), mul_rn(rhs[p], dr[p]));
        }
    }
    double carry = 0.0;
    for (int l = 0; l < lanes; l++) {
        const i64 base = l * chunk;
        for (i64 t = 0; t < chunk; t++) x[lo + (base + t) * step] = add_rn(mul_rn(aw[base + t], carry), cw[base + t]);
        carry = add_rn(mul_rn(aw[base + chunk - 1], carry), cw[base + chunk - 1]);
    }
    double xp = carry;
    i64 p = lo + lanes * chunk * step;
    for (i64 t = lanes * chunk; t < m; t++, p += step) {
        xp = mul_rn(sub_rn(rhs[p], mul_rn(off[p], xp)), dr[p]);
        x[p] = xp;
    }
}

extern "C" int64_t ntd_chain_work_doubles(int64_t n, int64_t chains) { return 2 * n * chains; }

extern "C" int ntd_chain_solve(const double *diag_recip, const double *offdiag, const double *b, double *x,
                               double *work, int64_t n, int64_t chains, int64_t backward, int64_t lanes,
                               void *stream)
{
    if (n < 0 || chains < 1 || lanes < 1 || (backward != 0 && backward != 1)) return NTD_EINVAL;
    if (n == 0) return NTD_OK;
    if (!diag_recip || !offdiag || !b || !x || !work) return NTD_EINVAL;
    const unsigned blocks = (unsigned)((chains + 63) / 64);
    k_chain<<<blocks, 64, 0, (cudaStream_t)stream>>>(diag_recip, offdiag, b, x, work, work + n * chains, n,
                                                     (int)backward, (int)lanes, chains);
    NTD_CHECK_LAUNCH("ntd_chain_solve");
}
