/*
 * ntd_oracle.c -- CPU restatement of the reference NTD-PCG path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker and the CPU
 * baseline ("port") for bench.py's reference arm.  Nothing in the product
 * package (paper_1909_09771_b200/) may link, load or call it.
 *
 * It restates, in plain C, the arithmetic of the reference numba kernels of
 * `ntdprecon` (/root/reference/pkg/src/ntdprecon), operation for operation and
 * in the same evaluation order, so that with -ffp-contract=off it reproduces
 * the reference bit for bit (pinned by tests/test_oracle_golden.py against
 * fixtures generated from the real reference by tests/golden/gen_golden.py).
 * The only non-bitwise part is the PCG dot products, which the reference
 * delegates to OpenBLAS ddot (banded_core.py:133-147); here they are a plain
 * left-to-right sum.
 *
 * Band layout (reference banded_core.py:44): data[7][N], rows
 *   0:-nxy 1:-nx 2:-1 3:0 4:+1 5:+nx 6:+nxy.
 * Preconditioner layout: l1,u1,l2,u2,l3,u3,m_recip (ntd_factor.py:461).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef int64_t i64;

/* ---------------------------------------------------------------- spmv */
/* banded_core.py:95-118 (_spmv_kernel): fixed order dg,-1,-nx,-nxy,+1,+nx,+nxy */
void orc_spmv(const double *data, const double *x, double *y, i64 n, i64 nx,
              i64 nxy, int nthreads)
{
    const double *lo3 = data, *lo2 = data + n, *lo1 = data + 2 * n;
    const double *dg = data + 3 * n, *up1 = data + 4 * n, *up2 = data + 5 * n,
                 *up3 = data + 6 * n;
    (void)nthreads;
#pragma omp parallel for schedule(static) num_threads(nthreads > 0 ? nthreads : 1)
    for (i64 r = 0; r < n; r++) {
        double s = dg[r] * x[r];
        if (r >= 1) s += lo1[r] * x[r - 1];
        if (r >= nx) s += lo2[r] * x[r - nx];
        if (r >= nxy) s += lo3[r] * x[r - nxy];
        if (r + 1 < n) s += up1[r] * x[r + 1];
        if (r + nx < n) s += up2[r] * x[r + nx];
        if (r + nxy < n) s += up3[r] * x[r + nxy];
        y[r] = s;
    }
}

/* ------------------------------------------------------- chain kernels */
/* ntd_solve.py:20-64 (_chain_scaled) */
static void chain_scaled(double *x, const double *dr, const double *off,
                         const double *rhs, i64 lo, i64 hi, i64 step,
                         double x_init, int lanes, double *aw, double *cw)
{
    i64 m = (hi - lo) * step + 1;
    if (m <= 0) return;
    if (lanes <= 1 || m < 2 * (i64)lanes) {
        double xp = x_init;
        i64 p = lo;
        for (i64 it = 0; it < m; it++) {
            xp = (rhs[p] - off[p] * xp) * dr[p];
            x[p] = xp;
            p += step;
        }
        return;
    }
    i64 chunk = m / lanes;
    for (int l = 0; l < lanes; l++) {
        i64 base = l * chunk;
        i64 p = lo + base * step;
        double a = -off[p] * dr[p];
        aw[base] = a;
        cw[base] = rhs[p] * dr[p];
        for (i64 t = 1; t < chunk; t++) {
            p += step;
            a = -off[p] * dr[p];
            aw[base + t] = a * aw[base + t - 1];
            cw[base + t] = a * cw[base + t - 1] + rhs[p] * dr[p];
        }
    }
    double carry = x_init;
    for (int l = 0; l < lanes; l++) {
        i64 base = l * chunk;
        for (i64 t = 0; t < chunk; t++)
            x[lo + (base + t) * step] = aw[base + t] * carry + cw[base + t];
        carry = aw[base + chunk - 1] * carry + cw[base + chunk - 1];
    }
    double xp = carry;
    i64 p = lo + lanes * chunk * step;
    for (i64 it = lanes * chunk; it < m; it++) {
        xp = (rhs[p] - off[p] * xp) * dr[p];
        x[p] = xp;
        p += step;
    }
}

/* ntd_solve.py:67-104 (_chain_unit) */
static void chain_unit(double *x, const double *dr, const double *off, i64 lo,
                       i64 hi, i64 step, double x_init, int lanes, double *aw,
                       double *cw)
{
    i64 m = (hi - lo) * step + 1;
    if (m <= 0) return;
    if (lanes <= 1 || m < 2 * (i64)lanes) {
        double xp = x_init;
        i64 p = lo;
        for (i64 it = 0; it < m; it++) {
            xp = x[p] - dr[p] * off[p] * xp;
            x[p] = xp;
            p += step;
        }
        return;
    }
    i64 chunk = m / lanes;
    for (int l = 0; l < lanes; l++) {
        i64 base = l * chunk;
        i64 p = lo + base * step;
        aw[base] = -dr[p] * off[p];
        cw[base] = x[p];
        for (i64 t = 1; t < chunk; t++) {
            p += step;
            double a = -dr[p] * off[p];
            aw[base + t] = a * aw[base + t - 1];
            cw[base + t] = a * cw[base + t - 1] + x[p];
        }
    }
    double carry = x_init;
    for (int l = 0; l < lanes; l++) {
        i64 base = l * chunk;
        for (i64 t = 0; t < chunk; t++)
            x[lo + (base + t) * step] = aw[base + t] * carry + cw[base + t];
        carry = aw[base + chunk - 1] * carry + cw[base + chunk - 1];
    }
    double xp = carry;
    i64 p = lo + lanes * chunk * step;
    for (i64 it = lanes * chunk; it < m; it++) {
        xp = x[p] - dr[p] * off[p] * xp;
        x[p] = xp;
        p += step;
    }
}

/* public wrapper of the chain (ntd_solve.py:272-300, chain_bidiagonal_solve) */
void orc_chain_solve(const double *dr, const double *off, const double *rhs,
                     double *x, i64 n, int backward, int lanes)
{
    double *aw = malloc(sizeof(double) * (n > 0 ? n : 1));
    double *cw = malloc(sizeof(double) * (n > 0 ? n : 1));
    if (n > 0) {
        if (!backward)
            chain_scaled(x, dr, off, rhs, 0, n - 1, 1, 0.0, lanes, aw, cw);
        else
            chain_scaled(x, dr, off, rhs, n - 1, 0, -1, 0.0, lanes, aw, cw);
    }
    free(aw);
    free(cw);
}

/* ntd_solve.py:107-121 (_line_lower) */
static void line_lower(double *x, const double *b, const double *mr,
                       const double *l1, const double *u1, i64 s, i64 e,
                       int lanes, double *aw, double *cw)
{
    i64 t = s + (e - s - 1) / 2;
    if (t - 1 >= s) chain_scaled(x, mr, l1, b, s, t - 1, 1, 0.0, lanes, aw, cw);
    if (t + 1 <= e - 1)
        chain_scaled(x, mr, u1, b, e - 1, t + 1, -1, 0.0, lanes, aw, cw);
    double acc = b[t];
    if (t > s) acc -= l1[t] * x[t - 1];
    if (t < e - 1) acc -= u1[t] * x[t + 1];
    x[t] = acc * mr[t];
}

/* ntd_solve.py:124-131 (_line_upper) */
static void line_upper(double *x, const double *mr, const double *l1,
                       const double *u1, i64 s, i64 e, int lanes, double *aw,
                       double *cw)
{
    i64 t = s + (e - s - 1) / 2;
    if (t - 1 >= s) chain_unit(x, mr, u1, t - 1, s, -1, x[t], lanes, aw, cw);
    if (t + 1 <= e - 1) chain_unit(x, mr, l1, t + 1, e - 1, 1, x[t], lanes, aw, cw);
}

/* ntd_solve.py:134-137 (_line_solve) */
static void line_solve(double *x, const double *b, const double *mr,
                       const double *l1, const double *u1, i64 s, i64 e,
                       int lanes, double *aw, double *cw)
{
    line_lower(x, b, mr, l1, u1, s, e, lanes, aw, cw);
    line_upper(x, mr, l1, u1, s, e, lanes, aw, cw);
}

/* ntd_solve.py:140-185 (_plane_solve); b is consumed. */
static void plane_solve(double *x, double *b, double *xs, double *bs,
                        const double *mr, const double *l1, const double *u1,
                        const double *l2, const double *u2, i64 base, i64 nx,
                        i64 ny, int lanes, double *aw, double *cw)
{
    i64 t = (ny - 1) / 2;
    i64 s;
    if (t > 0) {
        s = base;
        line_solve(x, b, mr, l1, u1, s, s + nx, lanes, aw, cw);
        for (i64 q = 1; q < t; q++) {
            s = base + q * nx;
            for (i64 r = s; r < s + nx; r++) b[r] -= l2[r] * x[r - nx];
            line_solve(x, b, mr, l1, u1, s, s + nx, lanes, aw, cw);
        }
    }
    if (t < ny - 1) {
        s = base + (ny - 1) * nx;
        line_solve(x, b, mr, l1, u1, s, s + nx, lanes, aw, cw);
        for (i64 q = ny - 2; q > t; q--) {
            s = base + q * nx;
            for (i64 r = s; r < s + nx; r++) b[r] -= u2[r] * x[r + nx];
            line_solve(x, b, mr, l1, u1, s, s + nx, lanes, aw, cw);
        }
    }
    s = base + t * nx;
    if (t > 0)
        for (i64 r = s; r < s + nx; r++) b[r] -= l2[r] * x[r - nx];
    if (t < ny - 1)
        for (i64 r = s; r < s + nx; r++) b[r] -= u2[r] * x[r + nx];
    line_solve(x, b, mr, l1, u1, s, s + nx, lanes, aw, cw);
    for (i64 q = t - 1; q >= 0; q--) {
        s = base + q * nx;
        for (i64 r = s; r < s + nx; r++) bs[r] = u2[r] * x[r + nx];
        line_solve(xs, bs, mr, l1, u1, s, s + nx, lanes, aw, cw);
        for (i64 r = s; r < s + nx; r++) x[r] -= xs[r];
    }
    for (i64 q = t + 1; q < ny; q++) {
        s = base + q * nx;
        for (i64 r = s; r < s + nx; r++) bs[r] = l2[r] * x[r - nx];
        line_solve(xs, bs, mr, l1, u1, s, s + nx, lanes, aw, cw);
        for (i64 r = s; r < s + nx; r++) x[r] -= xs[r];
    }
}

/* ntd_solve.py:188-253 (_apply_kernel); the two halves write disjoint rows,
 * so running them one after the other (or as a 2-thread team) is identical. */
static void apply_kernel(double *x, double *b, double *xs2, double *bs2,
                         double *xs3, double *bs3, const double *mr,
                         const double *l1, const double *u1, const double *l2,
                         const double *u2, const double *l3, const double *u3,
                         i64 nx, i64 ny, i64 nz, int lanes, int nthreads)
{
    i64 nxy = nx * ny;
    i64 t = (nz - 1) / 2;
    (void)nthreads;
#pragma omp parallel for num_threads(nthreads >= 2 ? 2 : 1) schedule(static, 1)
    for (int h = 0; h < 2; h++) {
        double *aw = malloc(sizeof(double) * nx), *cw = malloc(sizeof(double) * nx);
        if (h == 0) {
            if (t > 0) {
                plane_solve(x, b, xs2, bs2, mr, l1, u1, l2, u2, 0, nx, ny, lanes, aw, cw);
                for (i64 p = 1; p < t; p++) {
                    i64 base = p * nxy;
                    for (i64 r = base; r < base + nxy; r++) b[r] -= l3[r] * x[r - nxy];
                    plane_solve(x, b, xs2, bs2, mr, l1, u1, l2, u2, base, nx, ny, lanes, aw, cw);
                }
            }
        } else {
            if (t < nz - 1) {
                i64 base = (nz - 1) * nxy;
                plane_solve(x, b, xs2, bs2, mr, l1, u1, l2, u2, base, nx, ny, lanes, aw, cw);
                for (i64 p = nz - 2; p > t; p--) {
                    base = p * nxy;
                    for (i64 r = base; r < base + nxy; r++) b[r] -= u3[r] * x[r + nxy];
                    plane_solve(x, b, xs2, bs2, mr, l1, u1, l2, u2, base, nx, ny, lanes, aw, cw);
                }
            }
        }
        free(aw);
        free(cw);
    }
    i64 base = t * nxy;
    if (t > 0)
        for (i64 r = base; r < base + nxy; r++) b[r] -= l3[r] * x[r - nxy];
    if (t < nz - 1)
        for (i64 r = base; r < base + nxy; r++) b[r] -= u3[r] * x[r + nxy];
    {
        double *aw = malloc(sizeof(double) * nx), *cw = malloc(sizeof(double) * nx);
        plane_solve(x, b, xs2, bs2, mr, l1, u1, l2, u2, base, nx, ny, lanes, aw, cw);
        free(aw);
        free(cw);
    }
#pragma omp parallel for num_threads(nthreads >= 2 ? 2 : 1) schedule(static, 1)
    for (int h = 0; h < 2; h++) {
        double *aw = malloc(sizeof(double) * nx), *cw = malloc(sizeof(double) * nx);
        if (h == 0) {
            for (i64 p = t - 1; p >= 0; p--) {
                i64 bb = p * nxy;
                for (i64 r = bb; r < bb + nxy; r++) bs3[r] = u3[r] * x[r + nxy];
                plane_solve(xs3, bs3, xs2, bs2, mr, l1, u1, l2, u2, bb, nx, ny, lanes, aw, cw);
                for (i64 r = bb; r < bb + nxy; r++) x[r] -= xs3[r];
            }
        } else {
            for (i64 p = t + 1; p < nz; p++) {
                i64 bb = p * nxy;
                for (i64 r = bb; r < bb + nxy; r++) bs3[r] = l3[r] * x[r - nxy];
                plane_solve(xs3, bs3, xs2, bs2, mr, l1, u1, l2, u2, bb, nx, ny, lanes, aw, cw);
                for (i64 r = bb; r < bb + nxy; r++) x[r] -= xs3[r];
            }
        }
        free(aw);
        free(cw);
    }
}

/* ntd_solve.py:303-322 (ntd_apply); pre = [l1,u1,l2,u2,l3,u3,m_recip] x N */
void orc_ntd_apply(const double *pre, const double *b, double *x, i64 nx,
                   i64 ny, i64 nz, int lanes, int nthreads)
{
    i64 n = nx * ny * nz;
    double *ws = malloc(sizeof(double) * 5 * n);
    memcpy(ws, b, sizeof(double) * n);
    apply_kernel(x, ws, ws + n, ws + 2 * n, ws + 3 * n, ws + 4 * n, pre + 6 * n,
                 pre, pre + n, pre + 2 * n, pre + 3 * n, pre + 4 * n, pre + 5 * n,
                 nx, ny, nz, lanes, nthreads);
    free(ws);
}

/* -------------------------------------------------------------- factor */
/* ntd_factor.py:80-110 (_line_factor): returns -1 or the bad row */
static i64 line_factor(const double *td, const double *tl, const double *tu,
                       double *mr, i64 s, i64 e)
{
    i64 t = s + (e - s - 1) / 2;
    double piv;
    for (i64 i = s; i < t; i++) {
        if (i == s) piv = td[i];
        else piv = td[i] - tl[i] * tu[i - 1] * mr[i - 1];
        if (piv == 0.0 || !isfinite(piv)) return i;
        mr[i] = 1.0 / piv;
    }
    for (i64 i = e - 1; i > t; i--) {
        if (i == e - 1) piv = td[i];
        else piv = td[i] - tu[i] * tl[i + 1] * mr[i + 1];
        if (piv == 0.0 || !isfinite(piv)) return i;
        mr[i] = 1.0 / piv;
    }
    piv = td[t];
    if (t > s) piv -= tl[t] * tu[t - 1] * mr[t - 1];
    if (t < e - 1) piv -= tu[t] * tl[t + 1] * mr[t + 1];
    if (piv == 0.0 || !isfinite(piv)) return t;
    mr[t] = 1.0 / piv;
    return -1;
}

/* ntd_factor.py:113-144 (_correct_line) */
static i64 correct_line(i64 q, i64 m, const double *pl2, const double *pu2,
                        double *tdw, double *l1g, double *u1g, const double *mrg,
                        i64 nx, int lanes, double *aw, double *cw, double *xw,
                        double *bw)
{
    i64 sq = q * nx, sm = m * nx;
    if (m < q)
        for (i64 k = 0; k < nx; k++) bw[sm + k] = pu2[sm + k];
    else
        for (i64 k = 0; k < nx; k++) bw[sm + k] = pl2[sm + k];
    line_solve(xw, bw, mrg, l1g, u1g, sm, sm + nx, lanes, aw, cw);
    for (i64 k = 0; k < nx; k++) {
        double u = bw[sm + k];
        double bet = u != 0.0 ? xw[sm + k] / u : 0.0;
        if (!isfinite(bet)) return sm + k;
        xw[sm + k] = bet;
    }
    for (i64 k = 0; k < nx; k++) {
        double rs = m < q ? pl2[sq + k] : pu2[sq + k];
        double bet = xw[sm + k];
        tdw[sq + k] -= rs * (2.0 * bet - bet * tdw[sm + k] * bet) * bw[sm + k];
        if (k >= 1)
            l1g[sq + k] += rs * bet * l1g[sm + k] * xw[sm + k - 1] * bw[sm + k - 1];
        if (k + 1 < nx)
            u1g[sq + k] += rs * bet * u1g[sm + k] * xw[sm + k + 1] * bw[sm + k + 1];
    }
    return -1;
}

/* ntd_factor.py:147-219 (_factor_plane); returns code, writes *idx */
static int factor_plane(const double *pd, const double *pl1, const double *pu1,
                        const double *pl2, const double *pu2, i64 nx, i64 ny,
                        double *l1g, double *u1g, double *mrg, double *tdw,
                        int lanes, double *aw, double *cw, double *xw,
                        double *bw, i64 *idx)
{
    i64 t = (ny - 1) / 2, st;
    *idx = -1;
    if (t > 0) {
        for (i64 k = 0; k < nx; k++) { tdw[k] = pd[k]; l1g[k] = pl1[k]; u1g[k] = pu1[k]; }
        st = line_factor(tdw, l1g, u1g, mrg, 0, nx);
        if (st >= 0) { *idx = st; return 1; }
        for (i64 q = 1; q < t; q++) {
            i64 sq = q * nx;
            for (i64 k = sq; k < sq + nx; k++) { tdw[k] = pd[k]; l1g[k] = pl1[k]; u1g[k] = pu1[k]; }
            st = correct_line(q, q - 1, pl2, pu2, tdw, l1g, u1g, mrg, nx, lanes, aw, cw, xw, bw);
            if (st >= 0) { *idx = st; return 2; }
            st = line_factor(tdw, l1g, u1g, mrg, sq, sq + nx);
            if (st >= 0) { *idx = st; return 1; }
        }
    }
    if (t < ny - 1) {
        i64 sq = (ny - 1) * nx;
        for (i64 k = sq; k < sq + nx; k++) { tdw[k] = pd[k]; l1g[k] = pl1[k]; u1g[k] = pu1[k]; }
        st = line_factor(tdw, l1g, u1g, mrg, sq, sq + nx);
        if (st >= 0) { *idx = st; return 1; }
        for (i64 q = ny - 2; q > t; q--) {
            sq = q * nx;
            for (i64 k = sq; k < sq + nx; k++) { tdw[k] = pd[k]; l1g[k] = pl1[k]; u1g[k] = pu1[k]; }
            st = correct_line(q, q + 1, pl2, pu2, tdw, l1g, u1g, mrg, nx, lanes, aw, cw, xw, bw);
            if (st >= 0) { *idx = st; return 2; }
            st = line_factor(tdw, l1g, u1g, mrg, sq, sq + nx);
            if (st >= 0) { *idx = st; return 1; }
        }
    }
    i64 sq = t * nx;
    for (i64 k = sq; k < sq + nx; k++) { tdw[k] = pd[k]; l1g[k] = pl1[k]; u1g[k] = pu1[k]; }
    if (t > 0) {
        st = correct_line(t, t - 1, pl2, pu2, tdw, l1g, u1g, mrg, nx, lanes, aw, cw, xw, bw);
        if (st >= 0) { *idx = st; return 2; }
    }
    if (t < ny - 1) {
        st = correct_line(t, t + 1, pl2, pu2, tdw, l1g, u1g, mrg, nx, lanes, aw, cw, xw, bw);
        if (st >= 0) { *idx = st; return 2; }
    }
    st = line_factor(tdw, l1g, u1g, mrg, sq, sq + nx);
    if (st >= 0) { *idx = st; return 1; }
    return 0;
}

/* ntd_factor.py:222-239 (_plane_correction) */
static void plane_correction(double *pd, double *pl1, double *pu1, double *pl2,
                             double *pu2, const double *qd, const double *ql1,
                             const double *qu1, const double *ql2,
                             const double *qu2, const double *beta,
                             const double *rowscale, const double *colscale,
                             i64 nx, i64 nxy)
{
    for (i64 k = 0; k < nxy; k++) {
        double rs = rowscale[k], bet = beta[k];
        pd[k] -= rs * (2.0 * bet - bet * qd[k] * bet) * colscale[k];
        if (k >= 1) pl1[k] += rs * bet * ql1[k] * beta[k - 1] * colscale[k - 1];
        if (k + 1 < nxy) pu1[k] += rs * bet * qu1[k] * beta[k + 1] * colscale[k + 1];
        if (k >= nx) pl2[k] += rs * bet * ql2[k] * beta[k - nx] * colscale[k - nx];
        if (k + nx < nxy) pu2[k] += rs * bet * qu2[k] * beta[k + nx] * colscale[k + nx];
    }
}

typedef struct {
    double *pd, *pl1, *pu1, *pl2, *pu2;
} plane_bands;

typedef struct {
    i64 nx, ny, nz, nxy;
    int lanes;
    const double *ad, *al1, *au1, *al2, *au2;
    double *l1, *u1, *l2, *u2, *l3, *u3, *mr;
} fctx;

static void pb_alloc(plane_bands *b, i64 nxy)
{
    b->pd = malloc(sizeof(double) * 5 * nxy);
    b->pl1 = b->pd + nxy; b->pu1 = b->pd + 2 * nxy;
    b->pl2 = b->pd + 3 * nxy; b->pu2 = b->pd + 4 * nxy;
}

/* ntd_factor.py:372-376 (plane_bands_of) */
static void pb_load(const fctx *c, plane_bands *b, i64 p)
{
    i64 base = p * c->nxy, n = c->nxy;
    memcpy(b->pd, c->ad + base, sizeof(double) * n);
    memcpy(b->pl1, c->al1 + base, sizeof(double) * n);
    memcpy(b->pu1, c->au1 + base, sizeof(double) * n);
    memcpy(b->pl2, c->al2 + base, sizeof(double) * n);
    memcpy(b->pu2, c->au2 + base, sizeof(double) * n);
}

/* ntd_factor.py:378-404 (correct_from), incl. the sandwich adjustment
 * :387-399.  Returns 0, 2 (non-finite filter weight) or 3 (non-finite
 * sandwich adjustment). */
static int correct_from(const fctx *c, plane_bands *bands, i64 p, i64 m,
                        const plane_bands *nb)
{
    i64 nx = c->nx, ny = c->ny, nxy = c->nxy;
    i64 mb = m * nxy;
    const double *useg = m < p ? c->u3 + mb : c->l3 + mb;
    /* _apply_factored_plane (ntd_factor.py:336-348) */
    double *w = malloc(sizeof(double) * 5 * nxy);
    double *bb = w + nxy, *xs = w + 2 * nxy, *bs = w + 3 * nxy, *beta = w + 4 * nxy;
    double *aw = malloc(sizeof(double) * nx), *cw = malloc(sizeof(double) * nx);
    memcpy(bb, useg, sizeof(double) * nxy);
    plane_solve(w, bb, xs, bs, c->mr + mb, c->l1 + mb, c->u1 + mb, c->l2 + mb,
                c->u2 + mb, 0, nx, ny, c->lanes, aw, cw);
    int rc = 0;
    /* _beta_from (ntd_factor.py:242-249) */
    for (i64 k = 0; k < nxy; k++) {
        beta[k] = useg[k] != 0.0 ? w[k] / useg[k] : 0.0;
        if (!isfinite(beta[k])) rc = 2;
    }
    if (!rc) {
        /* _plane_band_action (ntd_factor.py:266-274) */
        double *qw = bb, *qd = bs;
        for (i64 k = 0; k < nxy; k++) qw[k] = nb->pd[k] * w[k];
        for (i64 k = 1; k < nxy; k++) qw[k] += nb->pl1[k] * w[k - 1];
        for (i64 k = 0; k + 1 < nxy; k++) qw[k] += nb->pu1[k] * w[k + 1];
        for (i64 k = nx; k < nxy; k++) qw[k] += nb->pl2[k] * w[k - nx];
        for (i64 k = 0; k + nx < nxy; k++) qw[k] += nb->pu2[k] * w[k + nx];
        for (i64 k = 0; k < nxy; k++) {
            qd[k] = nb->pd[k];
            if (w[k] != 0.0) qd[k] += (useg[k] - qw[k]) / w[k];
            if (!isfinite(qd[k])) rc = 3;
        }
        if (!rc) {
            i64 pb = p * nxy;
            const double *rowscale = m < p ? c->l3 + pb : c->u3 + pb;
            plane_correction(bands->pd, bands->pl1, bands->pu1, bands->pl2,
                             bands->pu2, qd, nb->pl1, nb->pu1, nb->pl2, nb->pu2,
                             beta, rowscale, useg, nx, nxy);
        }
    }
    free(w);
    free(aw);
    free(cw);
    return rc;
}

/* ntd_factor.py:406-419 (factor_one) */
static int factor_one(const fctx *c, i64 p, const plane_bands *bands, i64 *row)
{
    i64 nx = c->nx, nxy = c->nxy, base = p * nxy;
    memcpy(c->l2 + base, bands->pl2, sizeof(double) * nxy);
    memcpy(c->u2 + base, bands->pu2, sizeof(double) * nxy);
    double *tdw = malloc(sizeof(double) * 3 * nxy), *xw = tdw + nxy, *bw = tdw + 2 * nxy;
    double *aw = malloc(sizeof(double) * nx), *cw = malloc(sizeof(double) * nx);
    i64 idx;
    int code = factor_plane(bands->pd, bands->pl1, bands->pu1, bands->pl2,
                            bands->pu2, nx, c->ny, c->l1 + base, c->u1 + base,
                            c->mr + base, tdw, c->lanes, aw, cw, xw, bw, &idx);
    free(tdw);
    free(aw);
    free(cw);
    *row = code ? base + idx : -1;
    return code;
}

/* ntd_factor.py:425-434 (run_half).  status: code, plane, row */
static void run_half(const fctx *c, i64 p0, i64 p1, i64 step, plane_bands *prev,
                     i64 *prev_p, i64 *status)
{
    i64 nxy = c->nxy;
    plane_bands cur;
    pb_alloc(&cur, nxy);
    *prev_p = -1;
    for (i64 p = p0; p != p1; p += step) {
        pb_load(c, &cur, p);
        if (*prev_p >= 0) {
            int rc = correct_from(c, &cur, p, *prev_p, prev);
            if (rc) { status[0] = rc; status[1] = p; status[2] = -1; break; }
        }
        i64 row;
        int code = factor_one(c, p, &cur, &row);
        if (code) { status[0] = code; status[1] = p; status[2] = row; break; }
        memcpy(prev->pd, cur.pd, sizeof(double) * 5 * nxy);
        *prev_p = p;
    }
    free(cur.pd);
}

/* ntd_factor.py:351-458 (factor_level3).  a = 7 x N bands; pre = 7 x N output
 * (l1,u1,l2,u2,l3,u3,m_recip).  status[3] = (code, plane, row): code 0 ok,
 * 1 pivot, 2 filter weight, 3 sandwich adjustment. */
void orc_factor_level3(const double *a, double *pre, i64 nx, i64 ny, i64 nz,
                       int lanes, int nthreads, i64 *status)
{
    i64 n = nx * ny * nz, nxy = nx * ny;
    fctx c = {nx, ny, nz, nxy, lanes, a + 3 * n, a + 2 * n, a + 4 * n, a + n,
              a + 5 * n, pre, pre + n, pre + 2 * n, pre + 3 * n, pre + 4 * n,
              pre + 5 * n, pre + 6 * n};
    memset(pre, 0, sizeof(double) * 7 * n);
    memcpy(c.l3, a, sizeof(double) * n);
    memcpy(c.u3, a + 6 * n, sizeof(double) * n);
    i64 t3 = (nz - 1) / 2;
    plane_bands pa, pdsc;
    pb_alloc(&pa, nxy);
    pb_alloc(&pdsc, nxy);
    i64 sa[3] = {0, -1, -1}, sd[3] = {0, -1, -1}, pa_p = -1, pd_p = -1;
    (void)nthreads;
#pragma omp parallel for num_threads(nthreads >= 2 ? 2 : 1) schedule(static, 1)
    for (int h = 0; h < 2; h++) {
        if (h == 0) run_half(&c, 0, t3, 1, &pa, &pa_p, sa);
        else run_half(&c, nz - 1, t3, -1, &pdsc, &pd_p, sd);
    }
    status[0] = 0; status[1] = -1; status[2] = -1;
    /* the ascending half's error is reported first (fut_a.result() :442) */
    if (sa[0]) { memcpy(status, sa, sizeof(sa)); goto done; }
    if (sd[0]) { memcpy(status, sd, sizeof(sd)); goto done; }
    {
        plane_bands cur;
        pb_alloc(&cur, nxy);
        pb_load(&c, &cur, t3);
        int rc = 0;
        if (pa_p >= 0) rc = correct_from(&c, &cur, t3, pa_p, &pa);
        if (!rc && pd_p >= 0) rc = correct_from(&c, &cur, t3, pd_p, &pdsc);
        if (rc) { status[0] = rc; status[1] = t3; status[2] = -1; }
        else {
            i64 row;
            int code = factor_one(&c, t3, &cur, &row);
            if (code) { status[0] = code; status[1] = t3; status[2] = row; }
        }
        free(cur.pd);
    }
done:
    free(pa.pd);
    free(pdsc.pd);
}

/* ---------------------------------------------------------------- ilu0 */
/* ilu0.py:34-83 (_ilu0_half) */
static i64 ilu0_half(double *f, const double *orig, i64 n, i64 lo, i64 hi,
                     i64 nx, i64 nxy)
{
#define F(t, i) f[(t) * n + (i)]
#define O(t, i) orig[(t) * n + (i)]
    for (i64 i = lo; i < hi; i++) {
        for (int t = 0; t < 3; t++) {
            i64 d = t == 0 ? nxy : (t == 1 ? nx : 1);
            i64 k = i - d;
            if (k < lo || O(t, i) == 0.0) continue;
            double fac = F(t, i) / F(3, k);
            F(t, i) = fac;
            for (int s = 0; s < 3; s++) {
                i64 du = s == 0 ? 1 : (s == 1 ? nx : nxy);
                double uv = F(4 + s, k);
                if (uv == 0.0) continue;
                i64 j = k + du;
                if (j >= hi) continue;
                i64 dj = j - i;
                if (dj == 0) F(3, i) -= fac * uv;
                else if (dj == 1 && O(4, i) != 0.0) F(4, i) -= fac * uv;
                else if (dj == nx && O(5, i) != 0.0) F(5, i) -= fac * uv;
                else if (dj == nxy && O(6, i) != 0.0) F(6, i) -= fac * uv;
                else if (dj == -1 && O(2, i) != 0.0) F(2, i) -= fac * uv;
                else if (dj == -nx && O(1, i) != 0.0) F(1, i) -= fac * uv;
                else if (dj == -nxy && O(0, i) != 0.0) F(0, i) -= fac * uv;
            }
        }
        double piv = F(3, i);
        if (piv == 0.0 || !isfinite(piv)) return i;
    }
    return -1;
#undef F
#undef O
}

/* ilu0.py:134-156 (build_block_ilu0) incl. _drop_split_couplings :126-131.
 * Returns -1 or the min bad row. */
i64 orc_build_ilu0(const double *a, double *f, i64 nx, i64 ny, i64 nz,
                   i64 split, int nthreads)
{
    i64 n = nx * ny * nz, nxy = nx * ny;
    i64 offs[7] = {-nxy, -nx, -1, 0, 1, nx, nxy};
    memcpy(f, a, sizeof(double) * 7 * n);
    for (int idx = 0; idx < 7; idx++) {
        i64 d = offs[idx];
        if (d > 0) {
            for (i64 r = (split - d > 0 ? split - d : 0); r < split; r++) f[idx * n + r] = 0.0;
        } else if (d < 0) {
            i64 e = split - d < n ? split - d : n;
            for (i64 r = split; r < e; r++) f[idx * n + r] = 0.0;
        }
    }
    i64 st[2];
    (void)nthreads;
#pragma omp parallel for num_threads(nthreads >= 2 ? 2 : 1) schedule(static, 1)
    for (int h = 0; h < 2; h++)
        st[h] = h == 0 ? ilu0_half(f, a, n, 0, split, nx, nxy)
                       : ilu0_half(f, a, n, split, n, nx, nxy);
    i64 bad = -1;
    for (int h = 0; h < 2; h++)
        if (st[h] >= 0 && (bad < 0 || st[h] < bad)) bad = st[h];
    return bad;
}

/* ilu0.py:95-114 (_ilu0_apply_half) */
static void ilu0_apply_half(const double *f, i64 n, const double *r, double *z,
                            i64 lo, i64 hi, i64 nx, i64 nxy)
{
    const double *f0 = f, *f1 = f + n, *f2 = f + 2 * n, *f3 = f + 3 * n,
                 *f4 = f + 4 * n, *f5 = f + 5 * n, *f6 = f + 6 * n;
    for (i64 i = lo; i < hi; i++) {
        double acc = r[i];
        if (i - 1 >= lo) acc -= f2[i] * z[i - 1];
        if (i - nx >= lo) acc -= f1[i] * z[i - nx];
        if (i - nxy >= lo) acc -= f0[i] * z[i - nxy];
        z[i] = acc;
    }
    for (i64 i = hi - 1; i >= lo; i--) {
        double acc = z[i];
        if (i + 1 < hi) acc -= f4[i] * z[i + 1];
        if (i + nx < hi) acc -= f5[i] * z[i + nx];
        if (i + nxy < hi) acc -= f6[i] * z[i + nxy];
        z[i] = acc / f3[i];
    }
}

/* ilu0.py:159-169 (ilu0_apply) */
void orc_ilu0_apply(const double *f, const double *r, double *z, i64 nx,
                    i64 ny, i64 nz, i64 split, int nthreads)
{
    i64 n = nx * ny * nz, nxy = nx * ny;
    (void)nthreads;
#pragma omp parallel for num_threads(nthreads >= 2 ? 2 : 1) schedule(static, 1)
    for (int h = 0; h < 2; h++) {
        if (h == 0) ilu0_apply_half(f, n, r, z, 0, split, nx, nxy);
        else ilu0_apply_half(f, n, r, z, split, n, nx, nxy);
    }
}

/* ------------------------------------------------------ combined + pcg */
typedef struct {
    const double *a, *pre, *ilu;
    i64 nx, ny, nz, split;
    int lanes, nthreads;
    double *w, *t, *z2; /* scratch, N each */
} combined;

/* precond_pcg.py:57-65 (combined_apply) */
static void combined_apply(const combined *c, const double *r, double *z)
{
    i64 n = c->nx * c->ny * c->nz, nxy = c->nx * c->ny;
    orc_ilu0_apply(c->ilu, r, c->w, c->nx, c->ny, c->nz, c->split, c->nthreads);
    orc_spmv(c->a, c->w, c->t, n, c->nx, nxy, c->nthreads);
    for (i64 i = 0; i < n; i++) c->t[i] = r[i] - c->t[i];
    orc_ntd_apply(c->pre, c->t, z, c->nx, c->ny, c->nz, c->lanes, c->nthreads);
    for (i64 i = 0; i < n; i++) z[i] += c->w[i];
    orc_spmv(c->a, z, c->t, n, c->nx, nxy, c->nthreads);
    for (i64 i = 0; i < n; i++) c->t[i] = r[i] - c->t[i];
    orc_ilu0_apply(c->ilu, c->t, c->z2, c->nx, c->ny, c->nz, c->split, c->nthreads);
    for (i64 i = 0; i < n; i++) z[i] += c->z2[i];
}

void orc_combined_apply(const double *a, const double *pre, const double *ilu,
                        i64 nx, i64 ny, i64 nz, i64 split, int lanes,
                        int nthreads, const double *r, double *z)
{
    i64 n = nx * ny * nz;
    double *ws = malloc(sizeof(double) * 3 * n);
    combined c = {a, pre, ilu, nx, ny, nz, split, lanes, nthreads, ws, ws + n, ws + 2 * n};
    combined_apply(&c, r, z);
    free(ws);
}

static double sdot(const double *x, const double *y, i64 n)
{
    double s = 0.0;
    for (i64 i = 0; i < n; i++) s += x[i] * y[i];
    return s;
}

/* preconditioner of kind 1 (ntd+ilu0, precond_pcg.py:57-65) or 2 (ntd alone,
 * bench_cli.py:113-121: ntd_apply with the factor), else the identity */
static void precond(const combined *c, int kind, const double *r, double *z, i64 n)
{
    if (kind == 1)
        combined_apply(c, r, z);
    else if (kind == 2)
        orc_ntd_apply(c->pre, r, z, c->nx, c->ny, c->nz, c->lanes, c->nthreads);
    else
        memcpy(z, r, sizeof(double) * n);
}

/* precond_pcg.py:68-122 (pcg).  kind: 0 none, 1 ntd+ilu0, 2 ntd (pre, ilu given).
 * history must hold max_iters doubles.  Returns iterations; *conv set;
 * returns -1 on breakdown (DivergenceError). */
i64 orc_pcg(const double *a, const double *pre, const double *ilu, i64 nx,
            i64 ny, i64 nz, i64 split, int lanes, int nthreads, int kind,
            const double *b, double *x, double tol, i64 max_iters,
            double *history, int *conv)
{
    i64 n = nx * ny * nz, nxy = nx * ny;
    double *ws = malloc(sizeof(double) * 8 * n);
    double *r = ws, *z = ws + n, *p = ws + 2 * n, *ap = ws + 3 * n, *res = ws + 4 * n;
    combined c = {a, pre, ilu, nx, ny, nz, split, lanes, nthreads, ws + 5 * n, ws + 6 * n, ws + 7 * n};
    memset(x, 0, sizeof(double) * n);
    *conv = 0;
    double bnorm = sqrt(sdot(b, b, n));
    if (bnorm == 0.0) { free(ws); *conv = 1; return 0; }
    memcpy(r, b, sizeof(double) * n);
    precond(&c, kind, r, z, n);
    memcpy(p, z, sizeof(double) * n);
    double rz = sdot(r, z, n);
    i64 it = 0;
    for (it = 1; it <= max_iters; it++) {
        orc_spmv(a, p, ap, n, nx, nxy, nthreads);
        double pap = sdot(p, ap, n);
        if (pap <= 0.0 || !isfinite(pap)) { it = -1; break; }
        double alpha = rz / pap;
        for (i64 i = 0; i < n; i++) x[i] = alpha * p[i] + x[i];
        for (i64 i = 0; i < n; i++) r[i] = -alpha * ap[i] + r[i];
        orc_spmv(a, x, res, n, nx, nxy, nthreads);
        for (i64 i = 0; i < n; i++) res[i] = -1.0 * res[i] + b[i];
        double relres = sqrt(sdot(res, res, n)) / bnorm;
        history[it - 1] = relres;
        if (!isfinite(relres)) { it = -2; break; }
        if (relres < tol) { *conv = 1; break; }
        precond(&c, kind, r, z, n);
        double rz_new = sdot(r, z, n);
        double beta = rz_new / rz;
        for (i64 i = 0; i < n; i++) p[i] = beta * p[i] + z[i];
        rz = rz_new;
    }
    if (it > max_iters) it = max_iters;
    free(ws);
    return it;
}
