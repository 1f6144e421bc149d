// Latency + numerics check of the radix-4 line solve vs sl::line_solve.
#include <cstdio>
#include "ntd_apply_sl.cuh"
#include "ntd_line4.cuh"

template <int K>
__global__ void k_cmp(double *err, long long *cyc, int iters, int n)
{
    const int lane = threadIdx.x & 31, s = lane & 15;
    const int t = (n - 1) / 2;
    const int L = lane < 16 ? t : n - 1 - t, P0 = 16 * K - L;
    double aL[K], mr[K], aU[K], rhs[K], cr[K], x1[K], x2[K];
    for (int k = 0; k < K; k++) {
        const int j = s * K + k - P0;
        const bool v = j >= 0;
        mr[k] = v ? 0.25 + 0.01 * ((lane * 7 + k) % 5) : 0.0;
        aL[k] = v ? -0.2 - 0.003 * ((lane + 3 * k) % 7) : 0.0;
        aU[k] = v ? -0.21 + 0.002 * ((lane + k) % 3) : 0.0;
        rhs[k] = v ? 1.0 + 0.1 * lane - 0.05 * k : 0.0;
    }
    double xt1, xt2;
    sl::line_solve<K>(s, n, t, aL, mr, aU, rhs, 0.7, 0.3, -0.05, -0.06, x1, xt1);
    LinePrep P = line_prep<K>(s, aL, aU);
    for (int k = 0; k < K; k++) cr[k] = rhs[k] * mr[k];
    line_solve4<K>(P, n, t, aL, cr, aU, 0.7 * 0.3, -0.05, -0.06, x2, xt2);
    if (lane == 5 || lane == 20) printf("lane %d K=%d x1=%.17g %.17g x2=%.17g %.17g xt %.17g %.17g\n", lane, K, x1[0], x1[K-1], x2[0], x2[K-1], xt1, xt2);
    double e = fabs(xt1 - xt2) / fabs(xt1);
    for (int k = 0; k < K; k++) e = fmax(e, fabs(x1[k] - x2[k]) / (fabs(x1[k]) + 1e-300));
    for (int o = 16; o; o >>= 1) e = fmax(e, __shfl_xor_sync(0xffffffffu, e, o));
    long long t0 = clock64();
    double bt = 0.7;
    for (int it = 0; it < iters; it++) {
        line_solve4<K>(P, n, t, aL, cr, aU, bt, -0.05, -0.06, x2, xt2);
#pragma unroll
        for (int k = 0; k < K; k++) cr[k] = 0.3 - 0.1 * x2[k] * mr[k];
        bt = 0.7 - 0.01 * xt2;
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) {
        err[0] = e + 0.0 * x2[0];
        cyc[0] = t1 - t0;
    }
}

int main()
{
    double *err, h;
    long long *cyc, c;
    cudaMalloc(&err, 8);
    cudaMalloc(&cyc, 8);
    const int IT = 20000;
#define RUN(K, N)                                                                        \
    k_cmp<K><<<1, 32>>>(err, cyc, IT, N);                                                \
    k_cmp<K><<<1, 32>>>(err, cyc, IT, N);                                                \
    cudaMemcpy(&h, err, 8, cudaMemcpyDeviceToHost);                                      \
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);                                      \
    printf("K=%d n=%d  maxrel=%.2e  %.1f cycles/line\n", K, N, h, (double)c / IT);
    RUN(1, 32) RUN(1, 17) RUN(2, 64) RUN(2, 34) RUN(3, 96) RUN(3, 95) RUN(4, 128) RUN(11, 350)
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
