// Microbenchmark: latency floor of the warp line solve (registers only),
// plus dependent SHFL / DFMA chains.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_1909_09771_b200/csrc
#include <cstdio>
#include "ntd_kernels.cuh"

template <int K>
__global__ void k_line(double *out, long long *cyc, int iters, int n)
{
    const int lane = threadIdx.x & 31, s = lane & 15;
    LaneMap<K> m(n, lane, n);
    double aL[K], mr[K], aU[K], rhs[K], x[K];
    for (int k = 0; k < K; k++) {
        aL[k] = -0.2 - 0.001 * k;
        mr[k] = 0.25;
        aU[k] = -0.21;
        rhs[k] = 1.0 + lane;
    }
    double xt = 0.0, acc = 0.0;
    long long t0 = clock64();
    for (int it = 0; it < iters; it++) {
        line_solve_a<K>(s, n, m.t, aL, mr, aU, rhs, 1.0 + xt, 0.25, -1.0, -1.0, x, xt);
#pragma unroll
        for (int k = 0; k < K; k++) rhs[k] = 1.0 - 0.5 * x[k];
    }
    long long t1 = clock64();
    for (int k = 0; k < K; k++) acc += x[k];
    out[threadIdx.x] = acc + xt;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

__global__ void k_shfl(double *out, long long *cyc, int iters)
{
    double v = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < iters; i++) v = __shfl_up_sync(0xffffffffu, v, 1, 16) + 1.0;
    long long t1 = clock64();
    out[threadIdx.x] = v;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_dfma(double *out, long long *cyc, int iters)
{
    double v = threadIdx.x, a = 0.999;
    long long t0 = clock64();
    for (int i = 0; i < iters; i++) v = fma(a, v, 1.0);
    long long t1 = clock64();
    out[threadIdx.x] = v;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_lds(double *out, long long *cyc, int iters)
{
    __shared__ int buf[64];
    buf[threadIdx.x] = (threadIdx.x + 1) & 31;
    __syncwarp();
    int p = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < iters; i++) p = buf[p];
    long long t1 = clock64();
    out[threadIdx.x] = p;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

int main()
{
    double *out;
    long long *cyc, h;
    cudaMalloc(&out, 1024 * 8);
    cudaMalloc(&cyc, 8);
    const int IT = 20000;
#define RUN(KERN, ...)                                                   \
    KERN<<<1, 32>>>(out, cyc, IT, ##__VA_ARGS__);                        \
    KERN<<<1, 32>>>(out, cyc, IT, ##__VA_ARGS__);                        \
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);                      \
    printf("%-16s %8.1f cycles/iter\n", #KERN " " #__VA_ARGS__, (double)h / IT);
    RUN(k_shfl);
    RUN(k_dfma);
    RUN(k_lds);
    RUN(k_line<1>, 32);
    RUN(k_line<2>, 64);
    RUN(k_line<3>, 96);
    RUN(k_line<4>, 128);
    RUN(k_line<11>, 350);
    return 0;
}
