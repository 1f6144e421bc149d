// Dependent-instruction latencies on this GPU (one warp, clock64): DFMA, DADD,
// a 64-bit shuffle (2 x SHFL + re-pairing), a shared-memory load, and one
// radix-4 scan level of the NTD line solve (3 shuffles + combine).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/micro_lat tools/micro_lat.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int N = 1024;

__global__ void k_lat(double *out, long long *cyc, double a, double b)
{
    __shared__ double sh[64];
    const int lane = threadIdx.x;
    double x = a + lane;
    sh[lane] = x;
    sh[lane + 32] = x;
    __syncwarp();
    long long t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < N; i++) x = fma(x, b, a);
    long long t1 = clock64();
#pragma unroll 1
    for (int i = 0; i < N; i++) x = x + b;
    long long t2 = clock64();
#pragma unroll 1
    for (int i = 0; i < N; i++) x = __shfl_up_sync(0xffffffffu, x, 1, 16) + 0.0;
    long long t3 = clock64();
    int idx = lane;
#pragma unroll 1
    for (int i = 0; i < N; i++) {
        x = sh[idx] + x;
        idx = (int)(x * 0.0) + lane;  // dependent address
    }
    long long t4 = clock64();
#pragma unroll 1
    for (int i = 0; i < N; i++) {
        const double t1_ = __shfl_up_sync(0xffffffffu, x, 1, 16), t2_ = __shfl_up_sync(0xffffffffu, x, 2, 16),
                     t3_ = __shfl_up_sync(0xffffffffu, x, 3, 16);
        x = fma(a, t1_, x) + fma(b, t2_, a * t3_);
    }
    long long t5 = clock64();
    out[lane] = x;
    if (lane == 0) {
        cyc[0] = t1 - t0;
        cyc[1] = t2 - t1;
        cyc[2] = t3 - t2;
        cyc[3] = t4 - t3;
        cyc[4] = t5 - t4;
    }
}

int main()
{
    double *out;
    long long *cyc, h[5];
    cudaMalloc(&out, 32 * sizeof(double));
    cudaMalloc(&cyc, 5 * sizeof(long long));
    for (int rep = 0; rep < 2; rep++) k_lat<<<1, 32>>>(out, cyc, 1.0000001, 0.9999999);
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    const char *names[5] = {"DFMA (dependent)", "DADD (dependent)", "64-bit SHFL.UP + DADD", "LDS.64 + DADD (dep. addr)",
                            "radix-4 scan level (3 SHFL.64 + DFMA/DMUL/DADD)"};
    for (int i = 0; i < 5; i++) printf("%-48s %6.1f cycles\n", names[i], (double)h[i] / N);
    return 0;
}
