// Dependent-instruction latencies with the loop overhead amortised: each
// timed loop body is 32 dependent instructions (unrolled), 256 trips.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/micro_lat2.bin tools/micro_lat2.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_lat(double *out, long long *cyc, double a, double b)
{
    __shared__ double sh[64];
    const int lane = threadIdx.x;
    double x = a + lane, y = b + lane;
    sh[lane] = 0.0;
    sh[lane + 32] = 0.0;
    __syncwarp();
    long long t[8];
    t[0] = clock64();
#pragma unroll 1
    for (int i = 0; i < 256; i++) {
#pragma unroll
        for (int j = 0; j < 32; j++) x = fma(x, b, a);
    }
    t[1] = clock64();
#pragma unroll 1
    for (int i = 0; i < 256; i++) {
#pragma unroll
        for (int j = 0; j < 32; j++) x = x + b;
    }
    t[2] = clock64();
#pragma unroll 1
    for (int i = 0; i < 256; i++) {
#pragma unroll
        for (int j = 0; j < 32; j++) x = x * b;
    }
    t[3] = clock64();
#pragma unroll 1
    for (int i = 0; i < 256; i++) {
#pragma unroll
        for (int j = 0; j < 32; j++) x = __shfl_up_sync(0xffffffffu, x, 1);
    }
    t[4] = clock64();
    // two independent DFMA chains interleaved: issue vs latency
#pragma unroll 1
    for (int i = 0; i < 256; i++) {
#pragma unroll
        for (int j = 0; j < 32; j++) {
            x = fma(x, b, a);
            y = fma(y, b, a);
        }
    }
    t[5] = clock64();
    // shared load with dependent address
    int idx = lane;
#pragma unroll 1
    for (int i = 0; i < 256; i++) {
#pragma unroll
        for (int j = 0; j < 32; j++) {
            const double v = sh[idx];
            idx = lane + (int)__double_as_longlong(v);
        }
    }
    t[6] = clock64();
    // shuffle + fma alternating (a scan step)
#pragma unroll 1
    for (int i = 0; i < 256; i++) {
#pragma unroll
        for (int j = 0; j < 32; j++) x = fma(__shfl_up_sync(0xffffffffu, x, 1), b, a);
    }
    t[7] = clock64();
    out[lane] = x + y + idx;
    if (lane == 0)
        for (int i = 0; i < 7; i++) cyc[i] = t[i + 1] - t[i];
}

int main()
{
    double *out;
    long long *cyc, h[7];
    cudaMalloc(&out, 32 * sizeof(double));
    cudaMalloc(&cyc, 7 * sizeof(long long));
    for (int rep = 0; rep < 2; rep++) k_lat<<<1, 32>>>(out, cyc, 1.0000001, 0.9999999);
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    const char *names[7] = {"DFMA (dependent)", "DADD (dependent)", "DMUL (dependent)", "64-bit SHFL.UP (dependent)",
                            "2 interleaved DFMA chains (per pair)", "LDS.64 (dependent address)", "SHFL.64 + DFMA"};
    for (int i = 0; i < 7; i++) printf("%-44s %6.1f cycles\n", names[i], (double)h[i] / (256 * 32));
    return 0;
}
