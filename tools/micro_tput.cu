// Single-warp issue cost (cycles per instruction, independent instructions back to back).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/micro_tput.bin tools/micro_tput.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k(double *out, long long *cyc, double a, double b, int sh)
{
    __shared__ double smem[32 * 32];
    const int lane = threadIdx.x;
    for (int i = 0; i < 32; i++) smem[i * 32 + lane] = a * i + lane;
    __syncwarp();
    double x[16];
    for (int i = 0; i < 16; i++) x[i] = a + lane + i;
    int v[16];
    for (int i = 0; i < 16; i++) v[i] = lane * 3 + i;
    long long t[8];
    t[0] = clock64();
#pragma unroll 1
    for (int it = 0; it < 256; it++) {
#pragma unroll
        for (int i = 0; i < 16; i++) x[i] = fma(x[i], b, a);
    }
    t[1] = clock64();
#pragma unroll 1
    for (int it = 0; it < 256; it++) {
#pragma unroll
        for (int i = 0; i < 16; i++) v[i] = __shfl_up_sync(0xffffffffu, v[i], sh);
    }
    t[2] = clock64();
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem) + lane * 8;
    double acc = 0;
#pragma unroll 1
    for (int it = 0; it < 256; it++) {
        double y[16];
#pragma unroll
        for (int i = 0; i < 16; i++) asm volatile("ld.shared.f64 %0, [%1];" : "=d"(y[i]) : "r"(sa + i * 256));
#pragma unroll
        for (int i = 0; i < 16; i++) acc += y[i];
    }
    t[3] = clock64();
    const unsigned sb = (unsigned)__cvta_generic_to_shared(smem) + lane * 16;
#pragma unroll 1
    for (int it = 0; it < 256; it++) {
        double y[16];
#pragma unroll
        for (int i = 0; i < 8; i++)
            asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(y[2 * i]), "=d"(y[2 * i + 1]) : "r"(sb + i * 512));
#pragma unroll
        for (int i = 0; i < 16; i++) acc += y[i];
    }
    t[4] = clock64();
    // shuffle + dfma interleaved (independent)
#pragma unroll 1
    for (int it = 0; it < 256; it++) {
#pragma unroll
        for (int i = 0; i < 16; i++) {
            v[i] = __shfl_up_sync(0xffffffffu, v[i], sh);
            x[i] = fma(x[i], b, a);
        }
    }
    t[5] = clock64();
    // 64-bit shuffle feeding a dfma (8 independent chains)
#pragma unroll 1
    for (int it = 0; it < 256; it++) {
#pragma unroll
        for (int i = 0; i < 16; i++) x[i] = fma(__shfl_up_sync(0xffffffffu, x[i], sh), b, a);
    }
    t[6] = clock64();
#pragma unroll 1
    for (int it = 0; it < 256; it++) {
#pragma unroll
        for (int i = 0; i < 16; i++) asm volatile("st.shared.f64 [%0], %1;" ::"r"(sa + i * 256), "d"(x[i]));
    }
    t[7] = clock64();
    double s = acc;
    for (int i = 0; i < 16; i++) s += x[i] + v[i];
    out[lane] = s;
    if (lane == 0)
        for (int i = 0; i < 7; i++) cyc[i] = t[i + 1] - t[i];
}

int main()
{
    double *out;
    long long *cyc, h[7];
    cudaMalloc(&out, 32 * sizeof(double));
    cudaMalloc(&cyc, 7 * sizeof(long long));
    for (int rep = 0; rep < 2; rep++) k<<<1, 32>>>(out, cyc, 1.0000001, 0.9999999, 1);
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    const char *names[7] = {"DFMA (16 independent)", "SHFL.32 (16 independent)", "LDS.64 (16 independent, + 16 DADD)",
                            "LDS.128 (8 independent, + 16 DADD)", "SHFL.32 + DFMA pairs (per pair)",
                            "SHFL.64 -> DFMA, 16 independent (per 2 SHFL + DFMA)", "STS.64 (16 independent)"};
    const int per[7] = {16, 16, 16, 8, 16, 16, 16};
    for (int i = 0; i < 7; i++) printf("%-52s %6.2f cycles each\n", names[i], (double)h[i] / (256 * per[i]));
    return 0;
}
