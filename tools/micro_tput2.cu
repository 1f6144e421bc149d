// Shuffle / shared-load issue cost per warp as the number of warps on the SM grows
// (is the ~6-cycle cost a per-warp limit or a per-SM-sub-partition throughput?).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/micro_tput2.bin tools/micro_tput2.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k(double *out, long long *cyc, int sh)
{
    __shared__ double smem[32 * 16];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < 32 * 16; i += blockDim.x) smem[i] = i;
    __syncthreads();
    int v[16];
    for (int i = 0; i < 16; i++) v[i] = lane * 3 + i;
    long long t0 = clock64();
#pragma unroll 1
    for (int it = 0; it < 256; it++) {
#pragma unroll
        for (int i = 0; i < 16; i++) v[i] = __shfl_up_sync(0xffffffffu, v[i], sh);
    }
    long long t1 = clock64();
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem) + lane * 8;
    double acc = 0;
#pragma unroll 1
    for (int it = 0; it < 256; it++) {
        double y[16];
#pragma unroll
        for (int i = 0; i < 16; i++) asm volatile("ld.shared.f64 %0, [%1];" : "=d"(y[i]) : "r"(sa + i * 256));
#pragma unroll
        for (int i = 0; i < 16; i += 4) acc += (y[i] + y[i + 1]) + (y[i + 2] + y[i + 3]);
    }
    long long t2 = clock64();
    double s = acc;
    for (int i = 0; i < 16; i++) s += v[i];
    out[threadIdx.x] = s;
    if (lane == 0) {
        cyc[warp * 2] = t1 - t0;
        cyc[warp * 2 + 1] = t2 - t1;
    }
}

int main()
{
    double *out;
    long long *cyc, h[64];
    cudaMalloc(&out, 1024 * sizeof(double));
    cudaMalloc(&cyc, 64 * sizeof(long long));
    for (int warps : {1, 2, 4, 8, 16, 32}) {
        for (int rep = 0; rep < 2; rep++) k<<<1, warps * 32>>>(out, cyc, 1);
        cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
        double a = 0, b = 0;
        for (int w = 0; w < warps; w++) {
            a += h[2 * w];
            b += h[2 * w + 1];
        }
        printf("%2d warps on one SM: SHFL.32 %.2f cycles per instruction per warp (SM: %.2f per cycle), LDS.64 %.2f (+0.75 DADD)\n",
               warps, a / warps / 4096, warps * 4096.0 / (a / warps), b / warps / 4096);
    }
    return 0;
}
