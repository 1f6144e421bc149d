// Timing breakdown of the warp-specialised NTD apply (debug aid).
// nvcc -DNTD_TIMING ... micro_apply.cu ../paper_1909_09771_b200/csrc/blas.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "ntd_kernels.cuh"
#include "ntd_apply_sl.cuh"

int main(int argc, char **argv)
{
    const int nx = 96, ny = 96, nz = 96, B = argc > 1 ? atoi(argv[1]) : 8;
    const long n = (long)nx * ny * nz;
    std::vector<double> h(7 * n * B);
    for (long s = 0; s < B; s++)
        for (long i = 0; i < n; i++) {
            double *p = h.data() + s * 7 * n;
            p[i] = -0.15; p[n + i] = -0.15; p[2 * n + i] = -0.1; p[3 * n + i] = -0.1;
            p[4 * n + i] = -0.05; p[5 * n + i] = -0.05; p[6 * n + i] = 0.3;
        }
    double *pre, *b, *x, *w;
    cudaMalloc(&pre, 8 * 7 * n * B); cudaMalloc(&b, 8 * n * B); cudaMalloc(&x, 8 * n * B); cudaMalloc(&w, 8 * n * B);
    cudaMemcpy(pre, h.data(), 8 * 7 * n * B, cudaMemcpyHostToDevice);
    cudaMemset(b, 0, 8 * n * B);
    const int K = 3, LR = sl::lr_of(K);
    const long nsl = (long)ny * nz * LR;
    double *sv, *bs, *xs, *xss;
    const long nrec = (long)ny * nz * sl::recd_of(K); cudaMalloc(&sv, 8 * nrec * B); cudaMalloc(&bs, 8 * nsl * B); cudaMalloc(&xs, 8 * nsl * B); cudaMalloc(&xss, 8 * nsl * B);
    double *zp; cudaMalloc(&zp, 8 * ny * LR); cudaMemset(zp, 0, 8 * ny * LR);
    std::vector<double> hs(nrec * B);
    for (long i = 0; i < nrec * B; i++) { long o = i % sl::recd_of(K); hs[i] = o < 2 * LR ? -0.05 : (o < sl::blk_of(K) ? 0.01 : -0.03); }
    cudaMemcpy(sv, hs.data(), 8 * nrec * B, cudaMemcpyHostToDevice);
    cudaMemset(bs, 0, 8 * nsl * B); cudaMemset(xs, 0, 8 * nsl * B); cudaMemset(xss, 0, 8 * nsl * B);
    constexpr int D = sl::depth_of(3);
    size_t smem = (size_t)4 * D * sl::stage_of(K) * 8;
    cudaFuncSetAttribute(sl::k_apply<3, D, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    sl::k_apply<3, D, 2><<<B, 256, smem>>>(sv, bs, xs, xss, zp, nx, ny, nz, nullptr);
    cudaDeviceSynchronize();
#ifdef NTD_TIMING
    unsigned long long zero[64] = {0};
    cudaMemcpyToSymbol(g_ntd_timing, zero, sizeof(zero));
#endif
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    sl::k_apply<3, D, 2><<<B, 256, smem>>>(sv, bs, xs, xss, zp, nx, ny, nz, nullptr);
    cudaEventRecord(e1);
    cudaDeviceSynchronize();
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("apply %.3f ms  err=%s\n", ms, cudaGetErrorString(cudaGetLastError()));
#ifdef NTD_TIMING
    unsigned long long t[8][8];
    cudaMemcpyFromSymbol(t, g_ntd_timing, sizeof(t));
        const char *names[] = {"top", "lds+rhs", "solve", "store", "wlow", "wup<8", "wpro", "wup>=8"};
    double steps = 9409.0 / 1.0;
    for (int w = 0; w < 4; w++) {
        printf("warp %d:", w);
        for (int k = 0; k < 8; k++) printf(" %s=%.0f", names[k], t[w][k] / steps);
        printf("  (cycles per line-step, /9409)\n");
    }
#endif
    return 0;
}
