// Latency + numerics of the two-sided line solve (ntd_line_ts.cuh) against a
// host Thomas solve (long double), on a dependent line-to-line chain.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_1909_09771_b200/csrc -o /tmp/micro_line_ts tools/micro_line_ts.cu
#include <cmath>
#include <cstdio>
#include <vector>
#include "ntd_line_ts.cuh"

template <int K>
__global__ void __launch_bounds__(32, 1) k_ts(const double *eFg, const double *eBg, const double *rhog, double *xg, long long *cyc, int iters)
{
    const int lane = threadIdx.x & 31;
    double eF[K], eB[K], rho[K], x[K];
    for (int k = 0; k < K; k++) {
        eF[k] = eFg[lane * K + k];
        eB[k] = eBg[lane * K + k];
        rho[k] = rhog[lane * K + k];
    }
    const PrepTS P = ts::line_prep<K>(lane, eF, eB);
    ts::line_solve<K>(P, lane, eF, eB, rho, x);
    for (int k = 0; k < K; k++) xg[lane * K + k] = x[k];
    double c[K];
    for (int k = 0; k < K; k++) c[k] = rho[k];
    long long t0 = clock64();
    for (int it = 0; it < iters; it++) {
        ts::line_solve<K>(P, lane, eF, eB, c, x);
#pragma unroll
        for (int k = 0; k < K; k++) c[k] = fma(-0.1 * eF[k], x[k], rho[k]);
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
    xg[32 * K + lane] = x[0];
}

template <int K>
void run(int n, double dom)
{
    const int NS = 32 * K;
    std::vector<double> d(n), l(n), u(n), r(n), de(n), ga(n), nu(n), eF(NS, 0.0), eB(NS, 0.0), rho(NS, 0.0), xr(n);
    unsigned s = 12345u + n;
    auto rnd = [&]() { s = s * 1664525u + 1013904223u; return (s >> 8) / 16777216.0; };
    for (int j = 0; j < n; j++) {
        const double kl = std::pow(10.0, 6 * rnd() - 3), kr = std::pow(10.0, 6 * rnd() - 3);
        l[j] = j ? -kl : 0.0;
        u[j] = j < n - 1 ? -kr : 0.0;
        r[j] = 2 * rnd() - 1;
    }
    for (int j = 0; j + 1 < n; j++) l[j + 1] = u[j];  // symmetric
    for (int j = 0; j < n; j++) d[j] = -(l[j] + u[j]) * (1.0 + dom) + dom * 1e-3;
    de[0] = d[0];
    for (int j = 1; j < n; j++) de[j] = d[j] - l[j] * u[j - 1] / de[j - 1];
    ga[n - 1] = d[n - 1];
    for (int j = n - 2; j >= 0; j--) ga[j] = d[j] - u[j] * l[j + 1] / ga[j + 1];
    for (int j = 0; j < n; j++) nu[j] = de[j] + ga[j] - d[j];
    for (int j = 0; j < n; j++) {
        const double mu = 1.0 / nu[j];
        eF[j] = j ? -l[j] * mu * nu[j - 1] / de[j - 1] : 0.0;
        eB[j] = j < n - 1 ? -u[j] * mu * nu[j + 1] / ga[j + 1] : 0.0;
        rho[j] = mu * r[j];
    }
    {  // Thomas in long double
        std::vector<long double> cp(n), dp(n);
        cp[0] = u[0] / (long double)d[0];
        dp[0] = r[0] / (long double)d[0];
        for (int j = 1; j < n; j++) {
            const long double m = d[j] - l[j] * cp[j - 1];
            cp[j] = u[j] / m;
            dp[j] = (r[j] - l[j] * dp[j - 1]) / m;
        }
        long double xn = dp[n - 1];
        xr[n - 1] = (double)xn;
        for (int j = n - 2; j >= 0; j--) {
            xn = dp[j] - cp[j] * xn;
            xr[j] = (double)xn;
        }
    }
    double *g[4];
    long long *cyc, c1;
    for (auto &p : g) cudaMalloc(&p, (NS + 32) * 8);
    cudaMalloc(&cyc, 8);
    cudaMemcpy(g[0], eF.data(), NS * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(g[1], eB.data(), NS * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(g[2], rho.data(), NS * 8, cudaMemcpyHostToDevice);
    const int IT = 20000;
    for (int rep = 0; rep < 2; rep++) k_ts<K><<<1, 32>>>(g[0], g[1], g[2], g[3], cyc, IT);
    std::vector<double> x(NS);
    cudaMemcpy(x.data(), g[3], NS * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(&c1, cyc, 8, cudaMemcpyDeviceToHost);
    double err = 0, nrm = 0;
    for (int j = 0; j < n; j++) {
        err = std::fmax(err, std::fabs(x[j] - xr[j]));
        nrm = std::fmax(nrm, std::fabs(xr[j]));
    }
    for (int j = n; j < NS; j++) err = std::fmax(err, std::fabs(x[j]));
    printf("K=%2d n=%3d dom=%.0e  max err/max|x| = %.2e   two-sided %.1f cycles/line   (%s)\n", K, n,
           dom, err / nrm, (double)c1 / IT, cudaGetErrorString(cudaGetLastError()));
    for (auto &p : g) cudaFree(p);
    cudaFree(cyc);
}

int main()
{
    for (double dom : {1.0, 1e-4}) {
        run<1>(32, dom);
        run<1>(17, dom);
        run<2>(64, dom);
        run<3>(96, dom);
        run<3>(95, dom);
        run<4>(128, dom);
        run<6>(180, dom);
        run<11>(350, dom);
    }
    return 0;
}
