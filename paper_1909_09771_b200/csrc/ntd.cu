// ntd.cu -- C-ABI entry points of the NTD setup / apply kernels
// (ntd_kernels.cuh); per-K instantiations live in ntd_k<K>.cu so they
// compile in parallel.  K = ceil(nx/32) cells per lane per chain.
#include "ntd_kernels.cuh"

// instantiated K values (ntd_k<K>.cu); a line of nx cells uses the
// smallest instantiated K >= ceil(nx/32).
static const int KS[] = {1, 2, 3, 4, 5, 6, 8, 11, 12, 16};
static constexpr int MAX_K = 16;

static int pick_k(i64 nx)
{
    int need = (int)((nx + 31) / 32);
    for (int k : KS)
        if (k >= need) return k;
    return -1;
}

#define NTD_DISPATCH(FN, ...)            \
    switch (K) {                         \
    case 1: return FN<1>(__VA_ARGS__);   \
    case 2: return FN<2>(__VA_ARGS__);   \
    case 3: return FN<3>(__VA_ARGS__);   \
    case 4: return FN<4>(__VA_ARGS__);   \
    case 5: return FN<5>(__VA_ARGS__);   \
    case 6: return FN<6>(__VA_ARGS__);   \
    case 8: return FN<8>(__VA_ARGS__);   \
    case 11: return FN<11>(__VA_ARGS__); \
    case 12: return FN<12>(__VA_ARGS__); \
    case 16: return FN<16>(__VA_ARGS__); \
    default: return NTD_ENOTSUP;         \
    }

extern "C" int64_t ntd_max_nx(void) { return 32 * MAX_K; }

extern "C" int64_t ntd_apply_work_doubles(int64_t nx, int64_t ny, int64_t nz, int64_t batch)
{
    return nx * ny * nz * batch;
}

extern "C" int ntd_apply(const double *pre, const double *b, double *x, double *work, int64_t nx, int64_t ny,
                         int64_t nz, int64_t batch, const int32_t *active, void *stream)
{
    if (!pre || !b || !x || !work || nx < 1 || ny < 1 || nz < 1 || batch < 1) return NTD_EINVAL;
    int K = pick_k(nx);
    NTD_DISPATCH(launch_apply_k, pre, b, x, work, (int)nx, (int)ny, (int)nz, batch, active, (cudaStream_t)stream);
}

extern "C" int64_t ntd_factor_work_doubles(int64_t nx, int64_t ny, int64_t nz, int64_t batch)
{
    (void)nz;
    return batch * 2 * S_PER_PAIR * nx * ny;
}

extern "C" int ntd_factor(const double *a, double *pre, double *work, int64_t *status, int64_t nx, int64_t ny,
                          int64_t nz, int64_t batch, void *stream)
{
    if (!a || !pre || !work || !status || nx < 1 || ny < 1 || nz < 1 || batch < 1) return NTD_EINVAL;
    int K = pick_k(nx);
    NTD_DISPATCH(launch_factor_k, a, pre, work, status, (int)nx, (int)ny, (int)nz, batch, (cudaStream_t)stream);
}
