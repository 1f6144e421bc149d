// assemble.cu -- cell-centred finite-volume assembly of the 7-point
// diffusion operator from a cellwise kappa field, on the device.
//
// Restates the reference's _assemble_kernel
// (/root/reference/pkg/src/ntdprecon/problem_gen.py:87-133)
// with the same operation order, exactly rounded, so the bands are bitwise
// the reference's:
//   face(kc, kn) = 2*kc*kn / (kc + kn)          (problem_gen.py:98)
//   off-diagonal  = -face, diagonal = sum of the faces in the order
//   x-, x+, y-, y+, z-, z+; a Dirichlet boundary face adds the cell's kappa
//   at its place in that sum, a Neumann face (BASELINE config 2) adds nothing.
// The reference hard-wires Dirichlet on all six faces; `dirichlet` is a bit
// mask (bit 0 x-, 1 x+, 2 y-, 3 y+, 4 z-, 5 z+).
#include "common.cuh"

namespace asmb {

__device__ __forceinline__ double face(double kc, double kn)
{
    return __ddiv_rn(mul_rn(mul_rn(2.0, kc), kn), add_rn(kc, kn));
}

// one thread per cell; a (B, 7, N) in the reference band order -nxy,-nx,-1,0,+1,+nx,+nxy
__global__ void k_assemble(const double *__restrict__ kappa, double *__restrict__ a, int nx, int ny, int nz,
                           int dirichlet, i64 batch)
{
    const i64 nxy = (i64)nx * ny, n = nxy * nz;
    for (i64 e = blockIdx.x * (i64)blockDim.x + threadIdx.x; e < n * batch; e += (i64)gridDim.x * blockDim.x) {
        const i64 s = e / n, r = e - s * n;
        const int k = (int)(r / nxy);
        const i64 rr = r - (i64)k * nxy;
        const int j = (int)(rr / nx), i = (int)(rr - (i64)j * nx);
        const double *ks = kappa + s * n;
        const double kc = ks[r];
        double *as = a + s * 7 * n;
        double d = 0.0, c;
        // x-
        c = i > 0 ? face(kc, ks[r - 1]) : 0.0;
        as[2 * n + r] = i > 0 ? -c : 0.0;
        if (i > 0) d = add_rn(d, c);
        else if (dirichlet & 1) d = add_rn(d, kc);
        // x+
        c = i < nx - 1 ? face(kc, ks[r + 1]) : 0.0;
        as[4 * n + r] = i < nx - 1 ? -c : 0.0;
        if (i < nx - 1) d = add_rn(d, c);
        else if (dirichlet & 2) d = add_rn(d, kc);
        // y-
        c = j > 0 ? face(kc, ks[r - nx]) : 0.0;
        as[1 * n + r] = j > 0 ? -c : 0.0;
        if (j > 0) d = add_rn(d, c);
        else if (dirichlet & 4) d = add_rn(d, kc);
        // y+
        c = j < ny - 1 ? face(kc, ks[r + nx]) : 0.0;
        as[5 * n + r] = j < ny - 1 ? -c : 0.0;
        if (j < ny - 1) d = add_rn(d, c);
        else if (dirichlet & 8) d = add_rn(d, kc);
        // z-
        c = k > 0 ? face(kc, ks[r - nxy]) : 0.0;
        as[0 * n + r] = k > 0 ? -c : 0.0;
        if (k > 0) d = add_rn(d, c);
        else if (dirichlet & 16) d = add_rn(d, kc);
        // z+
        c = k < nz - 1 ? face(kc, ks[r + nxy]) : 0.0;
        as[6 * n + r] = k < nz - 1 ? -c : 0.0;
        if (k < nz - 1) d = add_rn(d, c);
        else if (dirichlet & 32) d = add_rn(d, kc);
        as[3 * n + r] = d;
    }
}

}  // namespace asmb

extern "C" int ntd_assemble(const double *kappa, double *a, int64_t nx, int64_t ny, int64_t nz, int64_t dirichlet,
                            int64_t batch, void *stream)
{
    if (!kappa || !a || nx < 1 || ny < 1 || nz < 1 || batch < 1 || dirichlet < 0 || dirichlet > 63)
        return NTD_EINVAL;
    const i64 total = nx * ny * nz * batch;
    i64 blocks = (total + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    asmb::k_assemble<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(kappa, a, (int)nx, (int)ny, (int)nz,
                                                                        (int)dirichlet, batch);
    NTD_CHECK_LAUNCH("ntd_assemble");
}
