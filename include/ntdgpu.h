/*
 * ntdgpu.h -- C ABI of the B200-native NTD-PCG hot path (libntdgpu.so).
 *
 * Drop-in boundary for the reference package `ntdprecon`
 * (/root/reference/pkg/src/ntdprecon).  Every entry point replaces one numba
 * kernel family of the reference (cited per function) and is bound from
 * Python with ctypes by paper_1909_09771_b200/_lib.py.
 *
 * Conventions
 *  - All array pointers are DEVICE pointers (fp64 unless stated), batch-major:
 *      banded operator / factor arrays  (B, 7, N)   system stride 7N, band stride N
 *      vectors                          (B, N)      system stride N
 *    with N = nx*ny*nz and row r = i + nx*j + nx*ny*k (i fastest), exactly the
 *    reference layout (banded_core.py:36-62).  Band order of an operator:
 *    -nxy,-nx,-1,0,+1,+nx,+nxy (banded_core.py:44).  Band order of an NTD
 *    factor: l1,u1,l2,u2,l3,u3,m_recip (ntd_factor.py:461).
 *  - `active` (int32[B], device, may be NULL = all active): systems with
 *    active[s]==0 are skipped by the kernel (their outputs are untouched).
 *  - Output arrays must not alias input arrays of the same call (the kernels
 *    are compiled with restrict-qualified pointers).
 *  - `stream` is a cudaStream_t; every call only enqueues work on it (no host
 *    synchronisation).  Results are bitwise run-to-run deterministic.
 *  - Return value: 0 on success, NTD_EINVAL for bad arguments, NTD_ENOTSUP for
 *    a grid the kernels were not instantiated for, NTD_ELAUNCH if the launch
 *    failed (ntd_last_error() has the CUDA message).
 *  - Factorisation failures are reported on the device in `status`
 *    (int64[B][3] = code, plane, row); code 0 ok, 1 zero/non-finite pivot,
 *    2 non-finite filter weight, 3 non-finite sandwich adjustment -- the
 *    reference's FactorizationError cases (ntd_factor.py:91-109,133-134,
 *    247-248,383-386,397-399; ilu0.py:80-83,153-155).
 */
#ifndef NTDGPU_H
#define NTDGPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NTD_OK 0
#define NTD_EINVAL (-1)
#define NTD_ENOTSUP (-2)
#define NTD_ELAUNCH (-3)

/* Library identification and the last CUDA error message (host string). */
const char *ntd_version(void);
const char *ntd_last_error(void);

/* Largest nx the line kernels are instantiated for. */
int64_t ntd_max_nx(void);

/* Cell-centred finite-volume assembly of the 7-point operator a (B,7,N) from
 * a cellwise kappa (B,N) (problem_gen.py:87-133 _assemble_kernel, same
 * operation order: bitwise).  dirichlet: bit mask of the Dirichlet faces
 * (bit 0 x-, 1 x+, 2 y-, 3 y+, 4 z-, 5 z+; 63 = the reference's all-Dirichlet);
 * a Neumann face adds nothing to the diagonal. */
int ntd_assemble(const double *kappa, double *a, int64_t nx, int64_t ny,
                 int64_t nz, int64_t dirichlet, int64_t batch, void *stream);

/* y = A x, bitwise equal to the reference (banded_core.py:95-130, spmv /
 * _spmv_kernel): same summation order, no FMA contraction. */
int ntd_spmv(const double *a, const double *x, double *y, int64_t nx,
             int64_t ny, int64_t nz, int64_t batch, const int32_t *active,
             void *stream);

/* t = r - A w (precond_pcg.py:58,62: `r - spmv(a, w)`), bitwise. If
 * z_out != NULL the operand is w + v (formed on the fly, bitwise equal to
 * numpy's `z = v; z += w`, precond_pcg.py:61) and is also stored to z_out. */
int ntd_residual(const double *a, const double *r, const double *w,
                 const double *v, double *z_out, double *t, int64_t nx,
                 int64_t ny, int64_t nz, int64_t batch, const int32_t *active,
                 void *stream);

/* Symmetric packed operator for the PCG-side stencil kernels.  a4 (B,4,N)
 * receives the bands 0,+1,+nx,+nxy of a; sym_ok[s] (int32, set to 1 by the
 * caller) is cleared when any mirrored pair A[r][r-d] / A[r-d][r] of system s
 * differs bitwise.  For systems with sym_ok == 1 the *_sym entry points below
 * read A[r][r-d] as A[r-d][r] and are bitwise equal to their 7-band forms
 * (same summation order, banded_core.py:105-117) while moving 32 instead of
 * 56 operator bytes per row.  The BASELINE operators (harmonic-mean faces,
 * problem_gen.py:98) are bitwise symmetric. */
int ntd_sym_pack(const double *a, double *a4, int32_t *sym_ok, int64_t nx,
                 int64_t ny, int64_t nz, int64_t batch, void *stream);
int ntd_residual_sym(const double *a4, const double *r, const double *w,
                     const double *v, double *z_out, double *t, int64_t nx,
                     int64_t ny, int64_t nz, int64_t batch,
                     const int32_t *active, void *stream);

/* out[s] = x_s . y_s (banded_core.py:133-136 dot / 146-147 norm2 when x==y,
 * fixed-order tree reduction).  work: >= ntd_dot_work_doubles(batch).  If
 * sqrt_out != 0 the square root is stored (norm2). */
int64_t ntd_dot_work_doubles(int64_t batch);
int ntd_dot(const double *x, const double *y, double *out, int sqrt_out,
            int64_t n, int64_t batch, double *work, const int32_t *active,
            void *stream);

/* out = alpha*x + y as a new vector (banded_core.py:139-143 axpy: product
 * rounded, then the sum; bitwise). */
int ntd_axpy(double alpha, const double *x, const double *y, double *out,
             int64_t n, void *stream);

/* chains independent bidiagonal recurrences of n cells each (arrays
 * (chains, n)), chain_bidiagonal_solve (ntd_solve.py:272-300):
 * x[i] = (b[i] - offdiag[i]*x[i_prev]) * diag_recip[i], forward (backward = 0)
 * or backward (1), with the reference's `lanes`-chunk affine composition
 * (_chain_scaled, ntd_solve.py:20-64); bitwise.  work >=
 * ntd_chain_work_doubles(n, chains). */
int64_t ntd_chain_work_doubles(int64_t n, int64_t chains);
int ntd_chain_solve(const double *diag_recip, const double *offdiag,
                    const double *b, double *x, double *work, int64_t n,
                    int64_t chains, int64_t backward, int64_t lanes,
                    void *stream);

/* -------- PCG building blocks (precond_pcg.py:68-122) ------------------
 * Per-system scalar state lives on the device: state (double[B][NTD_ST_N])
 * and flags (int32[B][NTD_FL_N]).  history: double[B][max_iters]. */
enum { NTD_ST_RZ = 0, NTD_ST_PAP, NTD_ST_ALPHA, NTD_ST_BETA, NTD_ST_BNORM,
       NTD_ST_RELRES, NTD_ST_TOL, NTD_ST_N = 8 };
enum { NTD_FL_ACTIVE = 0, NTD_FL_STATUS, NTD_FL_ITERS, NTD_FL_N = 4 };
/* NTD_FL_STATUS values */
enum { NTD_PCG_RUNNING = 0, NTD_PCG_CONVERGED = 1, NTD_PCG_BREAKDOWN = 2,
       NTD_PCG_NONFINITE = 3 };

/* Initialise: x = 0, r = b, bnorm = ||b||; zero rhs => converged at 0
 * iterations (precond_pcg.py:84-90).  active[s] mirrors flags[s][ACTIVE]. */
int ntd_pcg_init(const double *b, double *x, double *r, double *state,
                 int32_t *flags, int32_t *active, double tol, int64_t n,
                 int64_t batch, double *work, void *stream);
/* p = z, rz = r.z (precond_pcg.py:91-94) */
int ntd_pcg_start(const double *r, const double *z, double *p, double *state,
                  const int32_t *active, int64_t n, int64_t batch, double *work,
                  void *stream);
/* ap = A p; pap = p.ap; breakdown check; alpha = rz/pap (precond_pcg.py:98-102) */
int ntd_pcg_spmv_alpha(const double *a, const double *p, double *ap,
                       double *state, int32_t *flags, int32_t *active,
                       int64_t nx, int64_t ny, int64_t nz, int64_t batch,
                       double *work, void *stream);
/* x = alpha p + x; r = -alpha ap + r; relres = ||b - A x||/||b||; history;
 * convergence / non-finite flags (precond_pcg.py:103-114).  xtmp: scratch
 * (B,N) that receives the updated x before the true residual is formed. */
int ntd_pcg_update_residual(const double *a, const double *b, double *x,
                            double *r, const double *p, const double *ap,
                            double *state, int32_t *flags, int32_t *active,
                            double *history, int64_t max_iters, int64_t nx,
                            int64_t ny, int64_t nz, int64_t batch, double *work,
                            void *stream);
/* The same two steps on the symmetric packed operator (see ntd_sym_pack). */
int ntd_pcg_spmv_alpha_sym(const double *a4, const double *p, double *ap,
                           double *state, int32_t *flags, int32_t *active,
                           int64_t nx, int64_t ny, int64_t nz, int64_t batch,
                           double *work, void *stream);
int ntd_pcg_update_residual_sym(const double *a4, const double *b, double *x,
                                double *r, const double *p, const double *ap,
                                double *state, int32_t *flags,
                                int32_t *active, double *history,
                                int64_t max_iters, int64_t nx, int64_t ny,
                                int64_t nz, int64_t batch, double *work,
                                void *stream);
/* rz_new = r.z; beta = rz_new/rz; p = beta p + z (precond_pcg.py:116-119) */
int ntd_pcg_direction(const double *r, const double *z, double *p,
                      double *state, const int32_t *active, int64_t n,
                      int64_t batch, double *work, void *stream);

/* -------- NTD preconditioner -------------------------------------------
 * Setup: the nested twisted filtered factorisation, factor_level3
 * (ntd_factor.py:351-458, incl. the sandwich diagonal shift :387-399).
 * a: (B,7,N) operator; pre: (B,7,N) output; status: int64[B][3]. */
int64_t ntd_factor_work_doubles(int64_t nx, int64_t ny, int64_t nz,
                                int64_t batch);
int ntd_factor(const double *a, double *pre, double *work, int64_t *status,
               int64_t nx, int64_t ny, int64_t nz, int64_t batch, void *stream);

/* Solve records of a factor, derived data for the apply: per grid line, in
 * the apply's lane layout, the elimination multipliers of the two-sided line
 * solve (forward and backward pivots of every cell rebuilt from l1, u1,
 * m_recip by the reference's pivot recurrences, ntd_factor.py:86-110), the
 * factor-only scan coefficients (the reference composes its chain lanes
 * inside _chain_scaled/_chain_unit, ntd_solve.py:20-104) and l2, u2, l3, u3
 * scaled by the per-cell pivot reciprocal mu; mu of every cell follows.
 * solve: >= ntd_solve_doubles (0 = grid served by the direct path; then pass
 * solve = NULL to ntd_apply). */
int64_t ntd_solve_doubles(int64_t nx, int64_t ny, int64_t nz, int64_t batch);
int ntd_solve_bands(const double *pre, double *solve, int64_t nx, int64_t ny,
                    int64_t nz, int64_t batch, void *stream);

/* Apply: x = B^{-1} b, ntd_apply (ntd_solve.py:188-322).  b is not modified.
 * solve: from ntd_solve_bands, or NULL (then formed in work).
 * work: >= ntd_apply_work_doubles. */
int64_t ntd_apply_work_doubles(int64_t nx, int64_t ny, int64_t nz,
                               int64_t batch);
int ntd_apply(const double *pre, const double *solve, const double *b,
              double *x, double *work, int64_t nx, int64_t ny, int64_t nz,
              int64_t batch, const int32_t *active, void *stream);
/* ntd_apply with 1 or 2 CTAs per system (2: the two level-3 halves of each
 * system on two SMs, a thread-block cluster).  Bitwise the same result. */
int ntd_apply_ex(const double *pre, const double *solve, const double *b,
                 double *x, double *work, int64_t nx, int64_t ny, int64_t nz,
                 int64_t batch, const int32_t *active, int64_t ctas_per_system,
                 void *stream);

/* The direct-load apply on the reference band layout (the path every grid
 * without slot-layout records takes: nx > 352, or misaligned buffers),
 * exported so it can be checked against the slot-layout path on any grid.
 * work: >= ntd_apply_work_doubles.  Same result to rounding (<= 1e-10). */
int ntd_apply_direct(const double *pre, const double *b, double *x,
                     double *work, int64_t nx, int64_t ny, int64_t nz,
                     int64_t batch, const int32_t *active, void *stream);

/* Fused combined-preconditioner stages around the NTD apply (the middle of
 * precond_pcg.py:57-65), working on the apply's slot-layout buffers in
 * `work` (>= ntd_apply_work_doubles; zero-filled once by the caller) so the
 * apply needs no layout conversions.  a: the 7-band operator (bands == 7) or
 * the ntd_sym_pack operator (bands == 4).  Available when ntd_solve_doubles
 * is non-zero (NTD_ENOTSUP otherwise).
 *   ntd_residual_to_slot:   b' = (r - A w) * mu into the apply's input (mu: the
 *                           per-cell pivot reciprocals kept in `solve`)
 *   ntd_apply_slot:         the NTD apply of b' (ntd_solve.py:303-322)
 *   ntd_residual_from_slot: z_out = x + w, t = r - A z_out (x: the apply's
 *                           result), bitwise equal to ntd_residual(v = x). */
int ntd_residual_to_slot(const double *a, int64_t bands, const double *solve,
                         const double *r, const double *w, double *work,
                         int64_t nx, int64_t ny, int64_t nz, int64_t batch,
                         const int32_t *active, void *stream);
int ntd_apply_slot(const double *solve, double *work, int64_t nx, int64_t ny,
                   int64_t nz, int64_t batch, const int32_t *active,
                   void *stream);
/* ntd_apply_slot with ctas_per_system = 2: the two level-3 halves of each
 * system run on two SMs (a thread-block cluster), for batches that leave SMs
 * idle. */
int ntd_apply_slot_ex(const double *solve, double *work, int64_t nx,
                      int64_t ny, int64_t nz, int64_t batch,
                      const int32_t *active, int64_t ctas_per_system,
                      void *stream);
int ntd_residual_from_slot(const double *a, int64_t bands, const double *work,
                           const double *r, const double *w, double *z_out,
                           double *t, int64_t nx, int64_t ny, int64_t nz,
                           int64_t batch, const int32_t *active, void *stream);

/* -------- Block ILU0 (ilu0.py) ------------------------------------------
 * Factor of blkdiag(A[:split,:split], A[split:,split:]) on the 7-band
 * pattern, build_block_ilu0 (ilu0.py:34-92,126-156); bitwise equal to the
 * reference.  f: (B,7,N) output.  status: int64[B][3] (code 1, -1, min bad
 * row).  Requires the structured-grid zero pattern of BandedMatrix
 * (banded_core.py:39-42); the Python layer validates it. */
int ntd_ilu0_factor(const double *a, double *f, int64_t split, int64_t *status,
                    int64_t nx, int64_t ny, int64_t nz, int64_t batch,
                    void *stream);
/* z = (LU)^{-1} r per half, ilu0_apply (ilu0.py:95-123,159-169); bitwise.
 * If acc != NULL, acc += z is also formed (precond_pcg.py:64). */
int ntd_ilu0_apply(const double *f, int64_t split, const double *r, double *z,
                   double *acc, int64_t nx, int64_t ny, int64_t nz,
                   int64_t batch, const int32_t *active, void *stream);

/* Skewed-layout ILU0 solves (same arithmetic, bitwise equal; coalesced
 * per-step rows).  Available when split is a multiple of nx*ny:
 * ntd_ilu0_skew_doubles returns 0 otherwise.  coef is built once from the
 * factor f by ntd_ilu0_skew_build; work >= ntd_ilu0_skew_work_doubles.
 * r, z and acc are in the natural (B,N) layout: one kernel gathers r,
 * sweeps in the skewed layout (scratch in work) and writes z and/or
 * acc += z (precond_pcg.py:64) directly. */
int64_t ntd_ilu0_skew_doubles(int64_t nx, int64_t ny, int64_t nz, int64_t batch,
                              int64_t split);
int ntd_ilu0_skew_build(const double *f, double *coef, int64_t split,
                        int64_t nx, int64_t ny, int64_t nz, int64_t batch,
                        void *stream);
int64_t ntd_ilu0_skew_work_doubles(int64_t nx, int64_t ny, int64_t nz,
                                   int64_t batch);
int ntd_ilu0_skew_apply(const double *coef, int64_t split, const double *r,
                        double *z, double *acc, double *work, int64_t nx,
                        int64_t ny, int64_t nz, int64_t batch,
                        const int32_t *active, void *stream);
/* The same with ctas_per_half (1..8) CTAs of warps_per_cta (1..24) warps
 * sweeping each system half as a thread-block cluster, one CTA per SM
 * (progress words in distributed shared memory): more warps in flight and
 * fewer warps per SM sub-partition when the batch leaves SMs idle. */
int ntd_ilu0_skew_apply_ex(const double *coef, int64_t split, const double *r,
                           double *z, double *acc, double *work, int64_t nx,
                           int64_t ny, int64_t nz, int64_t batch,
                           const int32_t *active, int64_t ctas_per_half,
                           int64_t warps_per_cta, void *stream);

/* Hyperplane-synchronous ILU0 solves (same records and arithmetic as the
 * skewed kernels, bitwise equal): every 32-line unit of a half advances one
 * skewed step per barrier, neighbour rows passed through shared memory, so
 * the critical path is the wavefront length instead of progress-word chains.
 * A half runs on ctas_per_half CTAs splitting its planes: 1; 2..16 form a
 * thread-block cluster (boundary rows through distributed shared memory);
 * 17..74 are linked through global memory (boundary-row rings and progress
 * words, a cooperative launch: 2 * batch * ctas_per_half <= 148).  Each CTA
 * has warps_per_cta warps.  ntd_ilu0_hp_units returns the units of the larger
 * half (0: split is not a plane boundary); a CTA's share must be <= 380
 * units and <= 8 units per warp (1 unit per warp: <= 24 warps; 2-8:
 * <= 16 warps).  Two launches (forward, backward). */
int64_t ntd_ilu0_hp_units(int64_t nx, int64_t ny, int64_t nz, int64_t split);
int ntd_ilu0_hp_apply(const double *coef, int64_t split, const double *r,
                      double *z, double *acc, double *work, int64_t nx,
                      int64_t ny, int64_t nz, int64_t batch,
                      const int32_t *active, int64_t ctas_per_half,
                      int64_t warps_per_cta, void *stream);
/* ntd_ilu0_hp_apply with the link mode chosen by the caller: links = 1 a
 * thread-block cluster (<= 16 CTAs per half: boundary rows by DSMEM stores,
 * a cluster barrier per step), 2 global-memory rings with sentinel values
 * (a cluster launch up to 16 CTAs per half, a cooperative launch with
 * 2 * batch * ctas_per_half <= 148 above; what a lone system
 * uses), 0 = 2 above 16 CTAs per half, else 1.  Bitwise the same result. */
int ntd_ilu0_hp_apply_ex(const double *coef, int64_t split, const double *r,
                         double *z, double *acc, double *work, int64_t nx,
                         int64_t ny, int64_t nz, int64_t batch,
                         const int32_t *active, int64_t ctas_per_half,
                         int64_t warps_per_cta, int64_t links, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* NTDGPU_H */
