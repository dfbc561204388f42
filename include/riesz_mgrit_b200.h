/*
 * riesz_mgrit_b200 -- C ABI of the B200 hot path of non-intrusive MGRIT for
 * 2-D Riesz space-fractional diffusion (arXiv 1805.06688).
 *
 * The reference (riesz_mgrit 0.1.0, pure Python) has no FFI: its hot path sits
 * behind duck-typed Python objects.  Each entry point below replaces one of
 * those objects/functions; the citation names the reference interface
 * (paths relative to riesz_mgrit/).  The Python mirror of the reference API
 * (paper_1805_06688_b200/) binds these with ctypes.
 *
 * Conventions
 *  - all functions return 0 on success or a negative RM_E* code; the text of
 *    the last error is available from rm_last_error();
 *  - vectors are FP64, interior nodes x-fastest ([ny][nx], mesh.py:20-58);
 *    space-time arrays are [N+1][ndof] rows with a caller-given row stride;
 *  - every pointer argument named d_* is a device pointer owned by the caller;
 *    `stream` is a cudaStream_t (NULL = legacy default stream); calls are
 *    asynchronous and never allocate on the hot path;
 *  - no torch types cross this boundary.
 */
#ifndef RIESZ_MGRIT_B200_H
#define RIESZ_MGRIT_B200_H

#include <stdint.h>

#if defined(__GNUC__)
#define RM_API __attribute__((visibility("default")))
#else
#define RM_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define RM_OK 0
#define RM_EINVAL (-1)   /* bad argument (reference: ValueError) */
#define RM_ECUDA (-2)    /* CUDA runtime error */
#define RM_EUNSUP (-3)   /* size not supported by the compiled kernels */

/* CG failure codes reported through rm_fail_info (krylov.py:23-29, 60-63, 69-70, 87-92) */
#define RM_CG_BREAKDOWN 1 /* p'Ap <= 0 or non-finite */
#define RM_CG_NONFINITE 2 /* non-finite residual */
#define RM_CG_BUDGET 3    /* max_iter exhausted */

typedef struct rm_grid rm_grid;

/* Library version string. */
RM_API const char* rm_version(void);
/* Text of the last error on this thread. */
RM_API const char* rm_last_error(void);
/* Largest padded grid order (max(nx, ny) rounded up) the kernels support. */
RM_API int rm_max_order(void);

/*
 * Operator context of one spatial grid: mass, x- and y-stiffness in
 * block-tridiagonal-Toeplitz form.  Replaces the construction in
 * assembly.py:254-274 (mass_operator / stiffness_operator_x / _y) and the
 * cached dense Toeplitz blocks of ToeplitzGenerator.dense (assembly.py:58-60).
 *   t1x_col[nx], t1x_row[nx]  first column / row of the diagonal Toeplitz block along x
 *                             (A1, symmetric for the stiffness operator)
 *   t2x_col[nx], t2x_row[nx]  first column / row of the off-diagonal block (A2) along x
 *   t1y_*, t2y_*              the same along y (length ny)
 *   sx, sy             stiffness prefactors (assembly.py:259-274)
 *   kx, ky             diffusion coefficients (stepper.py:37-58)
 *   mass_scale         hx*hy/12 (assembly.py:172-187)
 * Host pointers; the context uploads generator tables to the current device.
 */
RM_API int rm_grid_create(int nx, int ny, const double* t1x_col, const double* t1x_row, const double* t2x_col,
                   const double* t2x_row, const double* t1y_col, const double* t1y_row, const double* t2y_col,
                   const double* t2y_row, double sx, double sy, double kx, double ky, double mass_scale,
                   rm_grid** out);
RM_API int rm_grid_destroy(rm_grid* grid);

/*
 * Batched operator apply, out[b] = op(dt[b]) v[b] for b < batch.
 * which = 0: combined step operator M + sign*dt/2*(kx Ax + ky Ay)
 *            (CombinedStepOperator.apply, assembly.py:155-161);
 *       = 1: mass M (BttbOperator.apply on mass_operator, assembly.py:100-115);
 *       = 2: x-stiffness Ax;  = 3: y-stiffness Ay (dt, sign ignored for 1..3).
 * d_dt: device array [batch] (may be NULL for which != 0).
 */
RM_API int rm_apply_batched(const rm_grid* grid, int which, int batch, const double* d_dt, int sign,
                     const double* d_v, int64_t v_stride, double* d_out, int64_t out_stride, void* stream);

/*
 * Sweep of propagation chains (the MGRIT relaxation / restriction / residual
 * hot path).  One chain c < nchains runs the time steps
 *     n = first + c*cstride, ..., min(first + c*cstride + clen - 1, nmax)
 * sequentially; chains are independent and run concurrently.  Step n solves
 *     [M + dt_n/2 K] x = b_n,   dt_n = d_dt[n-1],
 *     b_n = (explicit ? (M - dt_n/2 K) in_n : 0) + (d_f ? fs_n * F_n : 0),
 *     fs_n = d_fscale ? d_fscale[n] : 1,  F_n = d_f + n*f_stride (f_stride may be 0),
 * by CG with the reference stopping rule (krylov.py:32-92), starting from
 *     x0 = 0 (x0_mode 0), in_n (x0_mode 1, the warm start of
 *     Discretization.propagate, stepper.py:124-127) or d_x0 + n*x0_stride (x0_mode 2),
 * then forms y_n = [d_gadd ? G_n + x : x] - [d_sub ? S_n : 0] and stores
 *     d_out + (n / out_div) * out_stride  <- y_n            (if d_out)
 *     d_norms[n / out_div]                <- y_n . y_n      (if d_norms)
 *     d_keep + (n / out_div) * keep_stride <- y_n + S_n      (if d_keep)
 * The input of the first step of a chain is d_src + (n-1)*src_stride; later
 * steps take the previous step's output (requires d_out and out_div == 1).
 * Replaces: f_relax / c_relax (mgrit.py:147-165), restrict_residual (:174-182),
 * exact_solve (:192-197), the residual sweep of _global_residual (:253-273),
 * rhs_vector (stepper.py:142-146), sequential_solve (:173-184) and
 * spacetime_residual (:187-205), each as one launch.
 * d_counters[0] += number of spatial solves, d_counters[1] += CG iterations
 * (Discretization.spatial_solves / cg_iterations, stepper.py:95-96,114,121),
 * d_counters[2] += FP64 operator applies performed, d_counters[3] += preconditioner applications,
 * d_counters[4] += split-FP16 operator applies (lp_matvec) (FLOP accounting; the array must hold 5
 * counters).
 * A CG failure is recorded in the grid's failure slot (rm_fail_info).
 */
typedef struct rm_sweep {
  int nchains, first, cstride, clen, nmax;
  int explicit_rhs; /* 0/1 */
  int x0_mode;      /* 0 zero, 1 warm (in_n), 2 d_x0; 3 = preconditioner probe: x = P^-1 b_n, no CG
                       (needs precond > 0; grids up to 127^2); 4 = split-FP16 apply probe: x = (M + s K) b
                       through the in-iteration apply (needs precond 2 and lp_matvec; 63^2 .. 127^2) */
  int out_div;
  const double* d_dt;
  const double* d_src;
  int64_t src_stride;
  const double* d_x0;
  int64_t x0_stride;
  const double* d_f;
  int64_t f_stride;
  const double* d_fscale;
  const double* d_gadd;
  int64_t gadd_stride;
  const double* d_sub;
  int64_t sub_stride;
  double* d_out;
  int64_t out_stride;
  double* d_norms;
  double rel_tol;
  int64_t max_iter; /* <= 0: 10*ndof (CgOptions default, krylov.py:12-20) */
  unsigned long long* d_counters;
  int group;   /* CTAs per chain (cluster size); 0 = library choice */
  int precond; /* 0: plain CG (the reference algorithm); 1: tau-preconditioned CG (needs
                  rm_grid_set_tau), DST stages in FP64 (255^2 FFT kernel: FP32 FFTs); 2: the same
                  preconditioner with its DST stages on FP16 tensor cores (scaled, FP32 accumulation;
                  square grids, others run 1; 255^2 FFT kernel: tcgen05.mma GEMMs with the DST matrix
                  resident in tensor memory, RM_FFT_TC=0 falls back to 1);
                  all stop on ||b - A x|| <= rel_tol ||b|| in FP64 */
  /* optional second starting guess x0' = guess_n - G_n (G_n only when d_gadd): the solve starts
     from whichever of x0, x0' has the smaller initial residual (e.g. the iterate value this step
     is about to overwrite).  NULL: off. */
  const double* d_guess;
  int64_t guess_stride;
  /* optional: also write the step result before the subtraction, [G_n +] x, to d_keep[n / out_div]
     (the residual sweep keeps the C-relaxation values the next cycle would recompute).  NULL: off. */
  double* d_keep;
  int64_t keep_stride;
  /* 1: inside the PCG iteration (precond 2), apply the operator to the search direction as a three-term
     split-FP16 tensor-core product (~2^-22 relative; rm_device.cuh Mx), every stopping decision still on
     the FP64 true residual; grids 63^2 .. 127^2.  255^2 (FFT kernel, precond 2): the in-iteration applies run
     through FP32 FFTs once |r| <= 1e-6 |b| (RM_FFT_LP_THR), acceptance on the FP64 true residual as always.
     Other grids ignore the flag.  0: FP64 throughout. */
  int lp_matvec;
  /* optional (explicit_rhs chains): rows n = (M + dt_n/2 K) G_n, dt_n = d_dt[n-1], of the G added in the
     epilogue (d_gadd; zero rows if none).  Inside a chain the next step's explicit side then follows from
     the accepted solve without an operator apply (the step's input is y = x + G):
       (M - s K) y = (1 + s/s0) M y - (s/s0) (b - r + (M + s0 K) G).   NULL: apply as usual. */
  const double* d_hg;
  int64_t hg_stride;
  /* optional: A x = b - r of every accepted solve (r the FP64 true residual) to d_ax[n / out_div]; the
     setup sweep G_n = A^-1 F_n thereby yields the d_hg rows of the fine level without an apply.  NULL: off. */
  double* d_ax;
  int64_t ax_stride;
  /* optional (with d_guess): rows n = A x0' for the second guess x0' = guess_n [- G_n], i.e. the d_ax of the
     accepted solve that last wrote that point with the same operator and G: the guess' initial residual
     then needs no apply.  NULL: applied. */
  const double* d_gax;
  int64_t gax_stride;
  /* optional (with d_hg): rows n = A x of the accepted solve that wrote input point n (y = x + G): a chain's
     first explicit side then needs no apply either, (M - s K) y = (1 + s/s0) M y - (s/s0)(A x + A G).
     NULL: applied. */
  const double* d_ain;
  int64_t ain_stride;
  /* optional: compressed G (uniform steps, time-separable source: G_n = tau_n A^-1 M g): every row n of
     d_gadd and of d_hg is scaled by d_gscale[n] (pass them with stride 0 to store one vector each; the
     reference computes G_n = rhs_vector(n) one solve at a time, mgrit.py:131-134).  NULL: rows as stored. */
  const double* d_gscale;
} rm_sweep;

RM_API int rm_sweep_run(rm_grid* grid, const rm_sweep* sweep, void* stream);

/*
 * Install the tau (sine-transform) preconditioner: P(s) = (S_y (x) S_x) diag(dm + s*dk) (S_y (x) S_x)
 * with S the orthonormal DST-I matrices; dm, dk are host arrays [ny*nx] (x fastest), the diagonal of
 * the mass and stiffness parts of (S(x)S) A (S(x)S) (paper_1805_06688_b200/precond.py).  Extension of
 * cg_solve (krylov.py:32-92): same stopping rule, fewer iterations.
 */
RM_API int rm_grid_set_tau(rm_grid* grid, const double* dm, const double* dk);

/*
 * First CG failure since the last rm_fail_reset: returns 1 and fills
 * (code, time index n, iterations, residual norm) if one occurred, else 0.
 * Synchronous (reads a few bytes from the device).
 */
RM_API int rm_fail_info(rm_grid* grid, int* code, int* n, int64_t* iterations, double* residual_norm);
RM_API int rm_fail_reset(rm_grid* grid, void* stream);

/*
 * Execution flags chosen for a grid (no reference counterpart; informational):
 * bit 0 / bit 1 = the off-diagonal x / y Toeplitz segments of the matvec run merged
 * (T2 first column == first row shifted by one, as for the Riesz stiffness, assembly.py:239-249),
 * which cuts the matvec from 12 n^3 to 8 n^3 FLOPs; bit 2 = sweeps run the FFT chain kernel (255^2 grids:
 * operator applies and tau-preconditioner DSTs by 512-point FP64 FFTs; RM_NO_FFT=1 selects the dense DMMA
 * kernel instead).  Returns the flags, or -1 for a null grid.
 */
RM_API int rm_grid_flags(const rm_grid* grid);

/* Debug: per-phase cycle counters of CTA 0 (filled only by -DRM_TIMING builds). */
RM_API int rm_debug_timing(rm_grid* grid, long long* out16);

/*
 * coarse_correct (mgrit.py:185-189): U[k*m] += Uc[k] for k <= nc.
 */
RM_API int rm_correct(int ndof, int nc, int m, double* d_u, int64_t u_stride, const double* d_uc, int64_t uc_stride,
               void* stream);

/*
 * Squared Euclidean norm of a - b into d_out[0] (deterministic order).
 * Used for the initial-value term of _global_residual (mgrit.py:262).
 */
RM_API int rm_diff_sqnorm(int64_t n, const double* d_a, const double* d_b, double* d_out, void* stream);

/*
 * Vector algebra of cg_solve for an ARBITRARY operator (krylov.py:44: `op.apply` or a bare callable; the
 * reference's tests pass dense SPD matrices): d_out[0] = a . b in a fixed summation order, and
 * out = alpha x + beta y (out may alias x or y).  The package's own step operator never takes this route: its
 * CG runs fused inside the chain kernels (rm_sweep_run).
 */
RM_API int rm_vec_dot(int64_t n, const double* d_a, const double* d_b, double* d_out, void* stream);
RM_API int rm_vec_axpby(int64_t n, double alpha, const double* d_x, double beta, const double* d_y, double* d_out,
                        void* stream);

/*
 * numpy PCG64 uniform doubles, bit-identical to
 * np.random.default_rng(seed).random(): draw number (start + i) is written to
 * d_out[(i / row) * out_stride + i % row] for i < count.  state/inc are the
 * 128-bit PCG64 state and increment (bit_generator.state) split in 64-bit
 * halves.  Replaces the initial guess of solve() (mgrit.py:291-292).
 */
RM_API int rm_pcg64_uniform(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo, int64_t start,
                     int64_t count, int64_t row, double* d_out, int64_t out_stride, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* RIESZ_MGRIT_B200_H */
