/*
 * tvdeblur_b200.h -- C ABI of the B200-native PCG hot path of the reference
 * total-variation deblurring solver (tvdeblur, arXiv 1011.5964).
 *
 * The reference is pure Python; its "operator API" is the callable contract
 * of krylov.pcg (reference pkg/src/tvdeblur/krylov.py:82) plus the duck-typed
 * operator objects StructuredBlurOperator (blur.py:197-326),
 * DiffusionOperator (tv.py:74-187), FactoredPreconditioner /
 * assemble_preconditioner (precond.py:419-573) and the fixed-point driver
 * restore (pipeline.py:182-276).  Each entry point below replaces one of
 * those calls; the Python mirror in paper_1011_5964_b200/ binds them with
 * ctypes.
 *
 * Conventions
 *  - Arrays are caller-owned DEVICE buffers, float64, C-contiguous n x n
 *    (row = axis 0) unless stated; the context owns only scratch.
 *  - Inputs are never modified (out may alias nothing it reads unless noted).
 *  - Every call returns an int status; TVD_OK == 0.  tvd_last_error() gives a
 *    thread-local message for the last failure on the calling thread.
 *  - One context = one device + one stream, used by one host thread at a time.
 *    Calls on distinct contexts are reentrant.  Work is enqueued on the
 *    context stream; calls that return host scalars synchronise it.
 */
#ifndef TVDEBLUR_B200_H
#define TVDEBLUR_B200_H

#ifdef __cplusplus
extern "C" {
#endif

#define TVD_ABI_VERSION 3

/* status codes -> exception classes of the reference */
#define TVD_OK 0
#define TVD_ERR_INVALID 1    /* ValueError / ConfigurationError               */
#define TVD_ERR_DIVERGED 2   /* krylov.SolverDivergenceError (krylov.py:31)   */
#define TVD_ERR_INDEFINITE 3 /* krylov.IndefiniteOperatorError (krylov.py:39) */
#define TVD_ERR_PRECOND 4    /* precond.IndefinitePreconditionerError (:60)   */
#define TVD_ERR_SCALING 5    /* pipeline.InvalidScalingError (pipeline.py:60) */
#define TVD_ERR_CUDA 6       /* CUDA runtime failure                          */
#define TVD_ERR_BREAKDOWN 7  /* krylov.SolverBreakdownError (krylov.py:23-30) */

/* blur boundary conditions (blur.py:34-38; only these two are transform-
 * diagonalisable and in scope) */
#define TVD_BC_REFLECTIVE 2
#define TVD_BC_ANTI_REFLECTIVE 3

/* transforms (transforms.py:35-39); ANTI_REFLECTIVE is T = Shat (I + U) with the rank-2
 * border corrections (transforms.py:84-140) and also names the P preconditioner family */
#define TVD_TRANSFORM_DST1 0
#define TVD_TRANSFORM_SINE_HAT 1
#define TVD_TRANSFORM_DCT 2
#define TVD_TRANSFORM_ANTI_REFLECTIVE 3

/* diffusion ghost rules (tv.py:27-39) */
#define TVD_DBC_ZERO_NEUMANN 0
#define TVD_DBC_ANTI_REFLECTIVE 1

/* preconditioner variants of one family (precond.py:516-573) */
#define TVD_VARIANT_X 0   /* |lam_H|^2 + alpha proj(L)                */
#define TVD_VARIANT_D_X 1 /* same eigenvalues, wrapped by sqrt(1+a diag L) */
#define TVD_VARIANT_X_D 2 /* |lam_H|^2 |lam_D|^2 + alpha proj(s L s)     */

/* inner-solve preconditioner kinds (pipeline.py:225-241) */
#define TVD_PRECOND_NONE 0      /* apply_minv = None (identity)          */
#define TVD_PRECOND_DIAG 1      /* w / (1 + alpha diag L)                */
#define TVD_PRECOND_TRANSFORM 2 /* FactoredPreconditioner.apply_inverse  */

typedef struct tvd_ctx tvd_ctx;
typedef struct tvd_blur tvd_blur;

/* system A w = H^T H w + alpha L w   (pipeline.py:209-210), the re-blurred
 * H H w + alpha L w (reblur = 1, pipeline.py:173-174), optionally the diagonally
 * scaled s .* A(s .* w)   (pipeline.py:145-164, selector X_D). */
typedef struct tvd_system {
  tvd_blur* blur;
  double alpha;
  double spacing;
  const double* a_h; /* n x (n+1) horizontal diffusivities */
  const double* a_v; /* (n+1) x n vertical diffusivities   */
  const double* s;   /* NULL or n x n scaling              */
  int bc_l;          /* TVD_DBC_* ghosts of L              */
  int reblur;        /* 1: H H instead of H^T H            */
} tvd_system;

typedef struct tvd_precond {
  int kind;              /* TVD_PRECOND_*                                   */
  int family;            /* TVD_TRANSFORM_SINE_HAT, _DCT or _ANTI_REFLECTIVE */
  const double* inv_eig; /* TRANSFORM: n x n inverse eigenvalues            */
  const double* d;       /* DIAG: divisor; TRANSFORM: d_sqrt (D_X) or NULL  */
} tvd_precond;

int tvd_abi_version(void);
const char* tvd_last_error(void);

/* ---- context ---------------------------------------------------------- */
/* stream: a cudaStream_t (e.g. torch.cuda.current_stream().cuda_stream) or 0 */
int tvd_ctx_create(int device, void* stream, tvd_ctx** out);
int tvd_ctx_set_stream(tvd_ctx* ctx, void* stream);
int tvd_ctx_sync(tvd_ctx* ctx);
int tvd_ctx_destroy(tvd_ctx* ctx);
/* options.  TVD_OPT_GENERIC_FFT (per context) routes DST passes through the generic
 * mixed-radix engine instead of the odd-symmetric prime-factor engine.  The others are
 * process-wide (every context; setting one drops the context's captured solver graphs);
 * their defaults are the measured production configuration:
 *   TVD_OPT_SOLVER_GRAPH  1: replay captured PCG / BiCGstab iterations as CUDA graphs
 *   TVD_OPT_PDL           1: programmatic dependent launch attribute on the iteration kernels
 *   TVD_OPT_BAND_GENERIC  0: prime-core assembly projections on the generic engine, not Rader
 *   TVD_OPT_BAND_SLIDE    0: CUDA-core band passes instead of the fp64 tensor-core ones
 *   TVD_OPT_FIN_FUSION    1: PCG scalar steps folded into their producers' last CTA
 *   TVD_OPT_P_FUSION      1: direction update fused into the row band pass
 *   TVD_OPT_PFA_STAGES    3: (profiling) run only the first k stages of the DST engine
 *   TVD_OPT_GENERAL_BLUR  0: blurs created while set take the general 2D path (explicit
 *                            extension + direct convolution) even when the PSF is rank 1
 *   TVD_OPT_BAND_PREFETCH 0: column band pass prefetches its epilogue operands to L2 (1) / L1 (2)
 *   TVD_OPT_SPLIT_X       0: PCG x update on a second stream, overlapping the M^-1 passes
 *                            (bit-identical; measured no gain)
 *   TVD_OPT_GUARD_SLOTS   0: scratch allocated while set carries 4 KB guard bands checked by
 *                            tvd_ctx_check_guards (debugging: out-of-bounds kernel writes) */
#define TVD_OPT_GENERIC_FFT 1
#define TVD_OPT_SOLVER_GRAPH 2
#define TVD_OPT_PDL 3
#define TVD_OPT_BAND_GENERIC 4
#define TVD_OPT_BAND_SLIDE 5
#define TVD_OPT_FIN_FUSION 6
#define TVD_OPT_P_FUSION 7
#define TVD_OPT_PFA_STAGES 8
#define TVD_OPT_GENERAL_BLUR 9
#define TVD_OPT_BAND_PREFETCH 10
#define TVD_OPT_SPLIT_X 11
#define TVD_OPT_GUARD_SLOTS 12
int tvd_ctx_set_option(tvd_ctx* ctx, int option, int value);
int tvd_ctx_get_option(tvd_ctx* ctx, int option, int* value);
/* bytes of the guard bands of ctx's guarded scratch slots that no longer hold the fill
 * pattern (0 = no out-of-bounds write into the context's scratch) */
int tvd_ctx_check_guards(tvd_ctx* ctx, long long* bad_bytes, int* guarded_slots);
/* instrumentation: kernels launched through ctx so far */
int tvd_ctx_counters(tvd_ctx* ctx, long long* launches);
/* enable (1) / disable (0) CUDA-event timing around every launch; resets records */
int tvd_ctx_profile(tvd_ctx* ctx, int enable);
/* per-category launch time (ms) and launch count since tvd_ctx_profile(ctx, 1) */
int tvd_ctx_profile_read(tvd_ctx* ctx, int ncat, double* total_ms, long long* count);
/* category name for id, NULL past the last */
const char* tvd_profile_category(int id);

/* ---- blur operator H  (blur.py:197-326) -------------------------------- */
/* psf: HOST (2m+1) x (2m+1) quadrantally symmetric, normalised.
 * *separable receives 1 when the PSF is rank-1 (fast banded path). */
int tvd_blur_create(tvd_ctx* ctx, int n, const double* psf, int width, int bc, tvd_blur** out,
                    int* separable);
int tvd_blur_destroy(tvd_blur* blur);
/* exact H (transpose=0, blur.py:226-234) or H^T (transpose=1, blur.py:236-247) */
int tvd_blur_apply(tvd_blur* blur, const double* in, double* out, int transpose);
/* H^T H in  (reflective: H H, pipeline.py:175-176) */
int tvd_blur_normal_apply(tvd_blur* blur, const double* in, double* out);
/* eigenvalue grid lam[s,t] of the fast path (blur.py:265-291) */
int tvd_blur_eigenvalues(tvd_blur* blur, double* lam);

/* ---- TV diffusion  (tv.py:42-175, zero-Neumann) ------------------------ */
int tvd_diffusivity(tvd_ctx* ctx, int n, double beta, double spacing, const double* u, double* a_h,
                    double* a_v);
int tvd_diffusion_apply(tvd_ctx* ctx, int n, double spacing, const double* a_h, const double* a_v,
                        const double* w, double* out);
/* block bands: diag n x n, inner (0,+-1) n x (n-1), block (+-1,0) (n-1) x n */
int tvd_diffusion_bands(tvd_ctx* ctx, int n, double spacing, const double* a_h, const double* a_v,
                        double* diag, double* inner, double* block);
/* the same with a ghost rule TVD_DBC_* (tv.py:27-39); anti-reflective ghosts make the
 * (0,+1)/(0,-1) and (+1,0)/(-1,0) bands differ at one end (inner_lo, block_lo: may be NULL) */
int tvd_diffusivity_bc(tvd_ctx* ctx, int n, double beta, double spacing, int bc_l,
                       const double* u, double* a_h, double* a_v);
int tvd_diffusion_apply_bc(tvd_ctx* ctx, int n, double spacing, int bc_l, const double* a_h,
                           const double* a_v, const double* w, double* out);
int tvd_diffusion_bands_bc(tvd_ctx* ctx, int n, double spacing, int bc_l, const double* a_h,
                           const double* a_v, double* diag, double* inner_up, double* inner_lo,
                           double* block_up, double* block_lo);

/* ---- transforms  (transforms.py:52-171) -------------------------------- */
/* lines of length `len` (rows of a rows x len array when axis == 1, columns
 * of a len x cols array when axis == 0); inverse selects DCT analysis */
int tvd_transform_lines(tvd_ctx* ctx, int kind, int rows, int cols, int axis, const double* in,
                        double* out, int inverse);
/* Anti-reflective transform T (inverse 0, transpose 0), T^-1 (1, 0), T^T (0, 1), T^-T (1, 1)
 * of `rows` contiguous lines of length `cols` >= 5 (reference transforms.py:96-140 ar_apply;
 * the transposes feed the transform-domain blur adjoint, blur.py:302-314).  in == out ok. */
int tvd_ar_lines(tvd_ctx* ctx, int rows, int cols, const double* in, double* out, int inverse,
                 int transpose);
/* X G X^T on a square n x n grid: axis 0 then axis 1 (tensor_apply_2d) */
int tvd_transform_2d(tvd_ctx* ctx, int kind, int n, const double* in, double* out, int inverse);

/* ---- row windows: the FP-step setup of a row slab (slab.slab_operators) ---
 * Diffusivity of the global rows [row_lo, row_hi) of an n x n image (zero-Neumann ghosts):
 * a_h rows [row_lo, row_hi) ((row_hi-row_lo) x (n+1)), a_v rows [row_lo, row_hi]
 * ((row_hi-row_lo+1) x n), from a window u_win of the global rows [win_lo, win_lo+win_rows)
 * that holds the one-row halo.  Bit-identical to the rows of tvd_diffusivity. */
int tvd_diffusivity_rows(tvd_ctx* ctx, int n, double beta, double spacing, const double* u_win,
                         int win_lo, int win_rows, int row_lo, int row_hi, double* a_h,
                         double* a_v);
/* block bands (diag n, inner n-1, block n per row) of the global rows [row_lo, row_hi) from
 * the window's a_h / a_v (as written by tvd_diffusivity_rows); rows of tvd_diffusion_bands */
int tvd_diffusion_bands_rows(tvd_ctx* ctx, int n, double spacing, const double* a_h,
                             const double* a_v, int row_lo, int row_hi, double* diag,
                             double* inner, double* block);
/* one level of the band projection (precond.py:82-199) over nlines contiguous lines of n:
 * b0 the d = 0 band, b1 (nullable; line stride b1_stride, multiplicity c1) the |d| = 1
 * band; epi 0 stores the projection, epi 1 stores lamh^2 + alpha * projection and returns
 * its min / max (host) */
int tvd_band_project_lines(tvd_ctx* ctx, int family, int n, int nlines, const double* b0,
                           const double* b1, int b1_stride, double c1, int epi,
                           const double* lamh, double alpha, double* out, double* min_max);

/* ---- preconditioner  (precond.py:369-573) ------------------------------ */
/* Assemble eigenvalues of kind {R,D_R,R_D} (family DCT) or {M,D_M,M_D}
 * (family SINE_HAT) from the blur eigenvalues and the diffusion bands.
 * eig, inv_eig: n x n out.  dvec: n x n out, d_sqrt for D_X, s for X_D
 * (may be NULL for X).  Host scalars: min/max eigenvalue, clamped count.
 * TVD_ERR_PRECOND when 1 + alpha diag L or the eigenvalues are not > 0
 * (*min_eig then holds the offending minimum). */
int tvd_precond_assemble(tvd_ctx* ctx, int family, int variant, int n, double alpha,
                         const double* lam_h, const double* diag, const double* inner,
                         const double* block, double* eig, double* inv_eig, double* dvec,
                         double* min_eig, double* max_eig, long long* n_clamped);
/* the same assembly with its checks left on the device (no host synchronisation): d_check
 * (4 device doubles) receives [min(1 + alpha diag L), min eigenvalue, max eigenvalue, clamped
 * count] in stream order; the caller reads it when it next synchronises (e.g. after the
 * solve) and raises IndefinitePreconditionerError / logs the clamp warning then.  The
 * eigenvalues and their clamped inverse are those of tvd_precond_assemble (same kernels). */
int tvd_precond_assemble_async(tvd_ctx* ctx, int family, int variant, int n, double alpha,
                               const double* lam_h, const double* diag, const double* inner,
                               const double* block, double* eig, double* inv_eig, double* dvec,
                               double* d_check);
/* z = X (inv_eig .* X^T (r / d_sqrt)) / d_sqrt   (precond.py:456-477) */
int tvd_precond_apply_inverse(tvd_ctx* ctx, int family, int n, const double* inv_eig,
                              const double* d_sqrt, const double* in, double* out);
/* y = d_sqrt .* X (eig .* X^T (d_sqrt .* b))      (precond.py:463-469) */
int tvd_precond_apply(tvd_ctx* ctx, int family, int n, const double* eig, const double* d_sqrt,
                      const double* in, double* out);
/* d = 1 + alpha diag (may be NULL), d_sqrt = sqrt(d), s = d^-1/2 (each nullable);
 * TVD_ERR_SCALING when min d <= 0 (*min_d receives it). */
int tvd_scaling(tvd_ctx* ctx, long long count, double alpha, const double* diag, double* d,
                double* d_sqrt, double* s, double* min_d);

/* ---- system and PCG  (pipeline.py:209-224, krylov.py:82-116) ----------- */
int tvd_system_apply(tvd_ctx* ctx, const tvd_system* sys, const double* in, double* out);
/* Full device-resident PCG.  x receives the solution (may equal x0).
 * history: NULL or device buffer of max_iterations doubles (relative
 * residuals).  On TVD_ERR_DIVERGED / TVD_ERR_INDEFINITE, *err_iteration and
 * *err_value describe the failure as in the reference exceptions. */
int tvd_pcg_solve(tvd_ctx* ctx, const tvd_system* sys, const tvd_precond* pre, const double* b,
                  const double* x0, double* x, double tol, int max_iterations, double* history,
                  int* iterations, int* converged, int* err_iteration, double* err_value);
/* Device-resident right-preconditioned BiCGstab (krylov.py:119-174) for the nonsymmetric
 * systems (re-blurred and / or anti-reflective L).  Same arguments as tvd_pcg_solve; also
 * TVD_ERR_BREAKDOWN (*err_value: 1 rho, 2 shadow angle, 3 stabilizer, 4 omega vanished). */
int tvd_bicgstab_solve(tvd_ctx* ctx, const tvd_system* sys, const tvd_precond* pre,
                       const double* b, const double* x0, double* x, double tol,
                       int max_iterations, double* history, int* iterations, int* converged,
                       int* err_iteration, double* err_value);

/* ---- vector helpers for the generic callable path ---------------------- */
/* valid 2D convolution of an extended T x T device array with a width x width HOST psf
 * (harness.py:170-198, blur_and_observe's convolve2d(u_extended, h, 'valid')); out: device
 * (T-width+1)^2.  Rank-1 PSFs (or caller factors f1 (axis 0), f2 (axis 1), host, both
 * non-NULL) run as two 1D passes, bit-identical to the separable shifted-slice sums
 * sum_b f2[w-1-b] ext[:, b:] then sum_a f1[w-1-a] rows[a:, :]; others as a direct 2D
 * convolution.  Synchronises. */
int tvd_valid_convolve(tvd_ctx* ctx, const double* ext, int T, const double* psf, int width,
                       const double* f1, const double* f2, double* out);

/* ---- row-slab decomposition of one large problem over nranks ranks (config 5).
 * Rank `rank` owns the global rows [rank R, rank R + R), R = n / nranks.  The library runs the
 * kernels of each phase on the context stream; the caller runs the collectives between the
 * phases on the buffers tvd_slab_buffer exposes (paper_1011_5964_b200/slab.py):
 *   start:  MATVEC_ROWS, halo(T_EXT, khalo rows; P_EXT, 1 row), MATVEC_COLS, RESIDUAL,
 *           allgather(CONTRIB -> GATHER), START, precond, allgather, RZ0
 *   iter:   MATVEC_ROWS, halo, MATVEC_COLS, allgather, GAMMA_UPDATE, allgather, REL,
 *           precond, allgather, BETA_P
 *   precond (transform): PREC_ROWS, all-to-all(SEND -> RECV), PREC_COLS, all-to-all,
 *           PREC_FINAL;  (none / diagonal): PREC_ROWS only
 * sys: a_h = the slab's R x (n+1) rows of a_h, a_v = its R+1 rows [rank R, rank R + R] of a_v,
 * s = NULL, reblur = 0, separable PSF (tensor-core band passes, n >= 256).
 * pre: NONE; DIAG (d = slab of the divisor); TRANSFORM (family DST1 / SINE_HAT, inv_eig = rows
 * [rank R, rank R + R) of the TRANSPOSED inverse eigenvalue grid, d = slab of d_sqrt or NULL).
 * Replaces the inner solve krylov.pcg (krylov.py:82-116) for an image split across GPUs. */
typedef struct tvd_slab tvd_slab;
#define TVD_SLAB_MATVEC_ROWS 0
#define TVD_SLAB_MATVEC_COLS 1
#define TVD_SLAB_RESIDUAL 2
#define TVD_SLAB_START 3
#define TVD_SLAB_GAMMA_UPDATE 4
#define TVD_SLAB_REL 5
#define TVD_SLAB_PREC_ROWS 6
#define TVD_SLAB_PREC_COLS 7
#define TVD_SLAB_PREC_FINAL 8
#define TVD_SLAB_RZ0 9
#define TVD_SLAB_BETA_P 10
#define TVD_SLAB_BUF_X 0      /* R x n solution slab                                   */
#define TVD_SLAB_BUF_R 1
#define TVD_SLAB_BUF_Z 2
#define TVD_SLAB_BUF_Q 3
#define TVD_SLAB_BUF_P_EXT 4  /* (R + 2) x n: halo row, p slab, halo row               */
#define TVD_SLAB_BUF_T_EXT 5  /* (R + 2 khalo) x n: halo, t = p G_1^T slab, halo        */
#define TVD_SLAB_BUF_SEND 6   /* n x R all-to-all send blocks (block j -> rank j)      */
#define TVD_SLAB_BUF_RECV 7   /* n x R all-to-all receive blocks (block i <- rank i)   */
#define TVD_SLAB_BUF_CONTRIB 8 /* 1 double: this rank's partial of the current dot     */
#define TVD_SLAB_BUF_GATHER 9 /* nranks doubles: every rank's contribution, rank order */
int tvd_slab_create(tvd_ctx* ctx, const tvd_system* sys, const tvd_precond* pre, int nranks,
                    int rank, tvd_slab** out);
int tvd_slab_destroy(tvd_slab* slab);
/* info[8]: n, R, row_lo, khalo, p halo rows, nranks, rank, preconditioner exchanges (0/1) */
int tvd_slab_info(tvd_slab* slab, int* info);
int tvd_slab_buffer(tvd_slab* slab, int which, double** ptr, long long* count);
/* b, x0: this rank's R x n slabs (b must stay valid during the solve); history: NULL or
 * max_iterations doubles */
int tvd_slab_start(tvd_slab* slab, const double* b, const double* x0, double tol,
                   int max_iterations, double* history);
int tvd_slab_phase(tvd_slab* slab, int phase);
/* synchronises; TVD_ERR_DIVERGED / TVD_ERR_INDEFINITE once a failure ended the solve */
int tvd_slab_status(tvd_slab* slab, int* done, int* iterations, int* converged,
                    int* err_iteration, double* err_value);

int tvd_vec_dot(tvd_ctx* ctx, long long count, const double* x, const double* y, double* out);
/* out = a x + b y */
int tvd_vec_axpby(tvd_ctx* ctx, long long count, double a, const double* x, double b,
                  const double* y, double* out);
/* out = x * y (op 0) or x / y (op 1) */
int tvd_vec_binary(tvd_ctx* ctx, long long count, int op, const double* x, const double* y,
                   double* out);

#ifdef __cplusplus
}
#endif
#endif /* TVDEBLUR_B200_H */
