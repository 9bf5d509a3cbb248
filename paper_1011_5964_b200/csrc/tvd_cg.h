// PCG state machine and vector kernels (tvd_cg.cu).  Reference: krylov.py:70-116.
#pragma once

#include "tvd_common.cuh"

namespace tvd {

// Error codes (== TVD_ERR_* in include/tvdeblur_b200.h).
enum : int {
  kOk = 0,
  kErrInvalid = 1,
  kErrDiverged = 2,
  kErrIndefinite = 3,
  kErrPrecond = 4,
  kErrScaling = 5,
  kErrCuda = 6,
};

// Device-resident solver state; every iteration kernel returns immediately
// once `done` is set, so the host can enqueue iterations speculatively.
struct PcgState {
  double rz, r0, gamma, step, beta, rel;
  int k;          // current iteration (1-based)
  int done;       // 1 once converged / exhausted / failed
  int status;     // kOk or kErrDiverged / kErrIndefinite
  int err_iter;
  double err_val;
  int iters;
  int converged;
  int x_pending;  // gamma of iteration k accepted, x += step p not yet applied (split update)
};

// ---- scalar steps of the recurrence (krylov.py:99-116), thread 0 of one CTA, given the
// deterministic sum of the per-CTA partials
__device__ __forceinline__ void pcg_fin_gamma(PcgState* s, double pq) {
  s->gamma = pq;
  if (!isfinite(pq)) {
    s->status = kErrDiverged;
    s->err_iter = s->k;
    s->done = 1;
  } else if (pq <= 0.0) {
    s->status = kErrIndefinite;
    s->err_iter = s->k;
    s->err_val = pq;
    s->done = 1;
  } else {
    s->step = s->rz / pq;
    s->x_pending = 1;
  }
}
__device__ __forceinline__ void pcg_fin_rel(PcgState* s, double rr, double tol, double* hist) {
  const double rel = sqrt(rr) / s->r0;
  s->rel = rel;
  if (!isfinite(rel)) {
    s->status = kErrDiverged;
    s->err_iter = s->k;
    s->done = 1;
    return;
  }
  if (hist) hist[s->k - 1] = rel;
  if (rel < tol) {
    s->iters = s->k;
    s->converged = 1;
    s->done = 1;
  }
}
__device__ __forceinline__ void pcg_fin_beta(PcgState* s, double rz_next, int max_it) {
  s->beta = rz_next / s->rz;
  s->rz = rz_next;
  s->k += 1;
  if (s->k > max_it) {
    s->iters = max_it;
    s->converged = 0;
    s->done = 1;
  }
}

// A finalizer folded into the kernel that produces its partials: every CTA writes its
// partial, then the last CTA to finish (threadfence + atomic ticket) sums all partials in
// a fixed order and applies the step.  s == nullptr: the host launches the finalizer.
enum : int { kFinGamma = 1, kFinRel = 2, kFinBeta = 3 };
struct PcgFin {
  PcgState* s;
  unsigned* counter;  // zero between launches (the last CTA resets it)
  int kind;
  int max_it;
  double tol;
  double* hist;
};

// Call from every CTA after thread 0 has stored partial[blockIndex] (all threads).
__device__ __forceinline__ void pcg_fin_tail(const PcgFin& f, const double* partial, int nb,
                                             double* red) {
  __shared__ int last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(f.counter, 1u) == (unsigned)(nb - 1);
  __syncthreads();
  if (!last) return;
  __threadfence();
  double v = 0.0;
  for (int i = threadIdx.x; i < nb; i += blockDim.x) v += __ldcg(partial + i);
  const double sum = block_sum(v, red);
  if (threadIdx.x == 0) {
    if (f.kind == kFinGamma) pcg_fin_gamma(f.s, sum);
    else if (f.kind == kFinRel) pcg_fin_rel(f.s, sum, f.tol, f.hist);
    else pcg_fin_beta(f.s, sum, f.max_it);
    *f.counter = 0u;
  }
}

// ---- right-preconditioned BiCGstab (krylov.py:119-174).  `halt` = done or the early exit
// after the s-residual test; the kernels of the second half-step skip on it, the x / r
// update and the final check only on `done`.
enum : int { kErrBreakdown = 7 };
struct BicgState {
  double rho, alpha, omega, rho_next, beta, r0, rel;
  int k, done, halt, early, status, err_iter;
  double err_val;
  int iters, converged;
};
cudaError_t launch_bicg_start(BicgState* s, const double* partial, int nb, cudaStream_t st);
cudaError_t launch_bicg_rho(BicgState* s, const double* partial, int nb, cudaStream_t st);
cudaError_t launch_bicg_update_p(BicgState* s, double* p, const double* r, const double* v, long N,
                                 cudaStream_t st);
cudaError_t launch_bicg_alpha(BicgState* s, const double* partial, int nb, cudaStream_t st);
cudaError_t launch_bicg_s(BicgState* s, double* sv, const double* r, const double* v, long N,
                          double* partial, cudaStream_t st);
cudaError_t launch_bicg_srel(BicgState* s, const double* partial, double tol, cudaStream_t st);
cudaError_t launch_bicg_omega(BicgState* s, const double* p_ts, int nb_ts, const double* p_tt,
                              int nb_tt, cudaStream_t st);
cudaError_t launch_bicg_update_xr(BicgState* s, double* x, double* r, const double* p_hat,
                                  const double* s_hat, const double* sv, const double* t, long N,
                                  double* partial, cudaStream_t st);
cudaError_t launch_bicg_rel(BicgState* s, const double* partial, double tol, double* hist,
                            int max_it, cudaStream_t st);

cudaError_t launch_sum_partials(const double* partial, int nb, double* out, cudaStream_t st);
cudaError_t launch_residual_init(const double* b, const double* q, double* r, long N, double* partial,
                                 int nb, cudaStream_t st);
cudaError_t launch_pcg_start(PcgState* s, const double* partial, int nb, cudaStream_t st);
cudaError_t launch_pcg_rz0(PcgState* s, const double* partial, int nb, cudaStream_t st);
cudaError_t launch_copy(const double* src, double* dst, long N, const int* skip, cudaStream_t st);
cudaError_t launch_pcg_gamma(PcgState* s, const double* partial, int nb, cudaStream_t st);
cudaError_t launch_pcg_update_xr(PcgState* s, double* x, double* r, const double* p, const double* q,
                                 long N, double* partial, int nb, cudaStream_t st,
                                 const PcgFin* fin = nullptr);
cudaError_t launch_pcg_rel(PcgState* s, const double* partial, int nb, double tol, double* hist,
                           cudaStream_t st);
cudaError_t launch_pcg_beta(PcgState* s, const double* partial, int nb, int max_it, cudaStream_t st);
cudaError_t launch_pcg_update_p(PcgState* s, double* p, const double* z, long N, cudaStream_t st);
// split x / r update: r -= step q with r.r and the stop test (critical path), and
// x += step p (off the critical path: another stream overlaps it with the preconditioner
// passes; it applies iff iteration k's gamma was accepted, x_pending, which its last CTA
// clears through `counter`).  Same arithmetic and r.r partials as k_pcg_update_xr.
cudaError_t launch_pcg_update_r(PcgState* s, double* r, const double* q, long N, double* partial,
                                cudaStream_t st, const PcgFin* fin);
cudaError_t launch_pcg_update_x(PcgState* s, double* x, const double* p, long N, unsigned* counter,
                                cudaStream_t st);
cudaError_t launch_diag_solve(const double* r, const double* d, double* z, long N, double* partial,
                              int nb, const int* skip, cudaStream_t st);
cudaError_t launch_dot_partials(const double* x, const double* y, long N, double* partial, int nb,
                                const int* skip, cudaStream_t st);
// out = a * x + b * y  (numpy order: (a*x) + (b*y); a or b == 1 skips the multiply)
cudaError_t launch_axpby(double a, const double* x, double b, const double* y, double* out, long N,
                         cudaStream_t st);
cudaError_t launch_mul(const double* x, const double* y, double* out, long N, cudaStream_t st);
cudaError_t launch_div(const double* x, const double* y, double* out, long N, cudaStream_t st);
// d = 1 + alpha * diag; dsq = sqrt(d); s = d ** -0.5; partial mins of d
cudaError_t launch_scaling(const double* diag, double alpha, double* d, double* dsq, double* s, long N,
                           double* partial_min, int nb, cudaStream_t st);
// scaled bands for the X_D projection (precond.py:501-513)
cudaError_t launch_scale_bands(const double* diag, const double* inner, const double* block,
                               const double* s, int n, double* diag_s, double* inner_s,
                               double* block_s, cudaStream_t st);
// inv = 1 / max(lam, floor); partial counts of lam < floor
cudaError_t launch_invert_eigs(const double* lam, double floor, double* inv, long N, double* partial,
                               int nb, cudaStream_t st);
cudaError_t launch_invert_eigs_dev(const double* lam, const double* max_lam, double* inv, long N,
                                   double* partial, cudaStream_t st);
cudaError_t launch_reduce_min(const double* partial_min, int nb, double* out, cudaStream_t st);
cudaError_t launch_reduce_minmax(const double* partial_mm, int nb, double* out_min, double* out_max,
                                 cudaStream_t st);
int vec_blocks();

}  // namespace tvd
