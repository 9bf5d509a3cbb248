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
};

cudaError_t launch_sum_partials(const double* partial, int nb, double* out, cudaStream_t st);
cudaError_t launch_residual_init(const double* b, const double* q, double* r, long N, double* partial,
                                 int nb, cudaStream_t st);
cudaError_t launch_pcg_start(PcgState* s, const double* partial, int nb, cudaStream_t st);
cudaError_t launch_pcg_rz0(PcgState* s, const double* partial, int nb, cudaStream_t st);
cudaError_t launch_copy(const double* src, double* dst, long N, const int* skip, cudaStream_t st);
cudaError_t launch_pcg_gamma(PcgState* s, const double* partial, int nb, cudaStream_t st);
cudaError_t launch_pcg_update_xr(PcgState* s, double* x, double* r, const double* p, const double* q,
                                 long N, double* partial, int nb, cudaStream_t st);
cudaError_t launch_pcg_rel(PcgState* s, const double* partial, int nb, double tol, double* hist,
                           cudaStream_t st);
cudaError_t launch_pcg_beta(PcgState* s, const double* partial, int nb, int max_it, cudaStream_t st);
cudaError_t launch_pcg_update_p(PcgState* s, double* p, const double* z, long N, cudaStream_t st);
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
int vec_blocks();

}  // namespace tvd
