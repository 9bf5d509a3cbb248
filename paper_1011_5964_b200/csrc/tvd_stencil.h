// Declarations for the stencil / convolution kernels (tvd_stencil.cu).
#pragma once

#include "tvd_cg.h"
#include "tvd_common.cuh"

namespace tvd {

// One-dimensional banded operator B (n x n) of half-width w.  Rows in
// [B, n - B) are Toeplitz with the symmetric `taps`; the others read `table`.
struct BandOp {
  int n, w, B;
  const double* taps;       // 2w+1 (device)
  const double* table;      // n x (2w+1), table[i*(2w+1) + k + w] = B[i][i+k] (device)
  const double* taps_host;  // 2w+1 (host copy; becomes kernel-parameter constants)
  // Operator fragments of the border tiles for the tensor-core passes (tvd_band_mma.cu):
  // 8-output tile p < frag_l is block p, frag_r0 <= p < ceil(n/8) is block frag_l + p -
  // frag_r0, anything else the trailing zero block; block layout [S][32 lanes].
  const double* frag;
  int frag_l, frag_r0, frag_cnt;
};

// Epilogue of the normal-equation column pass:
//   q = [s *] (acc + alpha * L(lw)),  partial += dot_with . q
struct Epilogue {
  const double* a_h;
  const double* a_v;
  const double* lw;
  double alpha;
  double inv_h2;
  const double* s;
  const double* dot_with;
  double* partial;
  PcgFin fin;
  int bc_l;              // diffusion ghosts: 0 zero Neumann, 1 anti-reflective
  int prefetch;          // tensor-core column pass: L2 prefetch of the epilogue operands
  double* partial_self;  // optional per-CTA partials of q . q (BiCGstab t . t)  // gamma finalizer folded into the last CTA (tensor-core pass; s == nullptr: off)
};

// (L w)[i][j] of tv.py:96-108, reference op order.  Ghosts: bc 0 zero Neumann (w_{-1} =
// w_0), bc 1 anti-reflective (w_{-1} = 2 w_0 - w_1, one rounding as numpy's odd reflection).
__device__ __forceinline__ double ar_ghost(double w0, double w1) {
  return __dsub_rn(__dmul_rn(2.0, w0), w1);
}
__device__ __forceinline__ double diffusion_at(const double* __restrict__ a_h,
                                               const double* __restrict__ a_v,
                                               const double* __restrict__ w, int n, int i, int j,
                                               double inv_h2, int bc = 0) {
  const long g = (long)i * n + j;
  const double wc = w[g];
  const double wl = j > 0 ? w[g - 1] : (bc ? ar_ghost(wc, w[g + 1]) : wc);
  const double wr = j < n - 1 ? w[g + 1] : (bc ? ar_ghost(wc, w[g - 1]) : wc);
  const double wu = i > 0 ? w[g - n] : (bc ? ar_ghost(wc, w[g + n]) : wc);
  const double wd = i < n - 1 ? w[g + n] : (bc ? ar_ghost(wc, w[g - n]) : wc);
  const long h0 = (long)i * (n + 1) + j;
  const double fl = __dmul_rn(a_h[h0], __dsub_rn(wc, wl));
  const double fr = __dmul_rn(a_h[h0 + 1], __dsub_rn(wr, wc));
  const double fu = __dmul_rn(a_v[g], __dsub_rn(wc, wu));
  const double fd = __dmul_rn(a_v[g + n], __dsub_rn(wd, wc));
  return __dmul_rn(-inv_h2, __dadd_rn(__dsub_rn(fr, fl), __dsub_rn(fd, fu)));
}

// tensor-core (DMMA) band passes, tvd_band_mma.cu; used when band_mma_ok(op)
bool band_mma_ok(const BandOp& op);
int band_mma_koff(int w);  // k-offset of the tensor-core passes for half-width w (0: none)
int band_mma_cols_grid(int n, int rows = -1);
int band_mma_row_tile();  // output rows per column-pass CTA (row windows align to it)
// row_lo / row_hi: output rows [row_lo, row_hi) only (row-slab decomposition; -1 = all).
// Pointers index global rows (in + row * n); the column pass reads `in` rows
// [row_lo - KOFF, row_hi + KOFF) and the epilogue's lw rows row_lo - 1 .. row_hi (clipped to
// the image), a_v rows row_lo .. row_hi.
cudaError_t launch_band_mma_rows(const BandOp& op, const double* in, double* out, const int* skip,
                                 cudaStream_t st, int row_lo = 0, int row_hi = -1);
cudaError_t launch_band_mma_cols(const BandOp& op, const double* in, double* out,
                                 const Epilogue& ep, const int* skip, cudaStream_t st,
                                 int row_lo = 0, int row_hi = -1);
// row pass fused with the PCG direction update: p_new = z + beta p_old (in = p_old), out = p_new
// G^T; z == nullptr is the plain pass
cudaError_t launch_band_mma_rows_fused(const BandOp& op, const double* in, double* out,
                                       const int* skip, cudaStream_t st, const double* z,
                                       double* p_new, const PcgState* pst, int row_lo = 0,
                                       int row_hi = -1);

int band_rows_blocks(int n);
int band_cols_blocks(int n);          // upper bound over both column-pass variants
int band_cols_grid(const BandOp& op);  // exact grid of launch_band_cols for this operator
cudaError_t launch_band_rows(const BandOp& op, const double* in, double* out, const int* skip,
                             cudaStream_t st);
cudaError_t launch_band_cols(const BandOp& op, const double* in, double* out, const Epilogue& ep,
                             const int* skip, cudaStream_t st);
cudaError_t launch_diffusivity(const double* u, int n, double beta, double sp, double* a_h,
                               double* a_v, cudaStream_t st, int bc = 0);
cudaError_t launch_diffusion_apply(const double* a_h, const double* a_v, const double* w, int n,
                                   double inv_h2, double* out, cudaStream_t st, int bc = 0);
cudaError_t launch_diffusivity_rows(const double* u_win, int win_lo, int n, double beta, double sp,
                                    double* a_h, double* a_v, cudaStream_t st, int bc, int row_lo,
                                    int row_hi);
cudaError_t launch_diffusion_bands_rows(const double* a_h, const double* a_v, int n, double inv_h2,
                                        double* diag, double* inner, double* block, int row_lo,
                                        int row_hi, cudaStream_t st);
cudaError_t launch_diffusion_bands(const double* a_h, const double* a_v, int n, double inv_h2,
                                   double* diag, double* inner, double* block, cudaStream_t st,
                                   int bc = 0, double* inner_lo = nullptr,
                                   double* block_lo = nullptr);
cudaError_t launch_general_blur(const double* in, double* out, int n, int m, int bc,
                                const double* h, int transpose, double* scratch_a,
                                double* scratch_b, cudaStream_t st);
// valid convolution of an extended T x T array with a K x K PSF: separable (h == nullptr:
// factors g1 along axis 0, g2 along axis 1, scratch T x (T-K+1)) or direct 2D (h)
cudaError_t launch_valid_convolve(const double* ext, int T, int K, const double* g1,
                                  const double* g2, const double* h, double* scratch,
                                  double* out, cudaStream_t st);
cudaError_t launch_normal_epilogue(const double* base, const Epilogue& ep, int n, double* out,
                                   const int* skip, int nblocks, cudaStream_t st);
cudaError_t launch_eigenvalues(const double* cos_tab, const double* h, int n, int K, double* tmp,
                               double* lam, cudaStream_t st);

}  // namespace tvd
