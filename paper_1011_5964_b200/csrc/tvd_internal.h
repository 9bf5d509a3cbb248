// Internal (non-ABI) declarations shared by the tvdeblur CUDA translation units.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "tvd_fft.cuh"

namespace tvd {

// transform families (match include/tvdeblur_b200.h TVD_TRANSFORM_*)
enum Family : int { kFamDst1 = 0, kFamSineHat = 1, kFamDct = 2 };

// Lines of a strided fp64 array: element t of line l sits at l * ls + t * es.
// Rows of an R x C row-major array: len = C, nlines = R, ls = C, es = 1.
// Columns: len = R, nlines = C, ls = 1, es = C.
struct LineGeom {
  int len;
  int nlines;
  long ls;
  long es;
};

// Device-resident FFT plan plus the per-length twiddle tables of one family.
struct TrigPlan {
  int family;     // Family
  int n;          // array side
  int L;          // FFT length per line
  FftPlan fft;
  const double2* wfull;  // exp(-i pi k / L), k in [0, L)
  const double2* whalf;  // DCT only: exp(-i pi k / (2n)), k in [0, n)
  int max_items_line;    // largest per-line work-item count over the stages
  std::vector<void*> owned;
};

// Elementwise pre/post hooks of a line pass.
struct LineIO {
  const double* in;
  double* out;
  const double* pre;       // x = in / pre (pre_mul: in * pre) (nullable)
  const double* mid_mul;   // sandwich: y = T2(mid_mul * T1(x)) (nullable = single pass)
  const double* post;      // out = y / post (post_mul: y * post) (nullable)
  const double* dot_with;  // partial += out * dot_with (nullable)
  double* partial;         // per-CTA partials (nullable)
  const int* skip;         // device flag: return immediately when *skip != 0 (nullable)
  int pre_mul;
  int post_mul;
};

// Band projection of one batch of lines (preconditioner assembly).
struct BandLines {
  const double* b0; long b0_ls, b0_es;  // d = 0 band, n entries per line
  const double* b1; long b1_ls, b1_es;  // |d| = 1 band, n-1 entries per line (nullable)
  double c1;                              // multiplicity of the |d| = 1 band (0, 1, 2)
  int nlines;
  double* out; long out_ls, out_es;
  // epilogue (final stage only): lam = lamh^2 [* lamd^2] + alpha * proj
  int epi;              // 0 = store proj, 1 = X / D_X, 2 = X_D
  const double* lamh;
  const double* lamd;
  double alpha;
  double* partial_minmax;  // per-CTA (min, max) pairs (epi != 0)
};

struct Status {
  int code = 0;
  std::string msg;
};

// ---- launchers (tvd_lines.cu)
cudaError_t launch_trig(const TrigPlan& P, const LineGeom& g, int analysis, const LineIO& io,
                        int* nblocks_out, cudaStream_t st);
cudaError_t launch_band_project(const TrigPlan& P, int axis, const BandLines& b,
                                int* nblocks_out, cudaStream_t st);
int trig_lines_per_cta(const TrigPlan& P, bool contiguous, int* nthreads, size_t* smem);
int trig_blocks(const TrigPlan& P, const LineGeom& g);

}  // namespace tvd
