// Internal (non-ABI) declarations shared by the tvdeblur CUDA translation units.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "tvd_cg.h"
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

// ---- odd-symmetric prime-factor DST engine (tvd_pfa.cu)
// x / d == (x * m) >> 40 exactly for 0 <= x, d < 2^20.
struct FDiv {
  unsigned long long m;
  int d;
};
inline FDiv make_fdiv(int d) {
  FDiv f;
  f.d = d;
  f.m = ((1ULL << 40) + (unsigned long long)d - 1) / (unsigned long long)d;
  return f;
}

struct PfaStage {
  int q, H, st;        // DFT size along this dimension, (q-1)/2, layout stride
  int D1, D2, S1, S2;  // the other dimensions (sizes, strides); D1 = 1 when only one
  int Rcnt, h2, nch, kb;
  FDiv fRcnt, fD2, fnch, fH;
  const double2* M;    // [(r-1) * H + (k-1)] = (cos, sin)(2 pi r k / q), padded
  // tensor-core (DMMA) form: KP x RP row-major, KP = roundup(H+1, 8), RP = roundup(H, 4)
  int use_mma, KP, RP;
  const double* Cm;    // [k][r-1] = cos(2 pi r k / q), k = 0..H (row 0 all ones)
  const double* Sm;    // [k][r-1] = sin(2 pi r k / q)
  // the same tables in DMMA A-fragment order: [(kt * (RP / 4) + rs) * 32 + lane] =
  // Cm[(kt * 8 + (lane >> 2)) * RP + rs * 4 + (lane & 3)], so a warp's fragment load is one
  // contiguous 256-byte read (2 L1 wavefronts) instead of eight 32-byte row pieces
  const double* Cf;
  const double* Sf;
};

// Good-Thomas line layout (row-major over the factors).  Two-factor shapes pad the
// row pitch to pfa_row_pitch(q1) so the CRT gather and the DMMA fragment loads of a
// warp fall on distinct shared-memory banks; LP is the padded line size.
constexpr int pfa_row_pitch(int q1) { return q1 + ((2 - q1 % 4) + 4) % 4; }

struct PfaPlan {
  int L, d, LP;
  int q[3], stride[3], rinv[3];
  FDiv fq[3];
  FDiv fN;             // N = L - 1
  PfaStage st[3];
  // index tables for the compile-time specialised kernels (tvd_pfa_t.cuh)
  const unsigned* scat;     // t = 1..N: pos(c'_j of z_t) | pos(c'_{-j}) << 16
  const unsigned* gath;     // k = 1..N: pos(C'_k)
  const unsigned* reps[3];  // stage s, representative t: base | negated base << 16
  // Half-line layout of two-factor shapes (tvd_pfa_half.cuh): only b <= (q1 - 1) / 2 of the
  // q0 x q1 Good-Thomas grid is stored (row pitch P1h), the rest is -(value at (-a, -b)).
  int P1h, LPh;
  const unsigned* hscat;  // t: posA | negA << 15 | posB << 16 | hasB << 31 (B always negated)
  const unsigned* hgath;  // k: pos | neg << 15
  // general (not odd) complex DFT of length L on the same grid (the assembly's band
  // projections, k_band_pfa): every other-index tuple of a stage is its own line
  const unsigned* greps[3];  // stage s, tuple t: base | base << 16
  const unsigned* gscat;     // j = 0..L-1: pos(x_j) (Ruritanian input map)
};

// ---- Rader DST engine for prime odd cores (tvd_rader.cu / tvd_rader.h)
constexpr int kRaderMaxStages = 8;

// Plan of one prime length L: convolution length M = L - 1, Stockham stages of the
// length-M FFT (radix, product of the previous radices, register items per thread).
struct RaderPlan {
  int L, M, g;
  int nst;
  int radix[kRaderMaxStages], ns[kRaderMaxStages], slots[kRaderMaxStages];
  const unsigned* rin;   // t = 1..M: dlog_g(j(t)), the Rader position of c'_j (packing map)
  const unsigned* rout;  // k = 1..M: (M - dlog_g(k)) mod M, where C_k lands
  const double2* bh;     // FFT_M(b), b_q = exp(-2 pi i g^-q / L)
  const double2* tw;     // exp(-2 pi i e / M), e in [0, M)
  const unsigned* dlg;   // m = 1..M: dlog_g(m), the Rader position of input m (plain DFT)
  // negacyclic half-length form for the odd DST input (a_{n+H} = -a_n, H = M / 2):
  int H;
  const double2* psi;    // n < H: exp(i pi n / H)
  const double2* twh;    // e < H: exp(-2 pi i e / H)
  const double2* bhh;    // FFT_H of beta~, beta_n = b_n - b_{n+H}, beta~_n = beta_n psi^n
};

// Device-resident FFT plan plus the per-length twiddle tables of one family.
struct TrigPlan {
  int family;     // Family
  int n;          // line length
  int L;          // FFT length per line
  FftPlan fft;
  const double2* wfull;  // exp(-i pi k / L), k in [0, L)
  const double2* whalf;  // DCT only: exp(-i pi k / (2n)), k in [0, n)
  int max_items_line;    // largest per-line work-item count over the stages
  bool pfa_ok = false;   // DST family with an odd, <=3-factor coprime L
  PfaPlan pfa;
  bool rader_ok = false;  // DST family with a prime L (Rader engine)
  RaderPlan rader;
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
  PcgFin fin;  // finalizer over `partial` folded into the last CTA (pipeline pass; s == nullptr: off)
  // anti-reflective transform T = Shat (I + U) (transforms.py:96-140), pipeline passes only:
  // bit 0: T before the first transform (x_int += x_0 q_L + x_last q_R), bit 1: T^-1 after it
  // (y_int -= x_0 q_L + x_last q_R), bit 2: T before the sandwich's second transform
  int ar_mode;
  const double* ar_ql;
  const double* ar_qr;
  // segmented input rows (row-slab decomposition, pipeline and Rader passes): when in_seg > 0,
  // element e of line l is in[(e / in_seg) * in_seg_stride + l * in_seg + e % in_seg] -- the
  // layout an all-to-all of per-rank blocks leaves behind; 0 = row-major (l * len + e)
  int in_seg;
  long in_seg_stride;
  // generic engine (k_trig): element t of line l is written to out[t * nlines + l] (the pass
  // output transposed, so the next pass runs over contiguous rows); post / dot_with unused
  int out_trans;
  // pipeline passes: input in the pair-blocked layout of a pass launched with transposed = 2
  // (element e of line l at ((l >> 1) len + e) 2 + (l & 1)); row-major input otherwise
  int in_blocked;
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

// band projections (sine family) on the prime-factor engine: a general complex DFT of length
// L per line on the fp64 tensor cores (tvd_pfa.cu); -1 when the shape is not specialised
cudaError_t launch_band_pfa(const PfaPlan& P, const double2* wfull, int n, const BandLines& b,
                            int* nblocks_out, cudaStream_t st);
bool band_pfa_ok(const PfaPlan& P);
// shapes whose projections run on the column-owner kernel (one line per CTA): their level-2
// pass pays for transposed, contiguous lines
bool band_pfa_rowwise(const PfaPlan& P);

// ---- launchers (tvd_lines.cu)
cudaError_t launch_trig(const TrigPlan& P, const LineGeom& g, int analysis, const LineIO& io,
                        int* nblocks_out, cudaStream_t st);
cudaError_t launch_band_project(const TrigPlan& P, int axis, const BandLines& b,
                                int* nblocks_out, cudaStream_t st);
int trig_lines_per_cta(const TrigPlan& P, bool contiguous, int* nthreads, size_t* smem);
// AR (P family) projection: border eigenvalues of each projected line from its interior
// (weights c), optionally followed by the eigenvalue epilogue with per-CTA (min, max) pairs
cudaError_t launch_ar_corr_rows(double* x, int rows, int cols, double sign, const double* ql,
                                const double* qr, cudaStream_t st);
cudaError_t launch_ar_dots_rows(const double* src, int rows, int cols, const double* ql,
                                const double* qr, double* sums, cudaStream_t st);
cudaError_t launch_ar_border_add(double* x, int rows, int cols, double sign, const double* sums,
                                 cudaStream_t st);
cudaError_t launch_ar_corr(double* x, int n, int axis, double sign, const double* ql,
                           const double* qr, const int* skip, cudaStream_t st);
cudaError_t launch_ar_lines(double* proj, int nlines, int n, long ls, long es, const double* c,
                            int epi, const double* lamh, const double* lamd, double alpha,
                            double* partial_minmax, int* nblocks_out, cudaStream_t st);
int trig_blocks(const TrigPlan& P, const LineGeom& g);

// ---- odd-symmetric PFA DST-I pass (tvd_pfa.cu), family DST1 / SINE_HAT
cudaError_t launch_pfa(const PfaPlan& P, int family, int len, const LineGeom& g, const LineIO& io,
                       int* nblocks_out, cudaStream_t st);
int pfa_blocks(const PfaPlan& P, const LineGeom& g);
// persistent TMA-pipelined row pass over an nlines x len row-major array (even len, PFA
// specialised shapes); transposed != 0 writes the result transposed (len x nlines)
cudaError_t launch_pipe(const PfaPlan& P, int family, int len, int nlines, int transposed,
                        const LineIO& io, int* nblocks_out, cudaStream_t st);
int pipe_grid(const PfaPlan& P, int nlines);
// out = in^T for an n x n fp64 array (tvd_stencil.cu)
cudaError_t launch_transpose(const double* in, double* out, int n, cudaStream_t st);
// eig = epilogue(transpose(projT)) with per-CTA (min, max) pairs (tvd_stencil.cu k_transpose_eig)
cudaError_t launch_transpose_eig(const double* projT, int n, int epi, const double* lamh,
                                 const double* lamd, double alpha, double* eig,
                                 double* partial_minmax, int* nblocks_out, cudaStream_t st);
// out (cols x rows) = in^T for a rows x cols fp64 array
cudaError_t launch_transpose_rect(const double* in, double* out, int rows, int cols,
                                  const int* skip, cudaStream_t st);

}  // namespace tvd
