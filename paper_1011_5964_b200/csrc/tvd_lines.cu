#include <cstdlib>
// Line passes of the trigonometric transforms (reference transforms.py:52-171,
// precond.py:82-199 / 369-395 / 456-477).
//
// A CTA owns `nl` lines of an n x n fp64 array (rows when axis == 1, columns
// when axis == 0).  Each pass:
//   global -> real staging (smem, optional elementwise pre-division)
//   -> pack into complex FFT lines -> fft_lines -> unpack to real staging
//   [-> multiply by an eigenvalue grid -> second transform]   (sandwich)
//   -> global (optional post-division, optional fused dot partial).
// DST-I (and the bordered Shat) use one length-(N+1) complex FFT per line:
//   c_j = z_{2j} + i z_{2((j+h) mod L)+1}  (L odd, h = (L-1)/2),
// where z is the odd extension of the line; then
//   y_k = -(Im C_k - (-1)^k Re C_k) / 2 * sqrt(2/L).
// For even L the standard even/odd real-FFT split is used.
// DCT-II / DCT-III use Makhoul's reordering with two real lines packed into
// one complex FFT of length n.
#include "tvd_internal.h"
#include "tvd_rader.h"

namespace tvd {

struct TrigK {
  FftPlan fft;
  const double2* wfull;
  const double2* whalf;
  int family, n, L, nl, analysis, nlines;  // n = line length
  long ls, es;
  int P;   // real staging pitch (doubles)
  int LP;  // complex line pitch
  int ncx; // complex lines per CTA
  double s0, s1, inv_s0, inv_s1, dst_scale;
  LineIO io;
};

// ------------------------------------------------------------------ DST
__device__ __forceinline__ void dst_lines(const TrigK& p, double* real, double2* cbuf) {
  const int tid = threadIdx.x, nth = blockDim.x;
  const int off = p.family == kFamSineHat ? 1 : 0;
  const int L = p.L, N = L - 1;
  const bool odd = (L & 1);
  const int h = (L - 1) / 2;
  for (int i = tid; i < p.nl * L; i += nth) {
    const int l = i / L, j = i - l * L;
    const double* x = real + l * p.P + off - 1;  // x[t], t = 1..N
    auto z = [&](int t) -> double {
      if (t == 0 || t == L) return 0.0;
      return t < L ? x[t] : -x[2 * L - t];
    };
    int jj = j;
    if (odd) {
      jj = j + h;
      if (jj >= L) jj -= L;
    }
    cbuf[l * p.LP + j] = make_double2(z(2 * j), z(2 * jj + 1));
  }
  __syncthreads();
  fft_lines(cbuf, p.LP, p.nl, p.fft);
  for (int i = tid; i < p.nl * N; i += nth) {
    const int l = i / N, k = 1 + i - l * N;
    const double2* c = cbuf + l * p.LP;
    double y;
    if (odd) {
      const double2 C = c[k];
      y = (k & 1) ? -(C.y + C.x) : -(C.y - C.x);
    } else {
      const double2 C = c[k], Cr = cconj(c[L - k]);
      const double2 E = cscale(cadd(C, Cr), 0.5);
      const double2 D = csub(C, Cr);
      const double2 O = make_double2(0.5 * D.y, -0.5 * D.x);
      const double2 w = p.wfull[k];
      y = -(E.y + (w.x * O.y + w.y * O.x));
    }
    real[l * p.P + off + k - 1] = y * p.dst_scale;
  }
  __syncthreads();
}

// ------------------------------------------------------------------ DCT
__device__ __forceinline__ int makhoul(int j, int n) {
  return j < (n + 1) / 2 ? 2 * j : 2 * (n - 1 - j) + 1;
}

// DCT-II (analysis, C^T v), two lines per complex FFT.
__device__ __forceinline__ void dct2_lines(const TrigK& p, double* real, double2* cbuf) {
  const int tid = threadIdx.x, nth = blockDim.x, n = p.n;
  for (int i = tid; i < p.ncx * n; i += nth) {
    const int q = i / n, j = i - q * n, src = makhoul(j, n);
    cbuf[q * p.LP + j] = make_double2(real[(2 * q) * p.P + src], real[(2 * q + 1) * p.P + src]);
  }
  __syncthreads();
  fft_lines(cbuf, p.LP, p.ncx, p.fft);
  for (int i = tid; i < p.ncx * n; i += nth) {
    const int q = i / n, k = i - q * n;
    const double2* c = cbuf + q * p.LP;
    const double2 C = c[k], Cr = cconj(c[k == 0 ? 0 : n - k]);
    const double2 Va = cscale(cadd(C, Cr), 0.5);
    const double2 D = csub(C, Cr);
    const double2 Vb = make_double2(0.5 * D.y, -0.5 * D.x);
    const double2 w = p.whalf[k];
    const double s = k == 0 ? p.s0 : p.s1;
    real[(2 * q) * p.P + k] = s * (w.x * Va.x - w.y * Va.y);
    real[(2 * q + 1) * p.P + k] = s * (w.x * Vb.x - w.y * Vb.y);
  }
  __syncthreads();
}

// DCT-III (synthesis, C v), two lines per complex FFT.
__device__ __forceinline__ void dct3_lines(const TrigK& p, double* real, double2* cbuf) {
  const int tid = threadIdx.x, nth = blockDim.x, n = p.n;
  for (int i = tid; i < p.ncx * n; i += nth) {
    const int q = i / n, k = i - q * n;
    const double* ra = real + (2 * q) * p.P;
    const double* rb = real + (2 * q + 1) * p.P;
    const double is = k == 0 ? p.inv_s0 : p.inv_s1;
    const double ya = ra[k] * is, yb = rb[k] * is;
    const double yar = k == 0 ? 0.0 : ra[n - k] * p.inv_s1;
    const double ybr = k == 0 ? 0.0 : rb[n - k] * p.inv_s1;
    const double2 w = cconj(p.whalf[k]);  // exp(+i pi k / 2n)
    const double2 Va = cmul(w, make_double2(ya, -yar));
    const double2 Vb = cmul(w, make_double2(yb, -ybr));
    // V = Va + i Vb ; store conj(V) so a forward FFT yields n * conj(ifft(V))
    cbuf[q * p.LP + k] = make_double2(Va.x - Vb.y, -(Va.y + Vb.x));
  }
  __syncthreads();
  fft_lines(cbuf, p.LP, p.ncx, p.fft);
  const double inv_n = 1.0 / n;
  for (int i = tid; i < p.ncx * n; i += nth) {
    const int q = i / n, j = i - q * n, dst = makhoul(j, n);
    const double2 C = cbuf[q * p.LP + j];
    real[(2 * q) * p.P + dst] = C.x * inv_n;
    real[(2 * q + 1) * p.P + dst] = -C.y * inv_n;
  }
  __syncthreads();
}

__device__ __forceinline__ void transform_lines(const TrigK& p, double* real, double2* cbuf,
                                                bool analysis) {
  if (p.family == kFamDct) {
    if (analysis) dct2_lines(p, real, cbuf);
    else dct3_lines(p, real, cbuf);
  } else {
    dst_lines(p, real, cbuf);
  }
}

template <int NTH, int MINB>
__global__ void __launch_bounds__(NTH, MINB) k_trig(const TrigK p) {
  pdl_enter();
  const LineIO& io = p.io;
  if (io.skip && *io.skip) return;
  extern __shared__ double2 smem2[];
  double2* cbuf = smem2;
  double* real = reinterpret_cast<double*>(smem2 + (size_t)p.ncx * p.LP);
  __shared__ double red[32];
  const int tid = threadIdx.x, nth = blockDim.x, n = p.n;
  const int line0 = blockIdx.x * p.nl;
  const int nlv = min(p.nl, p.nlines - line0);
  const bool contig = p.es == 1;
  // (l, t) of the i-th element in memory-friendly order
  auto lt = [&](int i, int& l, int& t) {
    if (contig) { l = i / n; t = i - l * n; }
    else { t = i / nlv; l = i - t * nlv; }
  };
  auto gidx = [&](int l, int t) { return (long)(line0 + l) * p.ls + (long)t * p.es; };

  for (int i = tid; i < nlv * n; i += nth) {
    int l, t;
    lt(i, l, t);
    const long g = gidx(l, t);
    double v = io.in[g];
    if (io.pre) v = io.pre_mul ? v * io.pre[g] : v / io.pre[g];
    real[l * p.P + t] = v;
  }
  for (int i = tid; i < (p.nl - nlv) * n; i += nth) {
    const int l = nlv + i / n, t = i % n;
    real[l * p.P + t] = 0.0;
  }
  __syncthreads();

  const bool sandwich = io.mid_mul != nullptr;
  transform_lines(p, real, cbuf, sandwich ? true : p.analysis != 0);
  if (sandwich) {
    for (int i = tid; i < nlv * n; i += nth) {
      int l, t;
      lt(i, l, t);
      real[l * p.P + t] *= io.mid_mul[gidx(l, t)];
    }
    __syncthreads();
    transform_lines(p, real, cbuf, false);
  }

  double acc = 0.0;
  if (io.out_trans) {  // t-major: consecutive threads write the nlv adjacent lines of one t
    for (int i = tid; i < nlv * n; i += nth) {
      const int t = i / nlv, l = i - t * nlv;
      io.out[(long)t * p.nlines + line0 + l] = real[l * p.P + t];
    }
  } else {
    for (int i = tid; i < nlv * n; i += nth) {
      int l, t;
      lt(i, l, t);
      const long g = gidx(l, t);
      double v = real[l * p.P + t];
      if (io.post) v = io.post_mul ? v * io.post[g] : v / io.post[g];
      io.out[g] = v;
      if (io.dot_with) acc += v * io.dot_with[g];
    }
  }
  if (io.partial) {
    const double s = block_sum(acc, red);
    if (tid == 0) io.partial[blockIdx.x] = s;
    if (io.fin.s) pcg_fin_tail(io.fin, io.partial, gridDim.x, red);
  }
}

// ------------------------------------------------------ band projections
struct BandK {
  FftPlan fft;
  const double2* wfull;
  int family, n, L, nl, LP;
  BandLines b;
};

__global__ void __launch_bounds__(512) k_band(const BandK p) {
  extern __shared__ double2 smem2[];
  double2* cbuf = smem2;
  double* tot = reinterpret_cast<double*>(smem2 + (size_t)p.nl * p.LP);  // 2 * nl
  __shared__ double red[32];
  const int tid = threadIdx.x, nth = blockDim.x, n = p.n, L = p.L;
  const BandLines& b = p.b;
  const int line0 = blockIdx.x * p.nl;
  const int nlv = min(p.nl, b.nlines - line0);
  const bool sine = p.family != kFamDct;
  auto B0 = [&](int l, int j) { return b.b0[(long)(line0 + l) * b.b0_ls + (long)j * b.b0_es]; };
  auto B1 = [&](int l, int j) { return b.b1[(long)(line0 + l) * b.b1_ls + (long)j * b.b1_es]; };

  for (int i = tid; i < p.nl * L; i += nth) {
    const int l = i / L, j = i - l * L;
    double e = 0.0, o = 0.0;
    if (l < nlv) {
      if (sine) {
        // even slots 2j <- b0[j] (j = 1..N), odd slots 2j+1 <- c1 b1[j] (j = 1..N-1)
        if (j >= 1 && j <= L - 1) e = B0(l, j);
        if (b.b1 && j >= 1 && j <= L - 2) o = b.c1 * B1(l, j);
      } else {
        // even slots 2j <- c1 b1[j-1] (j = 1..n-1), odd slots 2j+1 <- b0[j]
        if (b.b1 && j >= 1) e = b.c1 * B1(l, j - 1);
        o = B0(l, j);
      }
    }
    cbuf[l * p.LP + j] = make_double2(e, o);
  }
  // per-line band totals (one warp per line, fixed order)
  {
    const int lane = tid & 31, wid = tid >> 5, nw = nth >> 5;
    for (int l = wid; l < p.nl; l += nw) {
      double t0 = 0.0, t1 = 0.0;
      if (l < nlv) {
        const int lo = sine ? 1 : 0, hi0 = sine ? n - 1 : n, hi1 = sine ? n - 2 : n - 1;
        for (int j = lo + lane; j < hi0; j += 32) t0 += B0(l, j);
        if (b.b1)
          for (int j = lo + lane; j < hi1; j += 32) t1 += B1(l, j);
      }
      t0 = warp_sum(t0);
      t1 = warp_sum(t1);
      if (lane == 0) {
        tot[2 * l] = t0;
        tot[2 * l + 1] = t1;
      }
    }
  }
  __syncthreads();
  fft_lines(cbuf, p.LP, p.nl, p.fft);

  double vmin = 1.0 / 0.0, vmax = -1.0 / 0.0;
  for (int i = tid; i < nlv * n; i += nth) {
    const int l = i / n, t = i - l * n;
    double v;
    if (sine && (t == 0 || t == n - 1)) {
      v = B0(l, t);
    } else {
      const double2* c = cbuf + l * p.LP;
      const int tr = t == 0 ? 0 : L - t;
      const double2 C = c[t], Cr = cconj(c[tr]);
      const double2 E = cscale(cadd(C, Cr), 0.5);
      const double2 D = csub(C, Cr);
      const double2 O = make_double2(0.5 * D.y, -0.5 * D.x);
      const double2 w = p.wfull[t];
      const double re_s = E.x + (w.x * O.x - w.y * O.y);
      const double t0 = tot[2 * l], t1 = tot[2 * l + 1];
      if (sine) {
        v = (t0 + b.c1 * t1 * w.x - re_s) / L;
      } else {
        const double rho2 = (t == 0 ? 1.0 : 2.0) / n;
        v = 0.5 * rho2 * (t0 + b.c1 * t1 * w.x + re_s);
      }
    }
    const long g = (long)(line0 + l) * b.out_ls + (long)t * b.out_es;
    if (b.epi == 1) {
      const double lh = b.lamh[g];
      v = lh * lh + b.alpha * v;
    } else if (b.epi == 2) {
      const double lh = b.lamh[g], ld = b.lamd[g];
      v = lh * lh * ld * ld + b.alpha * v;
    }
    b.out[g] = v;
    vmin = fmin(vmin, v);
    vmax = fmax(vmax, v);
  }
  if (b.epi != 0) {
    // deterministic block min / max
    for (int o = 16; o > 0; o >>= 1) {
      vmin = fmin(vmin, __shfl_xor_sync(0xffffffffu, vmin, o));
      vmax = fmax(vmax, __shfl_xor_sync(0xffffffffu, vmax, o));
    }
    __syncthreads();
    const int lane = tid & 31, wid = tid >> 5, nw = nth >> 5;
    if (lane == 0) {
      red[wid] = vmin;
      red[16 + wid] = vmax;
    }
    __syncthreads();
    if (tid == 0) {
      double a = red[0], z = red[16];
      for (int w = 1; w < nw; ++w) {
        a = fmin(a, red[w]);
        z = fmax(z, red[16 + w]);
      }
      b.partial_minmax[2 * blockIdx.x] = a;
      b.partial_minmax[2 * blockIdx.x + 1] = z;
    }
  }
}

// ------------------------------------------------------------- launchers
static int round_up(int x, int m) { return (x + m - 1) / m * m; }

// Lines per CTA / threads / smem for a trig pass.
int trig_lines_per_cta(const TrigPlan& P, bool contiguous, int* nthreads, size_t* smem) {
  const int n = P.n;
  const bool dct = P.family == kFamDct;
  const int pitch = n | 1;
  const size_t cbytes = (size_t)P.L * 16;
  const size_t rbytes = (size_t)pitch * 8;
  const size_t budget = 100 * 1024;
  int nl = contiguous ? 4 : 8;
  auto bytes = [&](int k) { return (dct ? (size_t)(k / 2) : (size_t)k) * cbytes + k * rbytes; };
  const int step = dct ? 2 : 1;
  while (nl > step && bytes(nl) > budget) nl -= step;
  if (bytes(nl) > 200 * 1024) return -1;
  int nth = round_up((P.max_items_line + kFftSlots - 1) / kFftSlots, 32);
  if (nth < 256) nth = 256;
  if (nth > 512) return -1;
  *nthreads = nth;
  *smem = bytes(nl);
  return nl;
}

int trig_blocks(const TrigPlan& P, const LineGeom& g) {
  int nth;
  size_t smem;
  const int nl = trig_lines_per_cta(P, g.es == 1, &nth, &smem);
  return nl <= 0 ? -1 : (g.nlines + nl - 1) / nl;
}

cudaError_t launch_trig(const TrigPlan& P, const LineGeom& g, int analysis, const LineIO& io,
                        int* nblocks_out, cudaStream_t st) {
  int nth;
  size_t smem;
  if (g.len != P.n) return cudaErrorInvalidValue;
  const int nl = trig_lines_per_cta(P, g.es == 1, &nth, &smem);
  if (nl <= 0) return cudaErrorInvalidConfiguration;
  TrigK k{};
  k.fft = P.fft;
  k.wfull = P.wfull;
  k.whalf = P.whalf;
  k.family = P.family;
  k.n = P.n;
  k.L = P.L;
  k.nl = nl;
  k.analysis = analysis;
  k.nlines = g.nlines;
  k.ls = g.ls;
  k.es = g.es;
  k.P = P.n | 1;
  k.LP = P.L;
  k.ncx = P.family == kFamDct ? nl / 2 : nl;
  k.s0 = sqrt(1.0 / P.n);
  k.s1 = sqrt(2.0 / P.n);
  k.inv_s0 = 1.0 / k.s0;
  k.inv_s1 = 1.0 / k.s1;
  k.dst_scale = 0.5 * sqrt(2.0 / P.L);
  k.io = io;
  const int nb = (g.nlines + nl - 1) / nl;
  if (nblocks_out) *nblocks_out = nb;
  if (nb == 0) return cudaSuccess;
  static bool attr_done = false;
  if (!attr_done) {
    cudaFuncSetAttribute(k_trig<512, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(k_trig<256, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr_done = true;
  }
  // 256-thread CTAs take the 255-register instance (the 512-thread bound caps the engine at
  // 128 registers and spills; c2b 10831 -> 10980 it/s)
  if (nth <= 256) return launch_pdl(k_trig<256, 1>, nb, nth, smem, st, k);
  return launch_pdl(k_trig<512, 1>, nb, nth, smem, st, k);
}

cudaError_t launch_band_project(const TrigPlan& P, int axis, const BandLines& b,
                                int* nblocks_out, cudaStream_t st) {
  (void)axis;
  // prime odd core (config 5, L = 8191): the length-L DFTs run on the Rader engine instead of
  // the generic engine's O(L) per point odd-radix stage (808 ms -> a few ms per assembly)
  if (P.family != kFamDct && P.rader_ok && P.rader.L == P.L && !option(kOptBandGeneric))
    return launch_band_rader(P.rader, P.n, P.wfull, b, nblocks_out, st);
  // the configs' composite odd cores (127, 511, 1023, 2047): a general DFT on the
  // prime-factor engine's fp64 tensor-core stages (tvd_pfa.cu k_band_pfa)
  if (P.family != kFamDct && P.pfa_ok && P.pfa.L == P.L && band_pfa_ok(P.pfa) &&
      !option(kOptBandGeneric))
    return launch_band_pfa(P.pfa, P.wfull, P.n, b, nblocks_out, st);
  BandK k{};
  k.fft = P.fft;
  k.wfull = P.wfull;
  k.family = P.family;
  k.n = P.n;
  k.L = P.L;
  k.LP = P.L;
  k.b = b;
  constexpr int nth_min = 256;  // minimum threads per CTA
  int nl = 2;                   // 2 lines: 792 vs 866 us per 2048^2 assembly for 4
  const size_t cbytes = (size_t)P.L * 16;
  while (nl > 1 && nl * cbytes > 100 * 1024) --nl;
  k.nl = nl;
  int nth = round_up((P.max_items_line + kFftSlots - 1) / kFftSlots, 32);
  if (nth < nth_min) nth = nth_min;
  if (nth > 512) return cudaErrorInvalidConfiguration;
  const size_t smem = nl * cbytes + 2 * nl * sizeof(double);
  const int nb = (b.nlines + nl - 1) / nl;
  if (nblocks_out) *nblocks_out = nb;
  static bool attr_done = false;
  if (!attr_done) {
    cudaFuncSetAttribute(k_band, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr_done = true;
  }
  // (a 255-register instance for 256-thread CTAs measured slower here: 1164 vs 805 us per
  // 2048^2 assembly -- occupancy, not the rarely executed spills, bounds this kernel)
  k_band<<<nb, nth, smem, st>>>(k);
  return cudaGetLastError();
}

// ------------------------------------------------ anti-reflective (P family) projection
// The AR algebra's interior eigenvalues are the sine projection's; its border eigenvalue
// 2 sum(z) - z_0 (precond.py:156-165, z the first-column representer of S diag(lam) S,
// precond.py:134-153) is the fixed linear functional sum_t c_t lam_t, c = s_1 .* S w,
// w_j = 2 (floor(j/2) + 1) - [j even] (host-built weights).  One thread per line (lanes
// = consecutive lines), deterministic sequential sums; epi as k_band's epilogue.
__global__ void k_ar_lines(double* __restrict__ proj, int nlines, int n, long ls, long es,
                           const double* __restrict__ c, int epi, const double* __restrict__ lamh,
                           const double* __restrict__ lamd, double alpha,
                           double* __restrict__ partial_minmax) {
  __shared__ double red[64];
  const int l = blockIdx.x * blockDim.x + threadIdx.x;
  double vmin = INFINITY, vmax = -INFINITY;
  if (l < nlines) {
    double* line = proj + (long)l * ls;
    double bsum = 0.0;
    for (int t = 1; t <= n - 2; ++t) bsum += c[t - 1] * line[(long)t * es];
    line[0] = bsum;
    line[(long)(n - 1) * es] = bsum;
    if (epi != 0) {
      for (int t = 0; t < n; ++t) {
        const long g = (long)l * ls + (long)t * es;
        double v = proj[g];
        if (epi == 1) {
          const double lh = lamh[g];
          v = lh * lh + alpha * v;
        } else {
          const double lh = lamh[g], ld = lamd[g];
          v = lh * lh * ld * ld + alpha * v;
        }
        proj[g] = v;
        vmin = fmin(vmin, v);
        vmax = fmax(vmax, v);
      }
    }
  }
  if (epi != 0) {
    for (int o = 16; o > 0; o >>= 1) {
      vmin = fmin(vmin, __shfl_xor_sync(0xffffffffu, vmin, o));
      vmax = fmax(vmax, __shfl_xor_sync(0xffffffffu, vmax, o));
    }
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    if (lane == 0) {
      red[wid] = vmin;
      red[32 + wid] = vmax;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double a = INFINITY, b = -INFINITY;
      for (int w = 0; w < nw; ++w) {
        a = fmin(a, red[w]);
        b = fmax(b, red[32 + w]);
      }
      partial_minmax[2 * blockIdx.x] = a;
      partial_minmax[2 * blockIdx.x + 1] = b;
    }
  }
}

cudaError_t launch_ar_lines(double* proj, int nlines, int n, long ls, long es, const double* c,
                            int epi, const double* lamh, const double* lamd, double alpha,
                            double* partial_minmax, int* nblocks_out, cudaStream_t st) {
  const int threads = 128, nb = (nlines + threads - 1) / threads;
  if (nblocks_out) *nblocks_out = nb;
  if (nlines <= 0) return cudaSuccess;
  k_ar_lines<<<nb, threads, 0, st>>>(proj, nlines, n, ls, es, c, epi, lamh, lamd, alpha,
                                     partial_minmax);
  return cudaGetLastError();
}

// x_int += sign (x_0 q_L + x_last q_R) along `axis` (1: rows, 0: columns) -- the rank-2 factor
// of T = Shat (I + U) (transforms.py:96-140); the borders are read from x itself (Shat leaves
// them unchanged, so before and after a transform they are the same).
__global__ void k_ar_corr(double* __restrict__ x, int n, int axis, double sign,
                          const double* __restrict__ ql, const double* __restrict__ qr,
                          const int* skip) {
  if (skip && *skip) return;
  const long N = (long)n * n;
  for (long g = blockIdx.x * (long)blockDim.x + threadIdx.x; g < N;
       g += (long)gridDim.x * blockDim.x) {
    const int i = (int)(g / n), j = (int)(g % n);
    const int t = axis == 1 ? j : i;  // position along the line
    if (t == 0 || t == n - 1) continue;
    const double b0 = axis == 1 ? x[(long)i * n] : x[j];
    const double b1 = axis == 1 ? x[(long)i * n + n - 1] : x[(long)(n - 1) * n + j];
    const double corr = __dadd_rn(__dmul_rn(b0, ql[t - 1]), __dmul_rn(b1, qr[t - 1]));
    x[g] = sign > 0 ? __dadd_rn(x[g], corr) : __dsub_rn(x[g], corr);
  }
}

cudaError_t launch_ar_corr(double* x, int n, int axis, double sign, const double* ql,
                           const double* qr, const int* skip, cudaStream_t st) {
  long nb = ((long)n * n + 255) / 256;
  if (nb > 16L * kSMs) nb = 16L * kSMs;
  k_ar_corr<<<(int)(nb < 1 ? 1 : nb), 256, 0, st>>>(x, n, axis, sign, ql, qr, skip);
  return cudaGetLastError();
}

// ---- 1D anti-reflective transform over contiguous lines (rows x cols, lines = rows)
// T = Shat (I + U), transforms.py:96-140.  The plain forms add / subtract the rank-2 border
// correction x_0 q_L + x_last q_R on the interior (k_ar_corr_rows); the transposed forms
// T^T = (I + U^T) Shat and T^-T = Shat (I - U^T) add / subtract the projections
// sum_t x_t q_L[t], sum_t x_t q_R[t] of the interior on the two border entries
// (k_ar_dots_rows: one warp per line, fixed lane-strided order + shuffle tree, then
// k_ar_border_add).
__global__ void k_ar_corr_rows(double* __restrict__ x, int rows, int cols, double sign,
                               const double* __restrict__ ql, const double* __restrict__ qr) {
  const long N = (long)rows * cols;
  for (long g = blockIdx.x * (long)blockDim.x + threadIdx.x; g < N;
       g += (long)gridDim.x * blockDim.x) {
    const long i = g / cols;
    const int t = (int)(g - i * cols);
    if (t == 0 || t == cols - 1) continue;
    const double b0 = x[i * cols], b1 = x[i * cols + cols - 1];
    const double corr = __dadd_rn(__dmul_rn(b0, ql[t - 1]), __dmul_rn(b1, qr[t - 1]));
    x[g] = sign > 0 ? __dadd_rn(x[g], corr) : __dsub_rn(x[g], corr);
  }
}

__global__ void k_ar_dots_rows(const double* __restrict__ src, int rows, int cols,
                               const double* __restrict__ ql, const double* __restrict__ qr,
                               double* __restrict__ sums) {
  const int lane = threadIdx.x & 31;
  const long wpb = blockDim.x >> 5;
  for (long line = blockIdx.x * wpb + (threadIdx.x >> 5); line < rows; line += (long)gridDim.x * wpb) {
    const double* x = src + line * cols;
    double sl = 0.0, sr = 0.0;
    for (int t = 1 + lane; t < cols - 1; t += 32) {
      sl += x[t] * ql[t - 1];
      sr += x[t] * qr[t - 1];
    }
    for (int o = 16; o > 0; o >>= 1) {
      sl += __shfl_down_sync(0xffffffffu, sl, o);
      sr += __shfl_down_sync(0xffffffffu, sr, o);
    }
    if (lane == 0) {
      sums[2 * line] = sl;
      sums[2 * line + 1] = sr;
    }
  }
}

__global__ void k_ar_border_add(double* __restrict__ x, int rows, int cols, double sign,
                                const double* __restrict__ sums) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < 2L * rows;
       i += (long)gridDim.x * blockDim.x) {
    const long line = i >> 1;
    double* p = x + line * cols + ((i & 1) ? cols - 1 : 0);
    *p = sign > 0 ? __dadd_rn(*p, sums[i]) : __dsub_rn(*p, sums[i]);
  }
}

static int ar_grid(long work, int per_block) {
  long nb = (work + per_block - 1) / per_block;
  if (nb > 16L * kSMs) nb = 16L * kSMs;
  return (int)(nb < 1 ? 1 : nb);
}

cudaError_t launch_ar_corr_rows(double* x, int rows, int cols, double sign, const double* ql,
                                const double* qr, cudaStream_t st) {
  k_ar_corr_rows<<<ar_grid((long)rows * cols, 256), 256, 0, st>>>(x, rows, cols, sign, ql, qr);
  return cudaGetLastError();
}

cudaError_t launch_ar_dots_rows(const double* src, int rows, int cols, const double* ql,
                                const double* qr, double* sums, cudaStream_t st) {
  k_ar_dots_rows<<<ar_grid(rows, 8), 256, 0, st>>>(src, rows, cols, ql, qr, sums);
  return cudaGetLastError();
}

cudaError_t launch_ar_border_add(double* x, int rows, int cols, double sign, const double* sums,
                                 cudaStream_t st) {
  k_ar_border_add<<<ar_grid(2L * rows, 256), 256, 0, st>>>(x, rows, cols, sign, sums);
  return cudaGetLastError();
}

}  // namespace tvd
