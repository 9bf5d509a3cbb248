// Rader DST-I engine for prime odd-core lengths (config 5: L = n - 1 = 8191).
//
// The DST-I of a line is the complex DFT of length L of the packed odd sequence c'
// (tvd_pfa.cu header).  For prime L, Rader's algorithm turns the DFT into a cyclic
// convolution of length M = L - 1 (g a generator of Z_L^*):
//   C_{g^-m} = c'_0 + sum_n c'_{g^n} w^{g^(n - m)},   w = exp(-2 pi i / L),
// i.e. a = (c'_{g^n})_n convolved with b = (w^{g^-q})_q.  c'_0 = 0 here (z_0 = z_L = 0).
// One line per CTA: the pack writes c'_j straight into Rader order (discrete-log table;
// the odd partner -j sits M/2 further), a forward Stockham FFT of length M runs in shared
// memory, the product with B = FFT_M(b) (host-built) is conjugated so a second forward FFT
// gives the inverse, and the unpack gathers C_k through the inverse-log table.
// M = 8190 = 2 3 3 5 7 13 keeps every stage's items in registers (compile-time slots).
// Reference semantics: transforms.py:52-81 (dst1_apply / sinehat_apply).
#include <cstdlib>

#include "tvd_internal.h"
#include "tvd_rader.h"

namespace tvd {
namespace {

// 512 threads (16 warps; 384 / 256 threads measured 12.8 / 15.5 ms per 8192^2 M^-1 against
// 11.5 ms here)
constexpr int kRaderThreads = 512;

// (cos, sin)(2 pi t / R) for t in [0, R), computed once per stage
template <int R>
__device__ __forceinline__ void odd_table(double2 (&cs)[R]) {
#pragma unroll
  for (int t = 0; t < R; ++t) {
    double s, c;
    sincospi(2.0 * t / R, &s, &c);
    cs[t] = make_double2(c, s);
  }
}

// forward DFT of an odd-length register vector with a precomputed table (see dft_odd_reg)
template <int R>
__device__ __forceinline__ void dft_odd_cs(double2 (&v)[R], const double2 (&cs)[R]) {
  constexpr int H = (R - 1) / 2;
  double2 a[H + 1], b[H + 1];
  const double2 x0 = v[0];
  double2 s0 = x0;
#pragma unroll
  for (int r = 1; r <= H; ++r) {
    a[r] = cadd(v[r], v[R - r]);
    b[r] = csub(v[r], v[R - r]);
    s0 = cadd(s0, a[r]);
  }
#pragma unroll
  for (int k = 1; k <= H; ++k) {
    double2 A = make_double2(0.0, 0.0), B = make_double2(0.0, 0.0);
#pragma unroll
    for (int r = 1; r <= H; ++r) {
      const double2 w = cs[(r * k) % R];
      A.x += a[r].x * w.x; A.y += a[r].y * w.x;
      B.x += b[r].x * w.y; B.y += b[r].y * w.y;
    }
    v[k] = make_double2(x0.x + A.x + B.y, x0.y + A.y - B.x);
    v[R - k] = make_double2(x0.x + A.x - B.y, x0.y + A.y + B.x);
  }
  v[0] = s0;
}

template <int R>
__device__ __forceinline__ void dft_any(double2 (&v)[R], const double2 (&cs)[R]) {
  if constexpr (R == 2 || R == 4 || R == 8 || R == 3 || R == 5 || R == 7 || R == 13) {
    dft_reg<R>(v);
  } else {
    dft_odd_cs<R>(v, cs);
  }
}

// One in-place Stockham stage of a single line of length M (see tvd_fft.cuh stage_reg):
// every item of the line sits in registers across the barrier (SLOTS items per thread).
// STASH: the butterflies beyond SLOTS * blockDim hold no registers across the barrier --
// their inputs are copied to `scratch` first and they run after it (the radix-13 / radix-7
// stages: two or three register slots of R complex values would exceed the 128-register
// budget of a 512-thread CTA and spill to local memory).
template <int R, int SLOTS, bool STASH = false>
__device__ __forceinline__ void rader_stage(double2* buf, int M, int ns,
                                            const double2* __restrict__ tw,
                                            double2* scratch = nullptr) {
  const int tid = threadIdx.x, nth = blockDim.x;
  const int nb = M / R, tstride = M / (ns * R);
  double2 cs[R];
  if constexpr (!(R == 2 || R == 4 || R == 8 || R == 3 || R == 5 || R == 7 || R == 13)) odd_table<R>(cs);
  const int jr = SLOTS * nth;  // first stashed butterfly
  if constexpr (STASH) {
    for (int i = tid; i < (nb - jr) * R; i += nth) {
      const int r = i / (nb - jr), j = jr + i - r * (nb - jr);
      scratch[i] = buf[j + r * nb];  // [r][j - jr]
    }
  }
  double2 v[SLOTS][R];
#pragma unroll
  for (int s = 0; s < SLOTS; ++s) {
    const int j = tid + s * nth;
    if (j < nb) {
      const int jm = j % ns;
      // twiddles w^(r e0), e0 = jm tstride: one table load per butterfly, the powers by
      // recurrence (R - 2 complex products; ~R ulp, far inside the 1e-12 parity bound) --
      // the per-element twiddle loads were the kernel's dominant long-scoreboard stall
      const double2 w1 = ns > 1 ? __ldg(&tw[jm * tstride]) : make_double2(1.0, 0.0);
      double2 wr = w1;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        double2 x = buf[j + r * nb];
        if (r > 0 && ns > 1) {
          x = cmul(x, wr);
          if (r + 1 < R) wr = cmul(wr, w1);
        }
        v[s][r] = x;
      }
      dft_any<R>(v[s], cs);
    }
  }
  __syncthreads();
#pragma unroll
  for (int s = 0; s < SLOTS; ++s) {
    const int j = tid + s * nth;
    if (j < nb) {
      const int jm = j % ns;
      const int d = (j / ns) * ns * R + jm;
#pragma unroll
      for (int r = 0; r < R; ++r) buf[d + r * ns] = v[s][r];
    }
  }
  if constexpr (STASH) {
    for (int j = jr + tid; j < nb; j += nth) {
      const int jm = j % ns;
      double2 w[R];
      const double2 w1 = ns > 1 ? __ldg(&tw[jm * tstride]) : make_double2(1.0, 0.0);
      double2 wr = w1;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        double2 x = scratch[r * (nb - jr) + j - jr];
        if (r > 0 && ns > 1) {
          x = cmul(x, wr);
          if (r + 1 < R) wr = cmul(wr, w1);
        }
        w[r] = x;
      }
      dft_any<R>(w, cs);
      const int d = (j / ns) * ns * R + jm;
#pragma unroll
      for (int r = 0; r < R; ++r) buf[d + r * ns] = w[r];
    }
  }
  __syncthreads();
}

// Compile-time stage lists (radix, register items per thread at kRaderThreads) of the
// supported convolution lengths; must match build_rader_plan's factorisation.
template <int M>
struct RaderStages;
template <>
struct RaderStages<8190> {  // 8190 = 2 3 3 5 7 13
  __device__ static void fft(double2* buf, const double2* tw, double2* scratch) {
    // butterflies 4095 / 2730 / 1638 / 1170 / 630 over 512 threads: register slots 8 / 6 /
    // 4, then 2 + 146 stashed (radix 7) and 1 + 118 stashed (radix 13)
    rader_stage<2, 8>(buf, 8190, 1, tw);
    rader_stage<3, 6>(buf, 8190, 2, tw);
    rader_stage<3, 6>(buf, 8190, 6, tw);
    rader_stage<5, 4>(buf, 8190, 18, tw);
    rader_stage<7, 2, true>(buf, 8190, 90, tw, scratch);
    rader_stage<13, 1, true>(buf, 8190, 630, tw, scratch);
  }
  static constexpr int kScratch = 118 * 13;  // double2 entries of the largest stash
};

// a <- conj(FFT(a) * Bh) in place, then FFT again: a_m = M conj(conv_m)
template <int M>
__device__ __forceinline__ void rader_convolve(double2* buf, const RaderPlan& P) {
  double2* scratch = buf + M;
  RaderStages<M>::fft(buf, P.tw, scratch);
  for (int m = threadIdx.x; m < M; m += blockDim.x) {
    const double2 x = cmul(buf[m], __ldg(&P.bh[m]));
    buf[m] = make_double2(x.x, -x.y);
  }
  __syncthreads();
  RaderStages<M>::fft(buf, P.tw, scratch);
}

// Half-length stage list: 4095 = 3 3 5 7 13 at kRaderNegThreads = 256 threads; butterflies
// 1365 / 1365 / 819 / 585 / 315 -> register slots 6 / 6 / 4 / 2 (+ 73 stashed) / 1 (+ 59)
constexpr int kRaderNegThreads = 256;
template <>
struct RaderStages<4095> {
  __device__ static void fft(double2* buf, const double2* tw, double2* scratch) {
    rader_stage<3, 6>(buf, 4095, 1, tw);
    rader_stage<3, 6>(buf, 4095, 3, tw);
    rader_stage<5, 4>(buf, 4095, 9, tw);
    rader_stage<7, 2, true>(buf, 4095, 45, tw, scratch);
    rader_stage<13, 1, true>(buf, 4095, 315, tw, scratch);
  }
  static constexpr int kScratch = 59 * 13;  // max(73 * 7, 59 * 13)
};

// DST input is odd (c'_{L-j} = -c'_j), so in Rader order a_{n+H} = -a_n (H = M / 2) and the
// length-M cyclic convolution folds into a length-H negacyclic one: with psi = exp(i pi / H),
// y_m = psi^-m (a psi^n (*) beta psi^n)_m for m < H and y_{m+H} = -y_m.  Half the FFT length,
// half the shared memory (two CTAs per SM).
template <int H>
__device__ __forceinline__ void rader_convolve_neg(double2* buf, const RaderPlan& P) {
  double2* scratch = buf + H;
  for (int m = threadIdx.x; m < H; m += blockDim.x) buf[m] = cmul(buf[m], __ldg(&P.psi[m]));
  __syncthreads();
  RaderStages<H>::fft(buf, P.twh, scratch);
  for (int m = threadIdx.x; m < H; m += blockDim.x) {
    const double2 x = cmul(buf[m], __ldg(&P.bhh[m]));
    buf[m] = make_double2(x.x, -x.y);
  }
  __syncthreads();
  RaderStages<H>::fft(buf, P.twh, scratch);
}

struct RaderK {
  RaderPlan pl;
  int n, off, nlines;
  double scale;  // 0.5 sqrt(2 / L) / M  (the 1/M of the inverse FFT folded in)
  LineIO io;
};

// One line (row) per CTA: row-major in, row-major out.
template <int MC>
__global__ void __launch_bounds__(kRaderThreads, 1) k_rader_rows(const RaderK p) {
  pdl_enter();
  const LineIO& io = p.io;
  if (io.skip && *io.skip) return;
  extern __shared__ __align__(16) double2 rbuf[];
  __shared__ double red[32];
  const int tid = threadIdx.x, nth = blockDim.x, n = p.n, line = blockIdx.x;
  constexpr int M = MC;
  const long rb = (long)line * n + p.off - 1;  // rb + t = element t (1..M) of the row
  const int half = M / 2;
  auto pack = [&](int t, double x) {
    const int q = (int)__ldg(&p.pl.rin[t - 1]);
    double* b = reinterpret_cast<double*>(rbuf) + (t & 1);
    b[2 * q] = x;
    int q2 = q + half;
    if (q2 >= M) q2 -= M;
    b[2 * q2] = -x;
  };
  auto unpack = [&](int k) {
    const double2 R = rbuf[__ldg(&p.pl.rout[k - 1])];  // C = conj(R) / M, 1/M in scale
    return ((k & 1) ? -(R.x - R.y) : -(-R.y - R.x)) * p.scale;
  };
  // element e of this line in the input (row-major or all-to-all segmented, LineIO::in_seg)
  auto in_at = [&](int e) {
    if (!io.in_seg) return io.in[(long)line * n + e];
    return io.in[(long)(e / io.in_seg) * io.in_seg_stride + (long)line * io.in_seg + e % io.in_seg];
  };
  for (int t = 1 + tid; t <= M; t += nth) {
    double x = in_at(p.off - 1 + t);
    if (io.pre) x = io.pre_mul ? x * io.pre[rb + t] : x / io.pre[rb + t];
    pack(t, x);
  }
  __syncthreads();
  rader_convolve<MC>(rbuf, p.pl);
  if (io.mid_mul) {
    constexpr int kV = (MC + kRaderThreads - 1) / kRaderThreads;
    double v[kV];
#pragma unroll
    for (int s = 0; s < kV; ++s) {
      const int t = 1 + tid + s * nth;
      v[s] = t <= M ? unpack(t) * io.mid_mul[rb + t] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int s = 0; s < kV; ++s) {
      const int t = 1 + tid + s * nth;
      if (t <= M) pack(t, v[s]);
    }
    __syncthreads();
    rader_convolve<MC>(rbuf, p.pl);
  }
  double acc = 0.0;
  for (int t = 1 + tid; t <= M; t += nth) {
    double y = unpack(t);
    if (io.post) y = io.post_mul ? y * io.post[rb + t] : y / io.post[rb + t];
    io.out[rb + t] = y;
    if (io.dot_with) acc += y * io.dot_with[rb + t];
  }
  if (p.off && tid < 2) {  // Shat borders pass through every transform
    const long g = (long)line * n + (tid ? n - 1 : 0);
    double v = in_at(tid ? n - 1 : 0);
    if (io.pre) v = io.pre_mul ? v * io.pre[g] : v / io.pre[g];
    if (io.mid_mul) v *= io.mid_mul[g];
    if (io.post) v = io.post_mul ? v * io.post[g] : v / io.post[g];
    io.out[g] = v;
    if (io.dot_with) acc += v * io.dot_with[g];
  }
  if (io.partial) {
    const double s = block_sum(acc, red);
    if (tid == 0) io.partial[blockIdx.x] = s;
    if (io.fin.s) pcg_fin_tail(io.fin, io.partial, gridDim.x, red);
  }
}

// The row pass on the negacyclic half-length convolution (HC = H); same I/O as k_rader_rows.
template <int HC>
__global__ void __launch_bounds__(kRaderNegThreads, 2) k_rader_rows_neg(const RaderK p) {
  pdl_enter();
  const LineIO& io = p.io;
  if (io.skip && *io.skip) return;
  extern __shared__ __align__(16) double2 rbuf[];
  __shared__ double red[32];
  const int tid = threadIdx.x, nth = blockDim.x, n = p.n, line = blockIdx.x;
  constexpr int H = HC, M = 2 * HC;  // M = L - 1 DST outputs per line
  const long rb = (long)line * n + p.off - 1;
  auto pack = [&](int t, double x) {  // position q >= H holds -a_{q-H}
    int q = (int)__ldg(&p.pl.rin[t - 1]);
    if (q >= H) {
      q -= H;
      x = -x;
    }
    reinterpret_cast<double*>(rbuf)[2 * q + (t & 1)] = x;
  };
  auto unpack = [&](int k) {  // C_k = sgn conj(psi^m' R_m') / H, 1/H in scale
    int m = (int)__ldg(&p.pl.rout[k - 1]);
    double sgn = 1.0;
    if (m >= H) {
      m -= H;
      sgn = -1.0;
    }
    const double2 P = cmul(__ldg(&p.pl.psi[m]), rbuf[m]);
    const double cx = sgn * P.x, cy = -sgn * P.y;
    return ((k & 1) ? -(cy + cx) : -(cy - cx)) * p.scale;
  };
  auto in_at = [&](int e) {
    if (!io.in_seg) return io.in[(long)line * n + e];
    return io.in[(long)(e / io.in_seg) * io.in_seg_stride + (long)line * io.in_seg + e % io.in_seg];
  };
  for (int t = 1 + tid; t <= M; t += nth) {
    double x = in_at(p.off - 1 + t);
    if (io.pre) x = io.pre_mul ? x * io.pre[rb + t] : x / io.pre[rb + t];
    pack(t, x);
  }
  __syncthreads();
  rader_convolve_neg<HC>(rbuf, p.pl);
  if (io.mid_mul) {
    constexpr int kV = (M + kRaderNegThreads - 1) / kRaderNegThreads;
    double v[kV];
#pragma unroll
    for (int s = 0; s < kV; ++s) {
      const int t = 1 + tid + s * nth;
      v[s] = t <= M ? unpack(t) * io.mid_mul[rb + t] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int s = 0; s < kV; ++s) {
      const int t = 1 + tid + s * nth;
      if (t <= M) pack(t, v[s]);
    }
    __syncthreads();
    rader_convolve_neg<HC>(rbuf, p.pl);
  }
  double acc = 0.0;
  for (int t = 1 + tid; t <= M; t += nth) {
    double y = unpack(t);
    if (io.post) y = io.post_mul ? y * io.post[rb + t] : y / io.post[rb + t];
    io.out[rb + t] = y;
    if (io.dot_with) acc += y * io.dot_with[rb + t];
  }
  if (p.off && tid < 2) {  // Shat borders pass through every transform
    const long g = (long)line * n + (tid ? n - 1 : 0);
    double v = in_at(tid ? n - 1 : 0);
    if (io.pre) v = io.pre_mul ? v * io.pre[g] : v / io.pre[g];
    if (io.mid_mul) v *= io.mid_mul[g];
    if (io.post) v = io.post_mul ? v * io.post[g] : v / io.post[g];
    io.out[g] = v;
    if (io.dot_with) acc += v * io.dot_with[g];
  }
  if (io.partial) {
    const double s = block_sum(acc, red);
    if (tid == 0) io.partial[blockIdx.x] = s;
    if (io.fin.s) pcg_fin_tail(io.fin, io.partial, gridDim.x, red);
  }
}

// Band projection of one line (sine family, k_band in tvd_lines.cu): the even slots carry b0,
// the odd slots c1 b1, packed as one complex sequence c_j = (b0_j, c1 b1_j), j = 1..L-1
// (c_0 = 0), whose length-L DFT the Rader convolution computes; the real FFT of length 2L is
// recombined per output t with w_t = exp(-i pi t / L).  One line per CTA.
struct BandRaderK {
  RaderPlan pl;
  int n, L;
  const double2* wfull;
  BandLines b;
};

template <int MC>
__global__ void __launch_bounds__(kRaderThreads, 1) k_band_rader(const BandRaderK p) {
  extern __shared__ __align__(16) double2 rbuf[];
  __shared__ double red[32];
  __shared__ double tots[2];
  const int tid = threadIdx.x, nth = blockDim.x, n = p.n, L = p.L, line = blockIdx.x;
  constexpr int M = MC;
  const BandLines& b = p.b;
  auto B0 = [&](int j) { return b.b0[(long)line * b.b0_ls + (long)j * b.b0_es]; };
  auto B1 = [&](int j) { return b.b1[(long)line * b.b1_ls + (long)j * b.b1_es]; };
  double t0 = 0.0, t1 = 0.0;
  for (int m = 1 + tid; m <= M; m += nth) {
    const double e = B0(m);  // m <= L - 1 = n - 2
    const double o = (b.b1 && m <= L - 2) ? b.c1 * B1(m) : 0.0;
    rbuf[__ldg(&p.pl.dlg[m - 1])] = make_double2(e, o);
    t0 += e;
    if (b.b1 && m <= L - 2) t1 += B1(m);
  }
  t0 = block_sum(t0, red);
  if (tid == 0) tots[0] = t0;
  t1 = block_sum(t1, red);
  if (tid == 0) tots[1] = t1;
  __syncthreads();
  rader_convolve<MC>(rbuf, p.pl);
  const double inv_m = 1.0 / M;
  auto Ck = [&](int k) {  // forward DFT coefficient k = 1..M: conj(R) / M
    const double2 R = rbuf[__ldg(&p.pl.rout[k - 1])];
    return make_double2(R.x * inv_m, -R.y * inv_m);
  };
  double vmin = 1.0 / 0.0, vmax = -1.0 / 0.0;
  const double T0 = tots[0], T1 = tots[1];
  for (int t = tid; t < n; t += nth) {
    double v;
    if (t == 0 || t == n - 1) {
      v = B0(t);
    } else {
      const double2 C = Ck(t), Cr = cconj(Ck(L - t));
      const double2 E = cscale(cadd(C, Cr), 0.5);
      const double2 D = csub(C, Cr);
      const double2 O = make_double2(0.5 * D.y, -0.5 * D.x);
      const double2 w = p.wfull[t];
      const double re_s = E.x + (w.x * O.x - w.y * O.y);
      v = (T0 + b.c1 * T1 * w.x - re_s) / L;
    }
    const long g = (long)line * b.out_ls + (long)t * b.out_es;
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

}  // namespace

cudaError_t launch_band_rader(const RaderPlan& P, int n, const double2* wfull, const BandLines& b,
                              int* nblocks_out, cudaStream_t st) {
  if (P.M != 8190 || n != P.L + 1 || !P.dlg) return cudaErrorInvalidConfiguration;
  BandRaderK k{};
  k.pl = P;
  k.n = n;
  k.L = P.L;
  k.wfull = wfull;
  k.b = b;
  const size_t smem = (size_t)(P.M + RaderStages<8190>::kScratch) * sizeof(double2);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_band_rader<8190>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         200 * 1024);
    attr = true;
  }
  if (nblocks_out) *nblocks_out = b.nlines;
  if (b.nlines == 0) return cudaSuccess;
  k_band_rader<8190><<<b.nlines, kRaderThreads, smem, st>>>(k);
  return cudaGetLastError();
}

bool rader_launchable(const RaderPlan& P, int len, int family) {
  return P.M == 8190 && (family == kFamSineHat ? len == P.M + 2 : len == P.M);
}

cudaError_t launch_rader_rows(const RaderPlan& P, int family, int len, int nlines,
                              const LineIO& io, int* nblocks_out, cudaStream_t st) {
  if (!rader_launchable(P, len, family)) return cudaErrorInvalidConfiguration;
  RaderK k{};
  k.pl = P;
  k.n = len;
  k.off = family == kFamSineHat ? 1 : 0;
  k.nlines = nlines;
  k.scale = 0.5 * sqrt(2.0 / (P.M + 1)) / P.M;
  k.io = io;
  const size_t smem = (size_t)(P.M + RaderStages<8190>::kScratch) * sizeof(double2);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_rader_rows<8190>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         200 * 1024);
    attr = true;
  }
  if (nblocks_out) *nblocks_out = nlines;
  if (nlines == 0) return cudaSuccess;
  if (P.H == 4095 && P.psi) {  // negacyclic half-length engine (the full one: 11.5 vs 7.75 ms)
    k.scale = 0.5 * sqrt(2.0 / (P.M + 1)) / P.H;
    const size_t smem_h = (size_t)(P.H + RaderStages<4095>::kScratch) * sizeof(double2);
    static bool attr_h = false;
    if (!attr_h) {
      cudaFuncSetAttribute(k_rader_rows_neg<4095>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)smem_h);
      attr_h = true;
    }
    return launch_pdl(k_rader_rows_neg<4095>, nlines, kRaderNegThreads, smem_h, st, k);
  }
  return launch_pdl(k_rader_rows<8190>, nlines, kRaderThreads, smem, st, k);
}

int rader_threads() { return kRaderThreads; }

}  // namespace tvd

// ------------------------------------------------------------------- host plan
#include <cmath>

namespace tvd {
namespace {

long long powmod(long long b, long long e, long long m) {
  long long r = 1 % m;
  b %= m;
  while (e > 0) {
    if (e & 1) r = r * b % m;
    b = b * b % m;
    e >>= 1;
  }
  return r;
}

template <class T>
bool upload_vec(const std::vector<T>& h, const T** out, std::vector<void*>& owned) {
  void* d = nullptr;
  if (cudaMalloc(&d, h.size() * sizeof(T)) != cudaSuccess) return false;
  owned.push_back(d);
  if (cudaMemcpy(d, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice) != cudaSuccess)
    return false;
  *out = static_cast<const T*>(d);
  return true;
}

// (cos, sin)(2 pi e / m) with exact integer reduction, long double
void cis_ld(long long e, long long m, long double* c, long double* s) {
  e %= m;
  if (e < 0) e += m;
  const long double a = 2.0L * 3.14159265358979323846264338327950288L * (long double)e / (long double)m;
  *c = cosl(a);
  *s = sinl(a);
}

}  // namespace

bool build_rader_plan(int L, RaderPlan* P, std::vector<void*>& owned) {
  *P = RaderPlan{};
  if (L < 5 || L - 1 > 8190) return false;
  for (int d = 2; (long long)d * d <= L; ++d)
    if (L % d == 0) return false;  // not prime
  const int M = L - 1;
  // stages: the length-M FFT factors into codelet radices
  std::vector<int> rad;
  int m = M;
  for (int p : {8, 4, 2, 3, 5, 7, 11, 13})
    while (m % p == 0) {
      rad.push_back(p);
      m /= p;
    }
  if (m != 1 || (int)rad.size() > kRaderMaxStages) return false;
  const int nth = rader_threads();
  P->L = L;
  P->M = M;
  P->nst = (int)rad.size();
  int ns = 1;
  for (int s = 0; s < P->nst; ++s) {
    const int items = M / rad[s];
    int sl = (items + nth - 1) / nth;
    if (sl > 16) return false;
    P->radix[s] = rad[s];
    P->ns[s] = ns;
    P->slots[s] = sl;
    ns *= rad[s];
  }
  // generator of Z_L^*
  std::vector<int> primes;
  for (int x = M, d = 2; x > 1; ++d)
    if (x % d == 0) {
      primes.push_back(d);
      while (x % d == 0) x /= d;
    }
  int g = 2;
  for (;; ++g) {
    bool ok = true;
    for (int p : primes)
      if (powmod(g, M / p, L) == 1) ok = false;
    if (ok) break;
  }
  P->g = g;
  std::vector<int> dlog(L, -1);
  long long pw = 1;
  for (int e = 0; e < M; ++e) {
    dlog[pw] = e;
    pw = pw * g % L;
  }
  const int h = (L - 1) / 2;
  std::vector<unsigned> rin(M), rout(M), dlg(M);
  for (int m = 1; m <= M; ++m) dlg[m - 1] = (unsigned)dlog[m];
  for (int t = 1; t <= M; ++t) {
    int j = (t & 1) == 0 ? t / 2 : (t - 1) / 2 - h;
    if (j < 0) j += L;
    rin[t - 1] = (unsigned)dlog[j];
    rout[t - 1] = (unsigned)((M - dlog[t]) % M);
  }
  // b_q = w^{g^-q}; bh = FFT_M(b) (direct, long double)
  const long long ginv = powmod(g, M - 1, L);
  std::vector<long double> bre(M), bim(M), cm(M), sm(M);
  pw = 1;
  for (int q = 0; q < M; ++q) {
    long double c, s;
    cis_ld(pw, L, &c, &s);
    bre[q] = c;
    bim[q] = -s;
    pw = pw * ginv % L;
  }
  for (int e = 0; e < M; ++e) cis_ld(e, M, &cm[e], &sm[e]);
  std::vector<double2> bh(M), tw(M);
  for (int k = 0; k < M; ++k) {
    long double xr = 0, xi = 0;
    int idx = 0;
    for (int q = 0; q < M; ++q) {  // sum_q b_q exp(-2 pi i q k / M)
      const long double c = cm[idx], s = sm[idx];
      xr += bre[q] * c + bim[q] * s;
      xi += bim[q] * c - bre[q] * s;
      idx += k;
      if (idx >= M) idx -= M;
    }
    bh[k] = make_double2((double)xr, (double)xi);
    tw[k] = make_double2((double)cm[k], -(double)sm[k]);
  }
  // negacyclic half-length tables: beta_n = b_n - b_{n+H}, beta~ = beta psi^n, bhh = FFT_H
  const int H = M / 2;
  std::vector<double2> psi(H), twh(H), bhh(H);
  std::vector<long double> tr(H), ti(H), ch(H), sh(H);
  for (int e = 0; e < H; ++e) {
    long double c, s;
    cis_ld(e, 2LL * H, &c, &s);  // exp(i pi e / H)
    psi[e] = make_double2((double)c, (double)s);
    tr[e] = (bre[e] - bre[e + H]) * c - (bim[e] - bim[e + H]) * s;
    ti[e] = (bre[e] - bre[e + H]) * s + (bim[e] - bim[e + H]) * c;
    cis_ld(e, H, &ch[e], &sh[e]);
    twh[e] = make_double2((double)ch[e], -(double)sh[e]);
  }
  for (int k = 0; k < H; ++k) {
    long double xr = 0, xi = 0;
    int idx = 0;
    for (int q = 0; q < H; ++q) {  // sum_q beta~_q exp(-2 pi i q k / H)
      xr += tr[q] * ch[idx] + ti[q] * sh[idx];
      xi += ti[q] * ch[idx] - tr[q] * sh[idx];
      idx += k;
      if (idx >= H) idx -= H;
    }
    bhh[k] = make_double2((double)xr, (double)xi);
  }
  P->H = H;
  if (!upload_vec(rin, &P->rin, owned) || !upload_vec(rout, &P->rout, owned) ||
      !upload_vec(bh, &P->bh, owned) || !upload_vec(tw, &P->tw, owned) ||
      !upload_vec(dlg, &P->dlg, owned) || !upload_vec(psi, &P->psi, owned) ||
      !upload_vec(twh, &P->twh, owned) || !upload_vec(bhh, &P->bhh, owned))
    return false;
  return true;
}

}  // namespace tvd
