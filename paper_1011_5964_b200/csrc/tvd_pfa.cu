// Odd-symmetric prime-factor DST-I engine (the Shat / M preconditioner passes).
//
// A DST-I of length N = L - 1 with L odd is one complex DFT of length L of the
// packed odd-extension sequence c'_j = z_{2j} + i z_{2((j+h) mod L)+1}
// (tvd_lines.cu).  c' is odd (c'_{L-j} = -c'_j), so is its DFT.  With
// L = q_1 q_2 ... q_d (pairwise coprime, d <= 3) the Good-Thomas map
//   input  j <-> (j_s = (j mod q_s) * (L/q_s)^{-1} mod q_s)   (Ruritanian)
//   output k <-> (k_s = k mod q_s)                            (CRT)
// turns the DFT into a d-dimensional DFT without twiddles, computed in place
// one dimension at a time.  Negating j negates every index, so along each
// dimension only one DFT of every {tau, -tau} pair of "other-index" tuples is
// computed; its partner line is written as the negated, index-reversed copy.
// That halves the arithmetic of the generic FFT, and the self-paired line
// (tau = 0) is odd, so its DFT needs only the sine half.  Each q-point DFT
// folds inputs into a_r = x_r + x_{q-r}, b_r = x_r - x_{q-r} and accumulates
// KB output pairs per work item from a (cos, sin) matrix laid out so the KB
// coefficients of one r are contiguous (immediate-offset loads).
// Reference semantics: transforms.py:52-81 (dst1_apply / sinehat_apply).
#include <cstdlib>

#include "tvd_internal.h"

namespace tvd {

__device__ __forceinline__ int fdiv(int x, const FDiv& f) {
  return (int)(((unsigned long long)(unsigned)x * f.m) >> 40);
}
__device__ __forceinline__ int fmodq(int x, const FDiv& f) { return x - fdiv(x, f) * f.d; }

struct PfaK {
  PfaPlan pl;
  int n, off, N, nl, nlines;
  int stages;  // number of PFA stages to run (profiling knob; default = all)
  long ls, es;
  double scale;  // 0.5 * sqrt(2 / L)
  int h;         // (L - 1) / 2
  LineIO io;
};

// representative "other-index" tuple t -> (a, b)
__device__ __forceinline__ void rep_tuple(int t, const PfaStage& S, int& a, int& b) {
  if (t < S.h2) {
    a = 0;
    b = t;
  } else {
    const int u = t - S.h2;
    const int qd = fdiv(u, S.fD2);
    a = 1 + qd;
    b = u - qd * S.D2;
  }
}

// fold x_r, x_{q-r} -> a_r = x_r + x_{q-r}, b_r = x_r - x_{q-r} for every representative line
__device__ __forceinline__ void pfa_fold(double2* buf, int LP, int nl, const PfaStage& S) {
  const int tid = threadIdx.x, nth = blockDim.x;
  const int q = S.q, H = S.H, st = S.st;
  const int nfold = nl * S.Rcnt * H;
  for (int i = tid; i < nfold; i += nth) {
    const int rest = fdiv(i, S.fRcnt);
    const int t = i - rest * S.Rcnt;
    const int line = fdiv(rest, S.fH);
    const int r = 1 + rest - line * H;
    int a, b;
    rep_tuple(t, S, a, b);
    double2* p = buf + line * LP + a * S.S1 + b * S.S2;
    const double2 x1 = p[r * st], x2 = p[(q - r) * st];
    p[r * st] = cadd(x1, x2);
    p[(q - r) * st] = csub(x1, x2);
  }
  __syncthreads();
}

// DFT index (line-major over the CTA's representative lines) -> (base, negated base, self)
__device__ __forceinline__ void dft_lines(int dft, const PfaStage& S, int LP, int& base, int& neg,
                                          bool& self) {
  const int line = fdiv(dft, S.fRcnt);
  const int t = dft - line * S.Rcnt;
  int a, b;
  rep_tuple(t, S, a, b);
  self = (t == 0);
  base = line * LP + a * S.S1 + b * S.S2;
  const int na = a == 0 ? 0 : S.D1 - a, nb = b == 0 ? 0 : S.D2 - b;
  neg = line * LP + na * S.S1 + nb * S.S2;
}

// D(8x8) += A(8x4) * B(4x8), fp64 tensor-core MMA (SASS DMMA.884).
__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

constexpr int kMmaTiles = 8;  // output tiles a warp holds across the in-place barrier

// One stage as a batched GEMM on the fp64 tensor cores:
//   A_k = sum_r cos(2 pi r k / q) a_r   (row k = 0 of the cosine matrix is all ones -> V_0)
//   B_k = sum_r sin(2 pi r k / q) b_r
// The columns of the data operand are (DFT, re/im) pairs of the CTA's representative lines;
// a warp tile covers 8 output rows k x 4 DFTs and keeps both accumulators, so every lane
// finishes with A_k, B_k (re, im) of one (k, DFT) pair and forms V_k, V_{q-k} directly.
__device__ __forceinline__ void pfa_dft_mma(double2* buf, int LP, int nl, const PfaStage& S) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int q = S.q, H = S.H, st = S.st;
  const int ndft = nl * S.Rcnt;
  const int nkt = S.KP >> 3, nct = (2 * ndft + 7) >> 3, nrs = S.RP >> 2;
  int ctr = (nw * kMmaTiles) / nkt;  // column tiles per round (all k-tiles of a column together)
  if (ctr < 1) ctr = 1;
  const double* bufd = reinterpret_cast<const double*>(buf);
  for (int ct0 = 0; ct0 < nct; ct0 += ctr) {
    const int ntile = nkt * min(ctr, nct - ct0);
    double2 vk[kMmaTiles], vm[kMmaTiles];
    int ob[kMmaTiles], on[kMmaTiles], oflag[kMmaTiles];
#pragma unroll
    for (int s = 0; s < kMmaTiles; ++s) {
      oflag[s] = 0;
      const int tile = warp + s * nw;
      if (tile < ntile) {  // warp-uniform
        const int ct = ct0 + tile / nkt, kt = tile - (tile / nkt) * nkt;
        double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
        const int colB = ct * 8 + (lane >> 2);
        const int dB = colB >> 1;
        const bool vB = dB < ndft;
        int baseB = 0, negB;
        bool selfB;
        if (vB) dft_lines(dB, S, LP, baseB, negB, selfB);
        const double* pb = bufd + 2 * baseB + (colB & 1);
        const int krow = kt * 8 + (lane >> 2);
        const double* cm = S.Cm + krow * S.RP + (lane & 3);
        const double* sm = S.Sm + krow * S.RP + (lane & 3);
        for (int rs = 0; rs < nrs; ++rs) {
          const int r = 1 + rs * 4 + (lane & 3);
          double xa = 0.0, xb = 0.0;
          if (vB && r <= H) {
            xa = pb[2 * r * st];
            xb = pb[2 * (q - r) * st];
          }
          dmma884(a0, a1, __ldg(cm + rs * 4), xa);
          dmma884(b0, b1, __ldg(sm + rs * 4), xb);
        }
        const int dO = ct * 4 + (lane & 3);
        if (krow <= H && dO < ndft) {
          int base, neg;
          bool self;
          dft_lines(dO, S, LP, base, neg, self);
          const double2 x0 = buf[base];
          vk[s] = make_double2(x0.x + a0 + b1, x0.y + a1 - b0);
          vm[s] = make_double2(x0.x + a0 - b1, x0.y + a1 + b0);
          ob[s] = base;
          on[s] = neg;
          oflag[s] = 1 | (self ? 2 : 0);
        }
      }
    }
    __syncthreads();
#pragma unroll
    for (int s = 0; s < kMmaTiles; ++s) {
      if (oflag[s]) {
        const int tile = warp + s * nw;
        const int kt = tile - (tile / nkt) * nkt;
        const int k = kt * 8 + (lane >> 2);
        double2* p = buf + ob[s];
        double2* pn = buf + on[s];
        const bool self = oflag[s] & 2;
        if (k == 0) {
          p[0] = vk[s];
          if (!self) pn[0] = make_double2(-vk[s].x, -vk[s].y);
        } else {
          p[k * st] = vk[s];
          p[(q - k) * st] = vm[s];
          if (!self) {
            pn[(q - k) * st] = make_double2(-vk[s].x, -vk[s].y);
            pn[k * st] = make_double2(-vm[s].x, -vm[s].y);
          }
        }
      }
    }
    __syncthreads();
  }
}

template <int KB>
__device__ __forceinline__ void pfa_stage(double2* buf, int LP, int nl, const PfaStage& S) {
  const int tid = threadIdx.x, nth = blockDim.x;
  const int q = S.q, H = S.H, st = S.st;
  pfa_fold(buf, LP, nl, S);
  if (S.use_mma) {
    pfa_dft_mma(buf, LP, nl, S);
    return;
  }
  const int nch = S.nch;
  const int ndft = nl * S.Rcnt;
  const bool all_self = S.D1 * S.D2 == 1;  // prime L: the only line is odd
  int dpr = nth / nch;  // DFTs per round (all chunks of a DFT share a round)
  for (int d0 = 0; d0 < ndft; d0 += dpr) {
    const int dr = min(dpr, ndft - d0);
    const int items = dr * nch;
    const bool active = tid < items;
    double2 A[KB], B[KB];
    double2 x0 = make_double2(0.0, 0.0), s0 = x0;
    int c = 0, base = 0, neg = 0;
    bool self = false;
    if (active) {
      // DFT index fastest across lanes: the chunk (coefficient rows) is warp-uniform
      c = tid / dr;
      const int dft = d0 + tid - c * dr;
      const int line = fdiv(dft, S.fRcnt);
      const int t = dft - line * S.Rcnt;
      int a, b;
      rep_tuple(t, S, a, b);
      self = (t == 0);
      base = line * LP + a * S.S1 + b * S.S2;
      const int na = a == 0 ? 0 : S.D1 - a, nb = b == 0 ? 0 : S.D2 - b;
      neg = line * LP + na * S.S1 + nb * S.S2;
#pragma unroll
      for (int k = 0; k < KB; ++k) {
        A[k] = make_double2(0.0, 0.0);
        B[k] = make_double2(0.0, 0.0);
      }
      const double2* p = buf + base;
      x0 = p[0];
      s0 = x0;
      const double2* m = S.M + c * KB;
      if (all_self) {  // odd line: a_r == 0, only the sine half contributes
#pragma unroll 2
        for (int r = 1; r <= H; ++r, m += H) {
          const double2 bb = p[(q - r) * st];
#pragma unroll
          for (int k = 0; k < KB; ++k) {
            const double sn = __ldg(&m[k].y);
            B[k].x += bb.x * sn;
            B[k].y += bb.y * sn;
          }
        }
      } else {
#pragma unroll 2
        for (int r = 1; r <= H; ++r, m += H) {
          const double2 aa = p[r * st], bb = p[(q - r) * st];
          s0 = cadd(s0, aa);
#pragma unroll
          for (int k = 0; k < KB; ++k) {
            const double2 w = __ldg(&m[k]);
            A[k].x += aa.x * w.x;
            A[k].y += aa.y * w.x;
            B[k].x += bb.x * w.y;
            B[k].y += bb.y * w.y;
          }
        }
      }
    }
    __syncthreads();
    if (active) {
      double2* p = buf + base;
      double2* pn = buf + neg;
      if (c == 0) {
        p[0] = s0;
        if (!self) pn[0] = make_double2(-s0.x, -s0.y);
      }
      const int k0 = 1 + c * KB;
#pragma unroll
      for (int kk = 0; kk < KB; ++kk) {
        const int k = k0 + kk;
        if (k <= H) {
          const double2 vk = make_double2(x0.x + A[kk].x + B[kk].y, x0.y + A[kk].y - B[kk].x);
          const double2 vm = make_double2(x0.x + A[kk].x - B[kk].y, x0.y + A[kk].y + B[kk].x);
          p[k * st] = vk;
          p[(q - k) * st] = vm;
          if (!self) {
            pn[(q - k) * st] = make_double2(-vk.x, -vk.y);
            pn[k * st] = make_double2(-vm.x, -vm.y);
          }
        }
      }
    }
    __syncthreads();
  }
}

// position of c'_j in the PFA layout (Ruritanian input map) and of c'_{-j}
__device__ __forceinline__ void in_pos(int j, const PfaPlan& pl, int& pos, int& npos) {
  pos = 0;
  npos = 0;
#pragma unroll
  for (int s = 0; s < 3; ++s) {
    if (s < pl.d) {
      const int m = fmodq(fmodq(j, pl.fq[s]) * pl.rinv[s], pl.fq[s]);
      pos += m * pl.stride[s];
      npos += (m == 0 ? 0 : pl.q[s] - m) * pl.stride[s];
    }
  }
}

__device__ __forceinline__ int out_pos(int k, const PfaPlan& pl) {
  int pos = 0;
#pragma unroll
  for (int s = 0; s < 3; ++s)
    if (s < pl.d) pos += fmodq(k, pl.fq[s]) * pl.stride[s];
  return pos;
}

// scatter x_t (t = 1..N) into the packed odd sequence: z_t = x_t, z_{2L-t} = -x_t
__device__ __forceinline__ void scatter_x(double2* line, int t, double v, const PfaK& p) {
  const int L = p.pl.L;
  int j, comp;
  if ((t & 1) == 0) {
    j = t >> 1;
    comp = 0;
  } else {
    j = ((t - 1) >> 1) - p.h;
    if (j < 0) j += L;
    comp = 1;
  }
  int pos, npos;
  in_pos(j, p.pl, pos, npos);
  double* a = reinterpret_cast<double*>(line + pos) + comp;
  double* b = reinterpret_cast<double*>(line + npos) + comp;
  *a = v;
  *b = -v;
}

__device__ __forceinline__ double gather_y(const double2* line, int k, const PfaK& p) {
  const double2 C = line[out_pos(k, p.pl)];
  const double y = (k & 1) ? -(C.y + C.x) : -(C.y - C.x);
  return y * p.scale;
}

__device__ __forceinline__ void pfa_transform(double2* buf, int LP, int nl, const PfaK& p) {
  for (int s = 0; s < p.pl.d; ++s) {
    const PfaStage& S = p.pl.st[s];
    pfa_stage<4>(buf, LP, nl, S);
  }
}

constexpr int kPfaMaxV = 8;   // per-thread register values in the sandwich re-pack
constexpr int kPfaBatch = 8;  // global loads in flight per thread in the pack

__global__ void __launch_bounds__(256, 2) k_pfa(const PfaK p) {
  const LineIO& io = p.io;
  if (io.skip && *io.skip) return;
  extern __shared__ double2 smem2[];
  __shared__ double red[32];
  const int tid = threadIdx.x, nth = blockDim.x;
  const int LP = p.pl.LP, N = p.N, nl = p.nl;
  const int line0 = blockIdx.x * nl;
  const int nlv = min(nl, p.nlines - line0);
  double2* buf = smem2;
  auto gidx = [&](int l, int t) {  // t: 1..N interior index
    return (long)(line0 + l) * p.ls + (long)(p.off + t - 1) * p.es;
  };
  // zero slot of every line (c'_0 = 0) and dead lines
  for (int i = tid; i < nl; i += nth) buf[i * LP] = make_double2(0.0, 0.0);
  for (int i = tid; i < (nl - nlv) * LP; i += nth) buf[nlv * LP + i] = make_double2(0.0, 0.0);
  // element i of this CTA's lines -> (line, t), memory-friendly order
  const bool contig = p.es == 1;
  auto split = [&](int i, int& l, int& t) {
    if (contig) {
      l = fdiv(i, p.pl.fN);
      t = 1 + i - l * N;
    } else {
      t = 1 + (nlv == 2 ? (i >> 1) : i / nlv);
      l = i - (t - 1) * nlv;
    }
  };
  // pack: kPfaBatch global loads in flight per thread, then the smem scatter
  const int total = nlv * N;
  for (int i0 = 0; i0 < total; i0 += kPfaBatch * nth) {
    double v[kPfaBatch];
#pragma unroll
    for (int s = 0; s < kPfaBatch; ++s) {
      const int i = i0 + tid + s * nth;
      if (i < total) {
        int l, t;
        split(i, l, t);
        const long g = gidx(l, t);
        v[s] = io.in[g];
        if (io.pre) v[s] = io.pre_mul ? v[s] * io.pre[g] : v[s] / io.pre[g];
      }
    }
#pragma unroll
    for (int s = 0; s < kPfaBatch; ++s) {
      const int i = i0 + tid + s * nth;
      if (i < total) {
        int l, t;
        split(i, l, t);
        scatter_x(buf + l * LP, t, v[s], p);
      }
    }
  }
  __syncthreads();
  pfa_transform(buf, LP, nl, p);

  if (io.mid_mul) {
    // y <- mid .* y, re-packed line by line through registers, then transform again
    for (int l = 0; l < nlv; ++l) {
      double v[kPfaMaxV];
#pragma unroll
      for (int s = 0; s < kPfaMaxV; ++s) {
        const int t = 1 + tid + s * nth;
        v[s] = t <= N ? gather_y(buf + l * LP, t, p) * io.mid_mul[gidx(l, t)] : 0.0;
      }
      __syncthreads();
#pragma unroll
      for (int s = 0; s < kPfaMaxV; ++s) {
        const int t = 1 + tid + s * nth;
        if (t <= N) scatter_x(buf + l * LP, t, v[s], p);
      }
      __syncthreads();
    }
    for (int l = nlv; l < nl; ++l)
      for (int i = tid; i < LP; i += nth) buf[l * LP + i] = make_double2(0.0, 0.0);
    for (int l = tid; l < nlv; l += nth) buf[l * LP] = make_double2(0.0, 0.0);  // c'_0
    __syncthreads();
    pfa_transform(buf, LP, nl, p);
  }

  // unpack + store
  double acc = 0.0;
  auto store = [&](long g, double v) {
    if (io.post) v = io.post_mul ? v * io.post[g] : v / io.post[g];
    io.out[g] = v;
    if (io.dot_with) acc += v * io.dot_with[g];
  };
  for (int i = tid; i < total; i += nth) {
    int l, t;
    split(i, l, t);
    store(gidx(l, t), gather_y(buf + l * LP, t, p));
  }
  if (p.off) {  // Shat borders pass through every transform
    for (int i = tid; i < 2 * nlv; i += nth) {
      const int l = i >> 1;
      const long g = (long)(line0 + l) * p.ls + (long)((i & 1) ? p.n - 1 : 0) * p.es;
      double v = io.in[g];
      if (io.pre) v = io.pre_mul ? v * io.pre[g] : v / io.pre[g];
      if (io.mid_mul) v *= io.mid_mul[g];
      store(g, v);
    }
  }
  if (io.partial) {
    const double s = block_sum(acc, red);
    if (tid == 0) io.partial[blockIdx.x] = s;
  }
}

// ------------------------------------------------ compile-time specialised kernel
#ifdef TVD_PIPE_TIMING
__device__ unsigned long long g_pipe_phase[8];      // profiling only
__device__ unsigned long long g_stage_t[2 * 16 * 4];  // [stage q=89|other][warp][phase]
#endif
#include "tvd_pfa_t.cuh"

constexpr int kPfaLinesT = 2;  // lines per CTA of the specialised kernel

template <int Q1, int Q2, int Q3>
__device__ __forceinline__ void pfa_transform_c(double2* buf, unsigned* const* reps,
                                                const PfaPlan& pl, int stages) {
  using SH = PfaShape<Q1, Q2, Q3>;
  if (stages >= 1)
    pfa_stage_c<PfaStageC<SH, 0>, kPfaLinesT, 4, 8>(buf, buf, reps[0], pl.st[0].Cm, pl.st[0].Sm,
                pl.st[0].Cf, pl.st[0].Sf);
  if constexpr (SH::d >= 2)
    if (stages >= 2)
      pfa_stage_c<PfaStageC<SH, 1>, kPfaLinesT, 4, 8>(buf, buf, reps[1], pl.st[1].Cm, pl.st[1].Sm,
                pl.st[1].Cf, pl.st[1].Sf);
  if constexpr (SH::d >= 3)
    if (stages >= 3)
      pfa_stage_c<PfaStageC<SH, 2>, kPfaLinesT, 4, 8>(buf, buf, reps[2], pl.st[2].Cm, pl.st[2].Sm,
                pl.st[2].Cf, pl.st[2].Sf);
}

template <int Q1, int Q2, int Q3>
__global__ void __launch_bounds__(256, 2) k_pfa_t(const PfaK p) {
  using SH = PfaShape<Q1, Q2, Q3>;
  constexpr int LP = SH::LP, N = SH::N, NL = kPfaLinesT;
  const LineIO& io = p.io;
  if (io.skip && *io.skip) return;
  extern __shared__ double2 smem2[];
  __shared__ double red[32];
  const int tid = threadIdx.x, nth = blockDim.x;
  double2* buf = smem2;
  unsigned* scat = reinterpret_cast<unsigned*>(buf + NL * LP);
  unsigned* gath = scat + N;
  unsigned* reps[3];
  reps[0] = gath + N;
  reps[1] = reps[0] + PfaStageC<SH, 0>::Rcnt;
  reps[2] = reps[1] + (SH::d >= 2 ? PfaStageC<SH, 1>::Rcnt : 0);
  const int line0 = blockIdx.x * NL;
  const int nlv = min(NL, p.nlines - line0);
  for (int i = tid; i < N; i += nth) {
    scat[i] = p.pl.scat[i];
    gath[i] = p.pl.gath[i];
  }
  for (int s = 0; s < SH::d; ++s) {
    const int rc = s == 0 ? PfaStageC<SH, 0>::Rcnt : (s == 1 ? PfaStageC<SH, 1>::Rcnt
                                                              : PfaStageC<SH, 2>::Rcnt);
    for (int i = tid; i < rc; i += nth) reps[s][i] = p.pl.reps[s][i];
  }
  for (int i = tid; i < NL; i += nth) buf[i * LP] = make_double2(0.0, 0.0);
  for (int i = tid; i < (NL - nlv) * LP; i += nth) buf[nlv * LP + i] = make_double2(0.0, 0.0);
  __syncthreads();
  const bool contig = p.es == 1;
  auto gidx = [&](int l, int t) { return (long)(line0 + l) * p.ls + (long)(p.off + t - 1) * p.es; };
  auto put = [&](int l, int t, double v) {
    const unsigned e = scat[t - 1];
    double* b = reinterpret_cast<double*>(buf + l * LP) + (t & 1);
    b[2 * (e & 0xffffu)] = v;
    b[2 * (e >> 16)] = -v;
  };
  auto get = [&](int l, int k) {
    const double2 C = buf[l * LP + gath[k - 1]];
    return ((k & 1) ? -(C.y + C.x) : -(C.y - C.x)) * p.scale;
  };
  // pack: batched global loads, then the table-driven scatter
  const int total = nlv * N;
  for (int i0 = 0; i0 < total; i0 += kPfaBatch * nth) {
    double v[kPfaBatch];
    int lt[kPfaBatch];
#pragma unroll
    for (int s = 0; s < kPfaBatch; ++s) {
      const int i = i0 + tid + s * nth;
      lt[s] = -1;
      if (i < total) {
        int l, t;
        if (contig) { l = i / N; t = 1 + i - l * N; }
        else { t = 1 + i / nlv; l = i - (t - 1) * nlv; }
        const long g = gidx(l, t);
        double x = io.in[g];
        if (io.pre) x = io.pre_mul ? x * io.pre[g] : x / io.pre[g];
        v[s] = x;
        lt[s] = l * 65536 + t;
      }
    }
#pragma unroll
    for (int s = 0; s < kPfaBatch; ++s)
      if (lt[s] >= 0) put(lt[s] >> 16, lt[s] & 0xffff, v[s]);
  }
  __syncthreads();
  pfa_transform_c<Q1, Q2, Q3>(buf, reps, p.pl, p.stages);
  if (io.mid_mul) {
    for (int l = 0; l < nlv; ++l) {
      double v[kPfaMaxV];
#pragma unroll
      for (int s = 0; s < kPfaMaxV; ++s) {
        const int t = 1 + tid + s * nth;
        v[s] = t <= N ? get(l, t) * io.mid_mul[gidx(l, t)] : 0.0;
      }
      __syncthreads();
#pragma unroll
      for (int s = 0; s < kPfaMaxV; ++s) {
        const int t = 1 + tid + s * nth;
        if (t <= N) put(l, t, v[s]);
      }
      __syncthreads();
    }
    for (int i = tid; i < NL; i += nth) buf[i * LP] = make_double2(0.0, 0.0);
    for (int i = tid; i < (NL - nlv) * LP; i += nth) buf[nlv * LP + i] = make_double2(0.0, 0.0);
    __syncthreads();
    pfa_transform_c<Q1, Q2, Q3>(buf, reps, p.pl, p.stages);
  }
  double acc = 0.0;
  auto store = [&](long g, double v) {
    if (io.post) v = io.post_mul ? v * io.post[g] : v / io.post[g];
    io.out[g] = v;
    if (io.dot_with) acc += v * io.dot_with[g];
  };
  for (int i = tid; i < total; i += nth) {
    int l, t;
    if (contig) { l = i / N; t = 1 + i - l * N; }
    else { t = 1 + i / nlv; l = i - (t - 1) * nlv; }
    store(gidx(l, t), get(l, t));
  }
  if (p.off) {
    for (int i = tid; i < 2 * nlv; i += nth) {
      const int l = i >> 1;
      const long g = (long)(line0 + l) * p.ls + (long)((i & 1) ? p.n - 1 : 0) * p.es;
      double v = io.in[g];
      if (io.pre) v = io.pre_mul ? v * io.pre[g] : v / io.pre[g];
      if (io.mid_mul) v *= io.mid_mul[g];
      store(g, v);
    }
  }
  if (io.partial) {
    const double s = block_sum(acc, red);
    if (tid == 0) io.partial[blockIdx.x] = s;
  }
}

// ------------------------------------- band projections on the prime-factor engine
// One level of level2_project for the sine family (precond.py:106-121, 168-199): per line
// the length-L complex DFT of c_j = (b0_j, c1 b1_j) (even / odd slots of the reference's
// length-2L rfft input), then the band form of k_band (tvd_lines.cu).  The DFT is the
// Good-Thomas grid of the DST engine run as a GENERAL transform (PfaStageG: every
// other-index tuple its own line, no odd-symmetry halving) on the same fp64 tensor-core
// stages -- instead of the generic engine's CUDA-core odd-radix stages.
struct BandPfaK {
  PfaPlan pl;
  const double2* wfull;
  int n;
  BandLines b;
};
constexpr int kBandPfaLines = 2;

template <int Q1, int Q2, int Q3>
__global__ void __launch_bounds__(256, 2) k_band_pfa(const BandPfaK p) {
  using SH = PfaShape<Q1, Q2, Q3>;
  constexpr int LP = SH::LP, L = SH::L, NL = kBandPfaLines;
  extern __shared__ double2 smem2[];
  __shared__ double red[32];
  __shared__ double tot[2 * NL];
  const int tid = threadIdx.x, nth = blockDim.x, n = p.n;
  double2* buf = smem2;
  unsigned* reps[3];
  reps[0] = reinterpret_cast<unsigned*>(buf + NL * LP);
  reps[1] = reps[0] + PfaStageG<SH, 0>::Rcnt;
  reps[2] = reps[1] + (SH::d >= 2 ? PfaStageG<SH, 1>::Rcnt : 0);
  for (int s = 0; s < SH::d; ++s) {
    const int rc = s == 0 ? PfaStageG<SH, 0>::Rcnt
                          : (s == 1 ? PfaStageG<SH, 1>::Rcnt : PfaStageG<SH, 2>::Rcnt);
    for (int i = tid; i < rc; i += nth) reps[s][i] = p.pl.greps[s][i];
  }
  const BandLines& b = p.b;
  const int line0 = blockIdx.x * NL;
  const int nlv = min(NL, b.nlines - line0);
  auto B0 = [&](int l, int j) { return b.b0[(long)(line0 + l) * b.b0_ls + (long)j * b.b0_es]; };
  auto B1 = [&](int l, int j) { return b.b1[(long)(line0 + l) * b.b1_ls + (long)j * b.b1_es]; };
  // every slot of the padded grid is read by some stage: zero it, then scatter the lines
  for (int i = tid; i < NL * LP; i += nth) buf[i] = make_double2(0.0, 0.0);
  __syncthreads();
  for (int i = tid; i < NL * L; i += nth) {
    const int l = i / L, j = i - l * L;
    if (l < nlv) {
      // even slots 2j <- b0[j] (j = 1..N), odd slots 2j+1 <- c1 b1[j] (j = 1..N-1)
      double e = 0.0, o = 0.0;
      if (j >= 1 && j <= L - 1) e = B0(l, j);
      if (b.b1 && j >= 1 && j <= L - 2) o = b.c1 * B1(l, j);
      buf[l * LP + __ldg(p.pl.gscat + j)] = make_double2(e, o);
    }
  }
  {  // per-line band totals (one warp per line, fixed order) as k_band
    const int lane = tid & 31, wid = tid >> 5, nw = nth >> 5;
    for (int l = wid; l < NL; l += nw) {
      double t0 = 0.0, t1 = 0.0;
      if (l < nlv) {
        for (int j = 1 + lane; j < n - 1; j += 32) t0 += B0(l, j);
        if (b.b1)
          for (int j = 1 + lane; j < n - 2; j += 32) t1 += B1(l, j);
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
  pfa_stage_c<PfaStageG<SH, 0>, NL, 4, 8>(buf, buf, reps[0], p.pl.st[0].Cm, p.pl.st[0].Sm,
                p.pl.st[0].Cf, p.pl.st[0].Sf);
  if constexpr (SH::d >= 2)
    pfa_stage_c<PfaStageG<SH, 1>, NL, 4, 8>(buf, buf, reps[1], p.pl.st[1].Cm, p.pl.st[1].Sm,
                p.pl.st[1].Cf, p.pl.st[1].Sf);
  if constexpr (SH::d >= 3)
    pfa_stage_c<PfaStageG<SH, 2>, NL, 4, 8>(buf, buf, reps[2], p.pl.st[2].Cm, p.pl.st[2].Sm,
                p.pl.st[2].Cf, p.pl.st[2].Sf);
  // the band form (k_band's epilogue; C_t from the CRT output position of t)
  auto at = [&](int l, int t) { return buf[l * LP + (t == 0 ? 0u : __ldg(p.pl.gath + t - 1))]; };
  double vmin = 1.0 / 0.0, vmax = -1.0 / 0.0;
  for (int i = tid; i < nlv * n; i += nth) {
    const int l = i / n, t = i - l * n;
    double v;
    if (t == 0 || t == n - 1) {
      v = B0(l, t);
    } else {
      const int tr = L - t;
      const double2 C = at(l, t), Cr = cconj(at(l, tr));
      const double2 E = cscale(cadd(C, Cr), 0.5);
      const double2 D = csub(C, Cr);
      const double2 O = make_double2(0.5 * D.y, -0.5 * D.x);
      const double2 w = p.wfull[t];
      const double re_s = E.x + (w.x * O.x - w.y * O.y);
      const double t0 = tot[2 * l], t1 = tot[2 * l + 1];
      v = (t0 + b.c1 * t1 * w.x - re_s) / L;
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
    for (int o = 16; o > 0; o >>= 1) {
      vmin = fmin(vmin, __shfl_xor_sync(0xffffffffu, vmin, o));
      vmax = fmax(vmax, __shfl_xor_sync(0xffffffffu, vmax, o));
    }
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

// The same projection on the column-owner, out-of-place stages of the DST engine (two-factor
// shapes with two tensor-core stages: 2047 = 89 x 23, 1023 = 33 x 31): one line per CTA in
// the full Good-Thomas layout, X -> Y -> X over two line buffers (one barrier per stage
// instead of two per round), fragment-ordered tables, two 6-warp CTAs per SM whose scatter /
// band-form phases overlap each other's stages.  Per output the DMMA sequence is the
// k-tile-owner stage's: bit-identical to k_band_pfa.
template <int Q1, int Q2, int NW>
__global__ void __launch_bounds__(NW * 32, 2) k_band_pfa_co(const BandPfaK p) {
  using SH = PfaShape<Q1, Q2, 1>;
  constexpr int LP = SH::LP, L = SH::L, NT = NW * 32;
  static_assert(FullStage<SH, 0>::mma && FullStage<SH, 1>::mma, "tensor-core stages only");
  extern __shared__ double2 smem2[];
  __shared__ double red[32];
  __shared__ double tot[2];
  const int tid = threadIdx.x, n = p.n;
  double2* X = smem2;
  double2* Y = smem2 + LP;
  const BandLines& b = p.b;
  const int line = blockIdx.x;
  auto B0 = [&](int j) { return b.b0[(long)line * b.b0_ls + (long)j * b.b0_es]; };
  auto B1 = [&](int j) { return b.b1[(long)line * b.b1_ls + (long)j * b.b1_es]; };
  // The scatter writes every cell the stages read (the L grid cells; the column-owner stages
  // never touch the pad columns), so the line buffer needs no zero fill.  The last warp sums
  // the band totals (one warp, fixed lane-strided order, as k_band) while the others scatter.
  if (tid < NT - 32) {
    for (int j = tid; j < L; j += NT - 32) {
      // even slots 2j <- b0[j] (j = 1..N), odd slots 2j+1 <- c1 b1[j] (j = 1..N-1)
      double e = 0.0, o = 0.0;
      if (j >= 1 && j <= L - 1) e = B0(j);
      if (b.b1 && j >= 1 && j <= L - 2) o = b.c1 * B1(j);
      X[__ldg(p.pl.gscat + j)] = make_double2(e, o);
    }
  } else {
    const int lane = tid & 31;
    double t0 = 0.0, t1 = 0.0;
    for (int j = 1 + lane; j < n - 1; j += 32) t0 += B0(j);
    if (b.b1)
      for (int j = 1 + lane; j < n - 2; j += 32) t1 += B1(j);
    t0 = warp_sum(t0);
    t1 = warp_sum(t1);
    if (lane == 0) {
      tot[0] = t0;
      tot[1] = t1;
    }
  }
  __syncthreads();
  half_stage_co<FullStage<SH, 0>, 1, NW>(X, p.pl.st[0].Cf, p.pl.st[0].Sf, Y);
  half_stage_co<FullStage<SH, 1>, 1, NW>(Y, p.pl.st[1].Cf, p.pl.st[1].Sf, X);
  // the band form (k_band's epilogue; C_t from the CRT output position of t).  Outputs t and
  // L - t read the same two grid cells, so one thread forms both (per output the operations
  // are k_band's; the mirrored output only swaps exact negations and commutative adds).
  auto at = [&](int t) { return X[__ldg(p.pl.gath + t - 1)]; };
  double vmin = 1.0 / 0.0, vmax = -1.0 / 0.0;
  auto emit = [&](int t, double v) {
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
  };
  if (tid < 2) emit(tid ? n - 1 : 0, B0(tid ? n - 1 : 0));
  const double t0 = tot[0], t1 = tot[1];
  for (int t = 1 + tid; t <= (L - 1) / 2; t += NT) {
    const int tr = L - t;
    const double2 Ct = at(t), Ctr = at(tr);
    {
      const double2 C = Ct, Cr = cconj(Ctr);
      const double2 E = cscale(cadd(C, Cr), 0.5);
      const double2 D = csub(C, Cr);
      const double2 O = make_double2(0.5 * D.y, -0.5 * D.x);
      const double2 w = p.wfull[t];
      const double re_s = E.x + (w.x * O.x - w.y * O.y);
      emit(t, (t0 + b.c1 * t1 * w.x - re_s) / L);
    }
    {
      const double2 C = Ctr, Cr = cconj(Ct);
      const double2 E = cscale(cadd(C, Cr), 0.5);
      const double2 D = csub(C, Cr);
      const double2 O = make_double2(0.5 * D.y, -0.5 * D.x);
      const double2 w = p.wfull[tr];
      const double re_s = E.x + (w.x * O.x - w.y * O.y);
      emit(tr, (t0 + b.c1 * t1 * w.x - re_s) / L);
    }
  }
  if (b.epi != 0) {
    for (int o = 16; o > 0; o >>= 1) {
      vmin = fmin(vmin, __shfl_xor_sync(0xffffffffu, vmin, o));
      vmax = fmax(vmax, __shfl_xor_sync(0xffffffffu, vmax, o));
    }
    const int lane = tid & 31, wid = tid >> 5;
    if (lane == 0) {
      red[wid] = vmin;
      red[16 + wid] = vmax;
    }
    __syncthreads();
    if (tid == 0) {
      double a = red[0], z = red[16];
      for (int w = 1; w < NW; ++w) {
        a = fmin(a, red[w]);
        z = fmax(z, red[16 + w]);
      }
      b.partial_minmax[2 * blockIdx.x] = a;
      b.partial_minmax[2 * blockIdx.x + 1] = z;
    }
  }
}

template <int Q1, int Q2, int NW>
static cudaError_t launch_band_pfa_co(const BandPfaK& k, cudaStream_t st) {
  using SH = PfaShape<Q1, Q2, 1>;
  const size_t smem = (size_t)2 * SH::LP * 16;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_band_pfa_co<Q1, Q2, NW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    attr = true;
  }
  k_band_pfa_co<Q1, Q2, NW><<<k.b.nlines, NW * 32, smem, st>>>(k);
  return cudaGetLastError();
}

template <int Q1, int Q2, int Q3>
static cudaError_t launch_band_pfa_t(const BandPfaK& k, int nb, cudaStream_t st) {
  using SH = PfaShape<Q1, Q2, Q3>;
  int reps = PfaStageG<SH, 0>::Rcnt;
  if (SH::d >= 2) reps += PfaStageG<SH, 1>::Rcnt;
  if (SH::d >= 3) reps += PfaStageG<SH, 2>::Rcnt;
  const size_t smem = (size_t)kBandPfaLines * SH::LP * 16 + reps * sizeof(unsigned);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_band_pfa<Q1, Q2, Q3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         200 * 1024);
    attr = true;
  }
  k_band_pfa<Q1, Q2, Q3><<<nb, 256, smem, st>>>(k);
  return cudaGetLastError();
}

// ------------------------------------- persistent TMA-pipelined DST row passes
// One CTA per SM walks batches of kPipeLines contiguous rows.  Thread 0 pulls the
// next batch into a staging buffer with cp.async.bulk (TMA bulk copy, completion on
// an mbarrier) as soon as the current batch has been packed, so global loads overlap
// the FFT stages and the unpack/stores of the current batch.  The output is written
// either row-major or transposed (column segments of kPipeLines doubles), which lets
// the 2D preconditioner run every pass over contiguous rows.
constexpr int kPipeLines = 2;     // lines per batch (power of two)

static bool pfa_specialised(const PfaPlan& P, int* which);

struct PipeK {
  PfaPlan pl;
  int n, off, nlines, transposed;
  int stages;  // profiling knob (TVD_PFA_STAGES): 0 = pack/unpack only
  double scale;
  const double* in;
  double* out;
  const double* pre;       // input layout
  const double* mid;       // input layout
  const double* post;      // output layout
  const double* dot_with;  // output layout
  double* partial;
  const int* skip;
  int pre_mul, post_mul;
  PcgFin fin;
  int ar_mode;  // LineIO::ar_mode
  const double* ar_ql;
  const double* ar_qr;
  int in_seg;          // LineIO::in_seg (0: row-major input)
  long in_seg_stride;
  int in_blocked;      // LineIO::in_blocked (dispatch only: PM bit 3)
};

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned phase) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "TVD_WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra TVD_WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}

// Phase counters of the pipeline kernel (build with -DTVD_PIPE_TIMING; profiling only).
#ifdef TVD_PIPE_TIMING
#define PIPE_T_INIT long long ph_[5] = {0, 0, 0, 0, 0}, tl_ = clock64()
#define PIPE_T(i)                   \
  do {                              \
    if (tid == 0) {                 \
      const long long c_ = clock64(); \
      ph_[i] += c_ - tl_;           \
      tl_ = c_;                     \
    }                               \
  } while (0)
#define PIPE_T_FLUSH                                                       \
  do {                                                                     \
    if (tid == 0)                                                          \
      for (int i_ = 0; i_ < 5; ++i_) atomicAdd(&g_pipe_phase[i_], (unsigned long long)ph_[i_]); \
    if (tid == 0) atomicAdd(&g_pipe_phase[7], 1ull);                       \
  } while (0)
#else
#define PIPE_T_INIT
#define PIPE_T(i) \
  do {            \
  } while (0)
#define PIPE_T_FLUSH \
  do {               \
  } while (0)
#endif

// PFA of the pipeline kernel.  kPipeOOP runs the stages out of place over two line
// buffers (stage 0 reads `a`, writes `b`, then they swap: one barrier per stage, no
// outputs held across barriers) -- measured no faster than in place on B200 at 2047, so
// off.  Returns the buffer holding the result.
constexpr bool kPipeOOP = false;
constexpr bool kPipeAliasStage = true;

template <int Q1, int Q2, int Q3, int NL, int NT, int TPW>
__device__ __forceinline__ double2* pfa_transform_nl(double2* a, double2* b, unsigned* const* reps,
                                                     const PfaPlan& pl, int stages = 3) {
  using SH = PfaShape<Q1, Q2, Q3>;
  constexpr int NW = NT / 32;
  constexpr bool O = kPipeOOP;
  double2* x = a;
  double2* y = O ? b : a;
  if (stages < 1) return a;
  pfa_stage_c<PfaStageC<SH, 0>, NL, 4, NW, TPW, O>(x, y, reps[0], pl.st[0].Cm, pl.st[0].Sm,
                pl.st[0].Cf, pl.st[0].Sf);
  if constexpr (SH::d >= 2) {
    if (stages < 2) return y;
    pfa_stage_c<PfaStageC<SH, 1>, NL, 4, NW, TPW, O>(y, x, reps[1], pl.st[1].Cm, pl.st[1].Sm,
                pl.st[1].Cf, pl.st[1].Sf);
  }
  if constexpr (SH::d >= 3) {
    if (stages < 3) return x;
    pfa_stage_c<PfaStageC<SH, 2>, NL, 4, NW, TPW, O>(x, y, reps[2], pl.st[2].Cm, pl.st[2].Sm,
                pl.st[2].Cf, pl.st[2].Sf);
  }
  return SH::d == 2 ? x : y;
}

// PM: pass mode known at compile time (bit 0: sandwich with mid, bit 1: transposed output),
// -1: read both from the parameters.  The specialised instances carry only their pass's code
// (smaller kernels, fewer live registers, no dead branches).
template <int Q1, int Q2, int Q3, int NT, int MINB, int TPW, bool HALF = false, int BL = kPipeLines,
          bool CSM = false, int PM = -1, bool HO = false, int CO = 0>
__global__ void __launch_bounds__(NT, MINB) k_dst_pipe(const PipeK p) {
  pdl_enter();
  const bool has_mid = PM < 0 ? p.mid != nullptr : (PM & 1) != 0;
  const bool trans = PM < 0 ? p.transposed != 0 : (PM & 2) != 0;
  // pair-blocked layouts (PM bits 2 / 3): element e of line l lives at ((l >> 1) n + e) 2 +
  // (l & 1), so a 2-line batch writes 2 n contiguous doubles and the next pass, whose lines
  // are the columns, reads one 16-byte pair per (block, line) -- instead of 16-byte column
  // segments written at a stride of n doubles
  constexpr bool BOUT = PM >= 0 && (PM & 4) != 0;
  constexpr bool BIN = PM >= 0 && (PM & 8) != 0;
  using SH = PfaShape<Q1, Q2, Q3>;
  static_assert(!HALF || SH::d == 2, "half-line layout is for two-factor lengths");
  // HALF: half-line Good-Thomas layout (tvd_pfa_t.cuh HalfShape), signed scatter / gather
  constexpr int LP = HALF ? HalfShape<Q1, Q2>::LPh : SH::LP, N = SH::N, B = BL;
  constexpr int kTpt = (N + NT - 1) / NT;  // t-values per thread per line
  static_assert((B & (B - 1)) == 0, "transposed store assumes power-of-two batches");
  if (p.skip && *p.skip) return;
  extern __shared__ __align__(16) unsigned char smraw[];
  __shared__ double red[32];
  __shared__ double bord[B][2];
  __shared__ __align__(8) unsigned long long mbar;
  const int tid = threadIdx.x, nth = blockDim.x, n = p.n;
  double2* buf = reinterpret_cast<double2*>(smraw);  // pack target (stage 0 input)
  constexpr bool OOPB = kPipeOOP || (HALF && HO);     // a second line buffer
  double2* buf2 = OOPB ? buf + B * LP : buf;          // second buffer of out-of-place stages
  double2* res = buf;                                 // buffer holding the transform result
  // AL: the staging rows alias the second line buffer (free from the end of a batch's last
  // stage until the next batch's first stage), so the next batch's rows are fetched while
  // this batch unpacks; the CTA then needs two line buffers only (three CTAs per SM at 2047)
  constexpr bool AL = HALF && HO && kPipeAliasStage;
  double* stage = AL ? reinterpret_cast<double*>(buf2)
                     : reinterpret_cast<double*>(buf + (OOPB ? 2 : 1) * B * LP);
  // scatter / gather tables are read coalesced (indexed by t) through L1, leaving the
  // shared memory to the padded lines and the staging rows
  const unsigned* __restrict__ scat = HALF ? p.pl.hscat : p.pl.scat;
  const unsigned* __restrict__ gath = HALF ? p.pl.hgath : p.pl.gath;
  unsigned* reps[3];
  reps[0] = AL ? reinterpret_cast<unsigned*>(buf + 2 * B * LP)
               : reinterpret_cast<unsigned*>(stage + B * n);
  reps[1] = reps[0] + PfaStageC<SH, 0>::Rcnt;
  reps[2] = reps[1] + (SH::d >= 2 ? PfaStageC<SH, 1>::Rcnt : 0);
  for (int s = 0; s < SH::d; ++s) {
    const int rc = s == 0 ? PfaStageC<SH, 0>::Rcnt
                          : (s == 1 ? PfaStageC<SH, 1>::Rcnt : PfaStageC<SH, 2>::Rcnt);
    for (int i = tid; i < rc; i += nth) reps[s][i] = p.pl.reps[s][i];
  }
  if constexpr (HALF && HO && !AL) {  // out-of-place stages: the second buffer's pads read as zero
    for (int i = tid; i < B * LP; i += nth) buf2[i] = make_double2(0.0, 0.0);
  }
  if constexpr (AL) {
    // aliased staging: the pads are re-zeroed after every pack (below); the tail of the
    // second buffer that no staging row covers starts out zero as well
    for (int i = tid + (int)((long)B * n / 2); i < B * LP; i += nth) buf2[i] = make_double2(0.0, 0.0);
  }
  // CSM: the q0 stage's cos / sin tables staged in shared memory (after the reps, 8-aligned)
  double* csm = nullptr;
  if constexpr (CSM) {
    using HC = HalfCoef<HalfShape<Q1, Q2>>;
    csm = reinterpret_cast<double*>(smraw) +
          (((reinterpret_cast<unsigned char*>(reps[2] + 64) - smraw) + 7) / 8);
    for (int i = tid; i < HC::n0; i += nth) {
      csm[i] = p.pl.st[0].Cf[i];
      csm[HC::n0 + i] = p.pl.st[0].Sf[i];
    }
  }
  // Batches: F full rounds in which CTA c takes lines (j G + c) B .. +B (concurrent CTAs
  // work on adjacent lines: their transposed column stores share sectors), then one
  // balanced round that spreads the remaining rem < B G lines evenly (at most B per CTA,
  // sizes differ by one), so the tail is not a partial wave of full batches.
  const int G = gridDim.x, c = blockIdx.x;
  const int F = p.nlines / (B * G), rem = p.nlines - F * B * G;
  const int tl0 = F * B * G + (int)((long)c * rem / G);
  const int tl1 = F * B * G + (int)((long)(c + 1) * rem / G);
  const int nb_cta = F + (tl1 > tl0 ? 1 : 0);
  auto first_of = [&](int j) { return j < F ? (j * G + c) * B : tl0; };
  auto rows_of = [&](int j) { return j < F ? B : tl1 - tl0; };
  // blocked input: every thread copies 16-byte pairs with cp.async (the staging row of line
  // t gets pair (2 b, 2 b + 1) from block b), completion by wait_group + the pack barrier
  auto issue_blocked = [&](int j) {
    const int first = first_of(j), rows = rows_of(j);
    const int nh = n >> 1;
    // one thread per block: the batch's lines are adjacent 16-byte pairs of one sector
    for (int b = tid; b < nh; b += nth) {
      const double* src = p.in + ((long)b * n + first) * 2;
      for (int l = 0; l < rows; ++l) {
        const unsigned dst = (unsigned)__cvta_generic_to_shared(stage + l * n + 2 * b);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(src + 2 * l));
      }
    }
    asm volatile("cp.async.commit_group;\n" ::);
    if (tid == 0) {
      for (int l = 0; l < rows; ++l) {
        const long r = (long)(first + l) * n;
        if (p.pre) bulk_prefetch_l2(p.pre + r, (unsigned)(n * 8));
        if (has_mid) bulk_prefetch_l2(p.mid + r, (unsigned)(n * 8));
        if (!trans) {
          if (p.post) bulk_prefetch_l2(p.post + r, (unsigned)(n * 8));
          if (p.dot_with) bulk_prefetch_l2(p.dot_with + r, (unsigned)(n * 8));
        }
      }
    }
  };
  auto issue = [&](int j) {
    const int first = first_of(j), rows = rows_of(j);
    mbar_expect_tx(&mbar, (unsigned)(rows * n * 8));
    for (int l = 0; l < rows; ++l) {
      const long r = (long)(first + l) * n;
      if (p.in_seg) {  // one bulk copy per all-to-all block of the row
        const long base = (long)(first + l) * p.in_seg;
        for (int s0 = 0; s0 < n; s0 += p.in_seg)
          bulk_g2s(stage + l * n + s0, p.in + (s0 / p.in_seg) * p.in_seg_stride + base,
                   (unsigned)(p.in_seg * 8), &mbar);
      } else {
        bulk_g2s(stage + l * n, p.in + r, (unsigned)(n * 8), &mbar);
      }
      // the row streams read with plain loads later in this batch: pull them into L2 now
      if (p.pre) bulk_prefetch_l2(p.pre + r, (unsigned)(n * 8));
      if (has_mid) bulk_prefetch_l2(p.mid + r, (unsigned)(n * 8));
      if (!trans) {
        if (p.post) bulk_prefetch_l2(p.post + r, (unsigned)(n * 8));
        if (p.dot_with) bulk_prefetch_l2(p.dot_with + r, (unsigned)(n * 8));
      }
    }
  };
  if (tid == 0) {
    mbar_init(&mbar, 1);
    if (!BIN && nb_cta > 0) issue(0);
  }
  if (BIN && nb_cta > 0) issue_blocked(0);
  __syncthreads();
  // y_k from the transformed line l, gather index gi = gath[k - 1] (0 for k out of range)
  auto unpack = [&](int l, unsigned gi, int k) {
    double2 C;
    if constexpr (HALF) {
      C = res[l * LP + (gi & 0x7fffu)];
      if (gi & 0x8000u) C = make_double2(-C.x, -C.y);
    } else {
      C = res[l * LP + gi];
    }
    return ((k & 1) ? -(C.y + C.x) : -(C.y - C.x)) * p.scale;
  };
  // rank-2 border correction of the AR transform at interior t: b0 q_L[t] + b1 q_R[t]
  auto arcorr = [&](double b0, double b1, int t) {
    return __dadd_rn(__dmul_rn(b0, __ldg(p.ar_ql + t - 1)), __dmul_rn(b1, __ldg(p.ar_qr + t - 1)));
  };
  // z_t -> its packed position(s) (t parity selects re / im)
  auto scatter = [&](double* bl, int t, unsigned e, double x) {
    double* b = bl + (t & 1);
    if constexpr (HALF) {
      b[2 * (e & 0x7fffu)] = (e & 0x8000u) ? -x : x;
      if (e >> 31) b[2 * ((e >> 16) & 0x7fffu)] = -x;
    } else {
      b[2 * (e & 0xffffu)] = x;
      b[2 * (e >> 16)] = -x;
    }
  };
  const long nl_out = p.nlines;
  auto oidx = [&](int line, int e) {
    if (BOUT) return ((long)(line >> 1) * n + e) * 2 + (line & 1);
    return trans ? (long)e * nl_out + line : (long)line * n + e;
  };
  double acc = 0.0;
  unsigned phase = 0;
  PIPE_T_INIT;
  for (int jb = 0; jb < nb_cta; ++jb) {
    const int line0 = first_of(jb), nlv = rows_of(jb);
    for (int i = tid; i < B; i += nth) {
      buf[i * LP] = make_double2(0.0, 0.0);
      if constexpr (HALF)  // pad read by padded r
        buf[i * LP + HalfShape<Q1, Q2 == 1 ? 3 : Q2>::PADI] = make_double2(0.0, 0.0);
    }
    for (int i = tid; i < (B - nlv) * LP; i += nth) buf[nlv * LP + i] = make_double2(0.0, 0.0);
    // pack from the staging rows (+ Shat borders parked in smem): thread owns
    // t = 1 + tid + k nth.  The scatter indices depend on t only: one batched load
    // serves every line of the batch and overlaps the wait for the TMA rows.
    unsigned e[kTpt];
#pragma unroll
    for (int k = 0; k < kTpt; ++k) {
      const int t = 1 + tid + k * NT;
      e[k] = (k < kTpt - 1 || t <= N) ? __ldg(scat + t - 1) : 0u;
    }
    if constexpr (BIN) {
      asm volatile("cp.async.wait_group 0;\n" ::: "memory");
      __syncthreads();
    } else {
      mbar_wait(&mbar, phase);
      phase ^= 1u;
    }
    PIPE_T(0);
    for (int l = 0; l < nlv; ++l) {
      const double* srow = stage + l * n + p.off - 1;  // srow[t] = x_t
      double x[kTpt];
#pragma unroll
      for (int k = 0; k < kTpt; ++k) {
        const int t = 1 + tid + k * NT;
        x[k] = (k < kTpt - 1 || t <= N) ? srow[t] : 0.0;
      }
      if (p.pre) {
        const double* __restrict__ prow = p.pre + (long)(line0 + l) * n + p.off - 1;
        double q[kTpt];
#pragma unroll
        for (int k = 0; k < kTpt; ++k) {
          const int t = 1 + tid + k * NT;
          q[k] = (k < kTpt - 1 || t <= N) ? prow[t] : 1.0;
        }
#pragma unroll
        for (int k = 0; k < kTpt; ++k) x[k] = p.pre_mul ? x[k] * q[k] : x[k] / q[k];
      }
      if (p.ar_mode & 1) {  // T: x_int += x_0 q_L + x_last q_R (borders after the pre-scaling)
        double b0 = stage[l * n], b1 = stage[l * n + n - 1];
        if (p.pre) {
          const double q0 = p.pre[(long)(line0 + l) * n], q1 = p.pre[(long)(line0 + l) * n + n - 1];
          b0 = p.pre_mul ? b0 * q0 : b0 / q0;
          b1 = p.pre_mul ? b1 * q1 : b1 / q1;
        }
#pragma unroll
        for (int k = 0; k < kTpt; ++k) {
          const int t = 1 + tid + k * NT;
          if (k < kTpt - 1 || t <= N) x[k] = __dadd_rn(x[k], arcorr(b0, b1, t));
        }
      }
      double* bl = reinterpret_cast<double*>(buf + l * LP);
#pragma unroll
      for (int k = 0; k < kTpt; ++k) {
        const int t = 1 + tid + k * NT;
        if (k < kTpt - 1 || t <= N) scatter(bl, t, e[k], x[k]);
      }
    }
    if (p.off && tid < 2 * nlv) {
      const int l = tid >> 1, e = (tid & 1) ? n - 1 : 0;
      double x = stage[l * n + e];
      if (p.pre) {
        const double q = p.pre[(long)(line0 + l) * n + e];
        x = p.pre_mul ? x * q : x / q;
      }
      bord[l][tid & 1] = x;
    }
    __syncthreads();
    PIPE_T(1);
    auto issue_next = [&]() {
      if (BIN) {
        if (jb + 1 < nb_cta) issue_blocked(jb + 1);
      } else if (tid == 0 && jb + 1 < nb_cta) {
        fence_proxy_async();  // staging was read / written through the generic proxy
        issue(jb + 1);
      }
    };
    if constexpr (AL) {
      // the rows just packed lay over the second buffer's line-end pads: zero them again
      // (stage 0's closing barrier orders this before stage 1's padded reads)
      {
        using HS = HalfShape<Q1, Q2>;
        constexpr int PADS = HS::P1h - HS::H1 - 1;  // pad columns per grid row
        if (tid < B) buf2[tid * LP + HS::PADI] = make_double2(0.0, 0.0);
        if constexpr (PADS > 0) {
          for (int i = tid; i < B * HS::Q0 * PADS; i += nth) {
            const int l = i / (HS::Q0 * PADS), rem = i - l * (HS::Q0 * PADS);
            const int a = rem / PADS, c = rem - a * PADS;
            buf2[l * LP + a * HS::P1h + HS::H1 + 1 + c] = make_double2(0.0, 0.0);
          }
        }
      }
    } else {
      issue_next();
    }
    if constexpr (HALF) {
      half_transform<Q1, Q2, B, NT / 32, TPW, CSM, HO, CO>(buf, p.pl, p.stages, csm, buf2);
      res = buf;
    } else {
      res = pfa_transform_nl<Q1, Q2, Q3, B, NT, TPW>(buf, buf2, reps, p.pl, p.stages);
    }
    PIPE_T(2);
    unsigned g[kTpt];  // gather indices of this thread's t values
#pragma unroll
    for (int k = 0; k < kTpt; ++k) {
      const int t = 1 + tid + k * NT;
      g[k] = (k < kTpt - 1 || t <= N) ? __ldg(gath + t - 1) : 0u;
    }
    if (has_mid) {
      double v[B][kTpt];
#pragma unroll
      for (int l = 0; l < B; ++l) {
        const double* __restrict__ mrow = p.mid + (long)(line0 + min(l, nlv - 1)) * n + p.off - 1;
#pragma unroll
        for (int k = 0; k < kTpt; ++k) {
          const int t = 1 + tid + k * NT;
          v[l][k] = (l < nlv && t <= N) ? mrow[t] : 0.0;
        }
      }
#pragma unroll
      for (int l = 0; l < B; ++l)
#pragma unroll
        for (int k = 0; k < kTpt; ++k) {
          const int t = 1 + tid + k * NT;
          if (l < nlv && t <= N) {
            double y = unpack(l, g[k], t);
            if (p.ar_mode & 2) y = __dsub_rn(y, arcorr(bord[l][0], bord[l][1], t));  // T^-1
            v[l][k] *= y;
          }
        }
      if (p.ar_mode & 4) {  // T before the second transform, borders scaled by mid
#pragma unroll
        for (int l = 0; l < B; ++l) {
          if (l < nlv) {
            const long rb = (long)(line0 + l) * n;
            const double b0 = bord[l][0] * p.mid[rb], b1 = bord[l][1] * p.mid[rb + n - 1];
#pragma unroll
            for (int k = 0; k < kTpt; ++k) {
              const int t = 1 + tid + k * NT;
              if (t <= N) v[l][k] = __dadd_rn(v[l][k], arcorr(b0, b1, t));
            }
          }
        }
      }
      __syncthreads();
#pragma unroll
      for (int l = 0; l < B; ++l) {
        double* bl = reinterpret_cast<double*>(buf + l * LP);
#pragma unroll
        for (int k = 0; k < kTpt; ++k) {
          const int t = 1 + tid + k * NT;
          if (l < nlv && t <= N) scatter(bl, t, e[k], v[l][k]);
        }
      }
      for (int i = tid; i < B; i += nth) buf[i * LP] = make_double2(0.0, 0.0);
      __syncthreads();
      if constexpr (HALF) {
        half_transform<Q1, Q2, B, NT / 32, TPW, CSM, HO, CO>(buf, p.pl, p.stages, csm, buf2);
        res = buf;
      } else {
        res = pfa_transform_nl<Q1, Q2, Q3, B, NT, TPW>(buf, buf2, reps, p.pl, p.stages);
      }
    }
    if constexpr (AL) issue_next();  // every stage is done with the second buffer
    PIPE_T(3);
    // unpack + store (transposed: line index fastest -> B-double column segments).
    // All global loads of a group are issued before its stores.
    if (trans) {
      const int l = tid & (B - 1);
      constexpr int TS = NT / B;
      constexpr int JT = (N + TS - 1) / TS;
      constexpr int JG = 8;
      if (l < nlv) {
        // ocol[t * ostr] = y_t: column segments (stride nl) or the pair-blocked layout (2)
        const long ostr = BOUT ? 2 : nl_out;
        const long cb = BOUT ? oidx(line0 + l, p.off - 1) : (long)(p.off - 1) * nl_out + line0 + l;
        double* __restrict__ ocol = p.out + cb;
        const double* __restrict__ dcol = p.dot_with ? p.dot_with + cb : nullptr;
        const double* __restrict__ qcol = p.post ? p.post + cb : nullptr;
        const int t0 = 1 + tid / B;
#pragma unroll
        for (int j0 = 0; j0 < JT; j0 += JG) {
          unsigned gg[JG];
          double y[JG];
#pragma unroll
          for (int j = 0; j < JG; ++j) {
            const int t = t0 + (j0 + j) * TS;
            gg[j] = (j0 + j < JT && t <= N) ? __ldg(gath + t - 1) : 0u;
          }
#pragma unroll
          for (int j = 0; j < JG; ++j) y[j] = unpack(l, gg[j], t0 + (j0 + j) * TS);
          if ((p.ar_mode & 2) && !has_mid) {  // T^-1 of the (only) transform
#pragma unroll
            for (int j = 0; j < JG; ++j) {
              const int t = t0 + (j0 + j) * TS;
              if (j0 + j < JT && t <= N) y[j] = __dsub_rn(y[j], arcorr(bord[l][0], bord[l][1], t));
            }
          }
          if (qcol) {
            double q[JG];
#pragma unroll
            for (int j = 0; j < JG; ++j) {
              const int t = t0 + (j0 + j) * TS;
              q[j] = (j0 + j < JT && t <= N) ? qcol[(long)t * ostr] : 1.0;
            }
#pragma unroll
            for (int j = 0; j < JG; ++j) y[j] = p.post_mul ? y[j] * q[j] : y[j] / q[j];
          }
          double dv[JG];
#pragma unroll
          for (int j = 0; j < JG; ++j) {
            const int t = t0 + (j0 + j) * TS;
            dv[j] = (dcol && j0 + j < JT && t <= N) ? dcol[(long)t * ostr] : 0.0;
          }
#pragma unroll
          for (int j = 0; j < JG; ++j) {
            const int t = t0 + (j0 + j) * TS;
            if (j0 + j < JT && t <= N) {
              ocol[(long)t * ostr] = y[j];
              acc += y[j] * dv[j];
            }
          }
        }
      }
    } else {
      for (int l = 0; l < nlv; ++l) {
        const long rowb = (long)(line0 + l) * n + p.off - 1;
        double* __restrict__ orow = p.out + rowb;
        const double* __restrict__ drow = p.dot_with ? p.dot_with + rowb : nullptr;
        const double* __restrict__ qrow = p.post ? p.post + rowb : nullptr;
        double y[kTpt];
#pragma unroll
        for (int k = 0; k < kTpt; ++k) y[k] = unpack(l, g[k], 1 + tid + k * NT);
        if ((p.ar_mode & 2) && !has_mid) {  // T^-1 of the (only) transform
#pragma unroll
          for (int k = 0; k < kTpt; ++k) {
            const int t = 1 + tid + k * NT;
            if (k < kTpt - 1 || t <= N) y[k] = __dsub_rn(y[k], arcorr(bord[l][0], bord[l][1], t));
          }
        }
        if (qrow) {
          double q[kTpt];
#pragma unroll
          for (int k = 0; k < kTpt; ++k) {
            const int t = 1 + tid + k * NT;
            q[k] = (k < kTpt - 1 || t <= N) ? qrow[t] : 1.0;
          }
#pragma unroll
          for (int k = 0; k < kTpt; ++k) y[k] = p.post_mul ? y[k] * q[k] : y[k] / q[k];
        }
        double dv[kTpt];
#pragma unroll
        for (int k = 0; k < kTpt; ++k) {
          const int t = 1 + tid + k * NT;
          dv[k] = (drow && (k < kTpt - 1 || t <= N)) ? drow[t] : 0.0;
        }
#pragma unroll
        for (int k = 0; k < kTpt; ++k) {
          const int t = 1 + tid + k * NT;
          if (k < kTpt - 1 || t <= N) {
            orow[t] = y[k];
            acc += y[k] * dv[k];
          }
        }
      }
    }
    if (p.off && tid < 2 * nlv) {
      const int l = tid >> 1, e = (tid & 1) ? n - 1 : 0;
      double y = bord[l][tid & 1];
      if (has_mid) y *= p.mid[(long)(line0 + l) * n + e];
      const long g = oidx(line0 + l, e);
      if (p.post) y = p.post_mul ? y * p.post[g] : y / p.post[g];
      p.out[g] = y;
      if (p.dot_with) acc += y * p.dot_with[g];
    }
    __syncthreads();
    PIPE_T(4);
  }
  PIPE_T_FLUSH;
  if (p.partial) {
    const double s = block_sum(acc, red);
    if (tid == 0) p.partial[blockIdx.x] = s;
    if (p.fin.s) pcg_fin_tail(p.fin, p.partial, gridDim.x, red);
  }
}

template <int Q1, int Q2, int Q3, int NT = 256, int MINB = 2, int TPW = 3, bool HALF = false,
          int BL = kPipeLines, bool CSM = false, int PM = -1, bool HO = false, int CO = 0>
static cudaError_t launch_pipe_t(const PipeK& k, int grid, cudaStream_t st) {
  using SH = PfaShape<Q1, Q2, Q3>;
  int reps = PfaStageC<SH, 0>::Rcnt;
  if (SH::d >= 2) reps += PfaStageC<SH, 1>::Rcnt;
  if (SH::d >= 3) reps += PfaStageC<SH, 2>::Rcnt;
  constexpr int LP = HALF ? HalfShape<Q1, Q2 == 1 ? 3 : Q2>::LPh : SH::LP;
  constexpr bool AL = HALF && HO && kPipeAliasStage;
  if (AL && (size_t)k.n * 8 > (size_t)LP * 16) return cudaErrorInvalidConfiguration;
  size_t smem = (size_t)((kPipeOOP && !HALF) || (HALF && HO) ? 2 : 1) * BL * LP * 16 +
                (AL ? 0 : (size_t)BL * k.n * 8) + (reps + 64) * sizeof(unsigned);
  if (CSM) smem = (smem + 7) / 8 * 8 + (size_t)HalfCoef<HalfShape<Q1, Q2 == 1 ? 3 : Q2>>::total * 8;
  if (smem > 220 * 1024) return cudaErrorInvalidConfiguration;
  if (HALF && !k.pl.hscat) return cudaErrorInvalidConfiguration;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_dst_pipe<Q1, Q2, Q3, NT, MINB, TPW, HALF, BL, CSM, PM, HO, CO>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    attr = true;
  }
  return launch_pdl(k_dst_pipe<Q1, Q2, Q3, NT, MINB, TPW, HALF, BL, CSM, PM, HO, CO>, grid, NT, smem,
                    st, k);
}

// the four pass-specialised instances of one launch shape
// pass modes: bit 0 sandwich, bit 1 transposed output, bit 2 pair-blocked output (with bit 1),
// bit 3 pair-blocked input.  The single-GPU M^-1 runs 6 -> 15 -> 8 (row pass into the blocked
// layout, sandwich blocked to blocked, row pass out of it); the row-slab passes 0..3.
template <int Q1, int Q2, int Q3, int NT, int MINB, int TPW, bool HALF, bool HO = false,
          int BL = kPipeLines, int CO = 0, bool CSM = false>
static cudaError_t launch_pipe_pm(const PipeK& k, int grid, cudaStream_t st) {
  const int pm = (k.mid ? 1 : 0) | (k.transposed ? 2 : 0) | (k.transposed == 2 ? 4 : 0) |
                 (k.in_blocked ? 8 : 0);
  switch (pm) {
    case 0: return launch_pipe_t<Q1, Q2, Q3, NT, MINB, TPW, HALF, BL, CSM, 0, HO, CO>(k, grid, st);
    case 1: return launch_pipe_t<Q1, Q2, Q3, NT, MINB, TPW, HALF, BL, CSM, 1, HO, CO>(k, grid, st);
    case 2: return launch_pipe_t<Q1, Q2, Q3, NT, MINB, TPW, HALF, BL, CSM, 2, HO, CO>(k, grid, st);
    case 3: return launch_pipe_t<Q1, Q2, Q3, NT, MINB, TPW, HALF, BL, CSM, 3, HO, CO>(k, grid, st);
    case 6: return launch_pipe_t<Q1, Q2, Q3, NT, MINB, TPW, HALF, BL, CSM, 6, HO, CO>(k, grid, st);
    case 8: return launch_pipe_t<Q1, Q2, Q3, NT, MINB, TPW, HALF, BL, CSM, 8, HO, CO>(k, grid, st);
    case 15: return launch_pipe_t<Q1, Q2, Q3, NT, MINB, TPW, HALF, BL, CSM, 15, HO, CO>(k, grid, st);
    default: return cudaErrorInvalidConfiguration;
  }
}

// Launch shape per specialisation (tools/pipe_variants.py swept these in round 1):
// * 2047 = 89 * 23 (config 3): half-line layout, stages out of place over a second line
//   buffer, two 6-warp CTAs per SM (the two CTAs overlap one batch's pack / unpack with the
//   other's DFT stages), column-owner tensor-core stages (tvd_pfa_t.cuh half_stage_co):
//   243.3 us per M^-1 vs 263.9 with k-tile-owner stages (bit-identical), 272.1 in place, 291
//   for one 12-warp CTA; one line per batch measured slower, and so did three CTAs per SM
//   once the staging rows aliased the second line buffer (69 KB per CTA): 3 x 6 warps at 96
//   registers 222 us, 3 x 4 warps at 168 registers 224 us vs 206 us for 2 x 6 warps; the
//   q = 89 fragment tables copied to shared memory (CSM) 209 vs 206 us through L1;
// * 1023 = 33 * 31 (config 4; the plan merges 11 . 3 into one tensor-core stage): the same
//   half-line, out-of-place, column-owner path as 2047 with four 4-warp CTAs per SM
//   (round 1 / early round 2: three in-place stages 31 . 11 . 3, four 2-warp CTAs, 86 us
//   per M^-1);
// * 511 = 73 * 7 (config 2a): half-line layout, two 6-warp CTAs (38.3 vs 40.4 us per M^-1);
// * 127 (config 1): two 8-warp CTAs.
// A warp-specialised producer / consumer variant of the 2047 pass measured 272-288 us per
// M^-1 against 275 us lock step (bit-identical) and was removed.
struct PipeVariant {
  int threads, ctas, tpw, lines;
};
static PipeVariant pipe_variant(int which) {
  switch (which) {
    case 1: return {192, 2, 1, 2};
    case 2: return {128, 4, 1, 2};
    case 3: return {192, 2, 1, 2};
    default: return {256, 2, 3, 2};
  }
}

int pipe_grid(const PfaPlan& P, int nlines) {
  int which;
  if (!pfa_specialised(P, &which)) return -1;
  const int bl = pipe_variant(which).lines;
  const int nbatch = (nlines + bl - 1) / bl;
  const int cap = kSMs * pipe_variant(which).ctas;
  return nbatch < cap ? nbatch : cap;
}

cudaError_t launch_pipe(const PfaPlan& P, int family, int len, int nlines, int transposed,
                        const LineIO& io, int* nblocks_out, cudaStream_t st) {
  int which;
  if (!pfa_specialised(P, &which) || (len & 1)) return cudaErrorInvalidConfiguration;
  PipeK k{};
  k.pl = P;
  k.n = len;
  k.off = family == kFamSineHat ? 1 : 0;
  k.nlines = nlines;
  k.transposed = transposed;
  k.scale = 0.5 * sqrt(2.0 / P.L);
  k.in = io.in;
  k.out = io.out;
  k.pre = io.pre;
  k.pre_mul = io.pre_mul;
  k.mid = io.mid_mul;
  k.post = io.post;
  k.post_mul = io.post_mul;
  k.dot_with = io.dot_with;
  k.partial = io.partial;
  k.skip = io.skip;
  k.fin = io.fin;
  k.ar_mode = io.ar_mode;
  k.ar_ql = io.ar_ql;
  k.ar_qr = io.ar_qr;
  if (io.in_seg && (io.in_seg % 2 || len % io.in_seg)) return cudaErrorInvalidValue;
  if (io.in_blocked && (io.in_seg || (len & 1) || nlines != len)) return cudaErrorInvalidValue;
  k.in_seg = io.in_seg;
  k.in_seg_stride = io.in_seg_stride;
  k.in_blocked = io.in_blocked;
  k.stages = option(kOptPfaStages);  // profiling: run only the first stages
  const int grid = pipe_grid(P, nlines);
  if (nblocks_out) *nblocks_out = grid;
  if (grid <= 0) return cudaSuccess;
  switch (which) {
    case 1: return launch_pipe_pm<89, 23, 1, 192, 2, 1, true, true, 2, 2>(k, grid, st);
    case 2: return launch_pipe_pm<33, 31, 1, 128, 4, 1, true, true, 2, 2>(k, grid, st);
    case 3: return launch_pipe_pm<73, 7, 1, 192, 2, 1, true>(k, grid, st);
    case 4: return launch_pipe_pm<127, 1, 1, 256, 2, 3, false>(k, grid, st);
    default: return cudaErrorInvalidConfiguration;
  }
}

template <int Q1, int Q2, int Q3>
static cudaError_t launch_pfa_t(const PfaK& k, int nb, cudaStream_t st) {
  using SH = PfaShape<Q1, Q2, Q3>;
  int reps = PfaStageC<SH, 0>::Rcnt;
  if (SH::d >= 2) reps += PfaStageC<SH, 1>::Rcnt;
  if (SH::d >= 3) reps += PfaStageC<SH, 2>::Rcnt;
  const size_t smem = (size_t)kPfaLinesT * SH::LP * 16 + (2 * SH::N + reps) * sizeof(unsigned);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_pfa_t<Q1, Q2, Q3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         200 * 1024);
    attr = true;
  }
  k_pfa_t<Q1, Q2, Q3><<<nb, 256, smem, st>>>(k);
  return cudaGetLastError();
}

// specialisations: the config lengths L = n - 1 of the Shat family (n = 128, 512, 1024, 2048)
static bool pfa_specialised(const PfaPlan& P, int* which) {
  auto is = [&](int a, int b, int c) {
    return P.q[0] == a && (P.d >= 2 ? P.q[1] : 1) == b && (P.d >= 3 ? P.q[2] : 1) == c;
  };
  *which = is(89, 23, 1) ? 1 : is(33, 31, 1) ? 2 : is(73, 7, 1) ? 3 : is(127, 1, 1) ? 4 : 0;
  return *which != 0 && P.scat != nullptr;
}

static int pfa_config(const PfaPlan& P, bool contiguous, int* nl, int* nth, size_t* smem) {
  const size_t line_bytes = (size_t)P.LP * 16;
  int k = 2;
  (void)contiguous;
  while (k > 1 && k * line_bytes > 150 * 1024) k >>= 1;
  if (line_bytes * k > 200 * 1024) return -1;
  const int t = 256;
  // the sandwich re-pack holds kPfaMaxV values per thread
  if ((P.L - 1) > kPfaMaxV * t) return -1;
  *nl = k;
  *nth = t;
  *smem = k * line_bytes;
  return 0;
}

int pfa_blocks(const PfaPlan& P, const LineGeom& g) {
  int nl, nth, which;
  size_t smem;
  if (pfa_specialised(P, &which)) return (g.nlines + kPfaLinesT - 1) / kPfaLinesT;
  if (pfa_config(P, g.es == 1, &nl, &nth, &smem)) return -1;
  return (g.nlines + nl - 1) / nl;
}

bool band_pfa_ok(const PfaPlan& P) {
  int which;
  return pfa_specialised(P, &which) && P.gscat != nullptr && P.greps[0] != nullptr;
}

bool band_pfa_rowwise(const PfaPlan& P) {
  int which;
  return band_pfa_ok(P) && pfa_specialised(P, &which) && (which == 1 || which == 2);
}

cudaError_t launch_band_pfa(const PfaPlan& P, const double2* wfull, int n, const BandLines& b,
                            int* nblocks_out, cudaStream_t st) {
  int which;
  if (!band_pfa_ok(P)) return cudaErrorInvalidConfiguration;
  pfa_specialised(P, &which);
  BandPfaK k{};
  k.pl = P;
  k.wfull = wfull;
  k.n = n;
  k.b = b;
  if (which == 1 || which == 2) {  // column-owner variant (two tensor-core stages)
    if (nblocks_out) *nblocks_out = b.nlines;
    if (b.nlines == 0) return cudaSuccess;
    return which == 1 ? launch_band_pfa_co<89, 23, 6>(k, st) : launch_band_pfa_co<33, 31, 4>(k, st);
  }
  const int nb = (b.nlines + kBandPfaLines - 1) / kBandPfaLines;
  if (nblocks_out) *nblocks_out = nb;
  if (nb == 0) return cudaSuccess;
  switch (which) {
    case 1: return launch_band_pfa_t<89, 23, 1>(k, nb, st);
    case 2: return launch_band_pfa_t<33, 31, 1>(k, nb, st);
    case 3: return launch_band_pfa_t<73, 7, 1>(k, nb, st);
    case 4: return launch_band_pfa_t<127, 1, 1>(k, nb, st);
    default: return cudaErrorInvalidConfiguration;
  }
}

cudaError_t launch_pfa(const PfaPlan& P, int family, int len, const LineGeom& g, const LineIO& io,
                       int* nblocks_out, cudaStream_t st) {
  int nl, nth, which = 0;
  size_t smem;
  const bool spec = pfa_specialised(P, &which);
  if (spec) {
    nl = kPfaLinesT;
  } else if (pfa_config(P, g.es == 1, &nl, &nth, &smem)) {
    return cudaErrorInvalidConfiguration;
  }
  PfaK k{};
  k.pl = P;
  k.n = len;
  k.off = family == kFamSineHat ? 1 : 0;
  k.N = P.L - 1;
  k.nl = nl;
  k.nlines = g.nlines;
  k.ls = g.ls;
  k.es = g.es;
  k.scale = 0.5 * sqrt(2.0 / P.L);
  k.h = (P.L - 1) / 2;
  k.stages = option(kOptPfaStages);  // profiling: run only the first stages
  k.io = io;
  const int nb = (g.nlines + nl - 1) / nl;
  if (nblocks_out) *nblocks_out = nb;
  if (nb == 0) return cudaSuccess;
  switch (which) {
    case 1: return launch_pfa_t<89, 23, 1>(k, nb, st);
    case 2: return launch_pfa_t<33, 31, 1>(k, nb, st);
    case 3: return launch_pfa_t<73, 7, 1>(k, nb, st);
    case 4: return launch_pfa_t<127, 1, 1>(k, nb, st);
    default: break;
  }
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_pfa, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  k_pfa<<<nb, nth, smem, st>>>(k);
  return cudaGetLastError();
}

}  // namespace tvd

// profiling only: per-phase cycle sums of the pipeline kernel (-DTVD_PIPE_TIMING builds)
extern "C" int tvd_debug_stage_times(unsigned long long* out128, int reset) {
#ifdef TVD_PIPE_TIMING
  if (out128 && cudaMemcpyFromSymbol(out128, tvd::g_stage_t, 128 * sizeof(unsigned long long)) !=
                    cudaSuccess)
    return -1;
  if (reset) {
    unsigned long long z[128] = {};
    cudaMemcpyToSymbol(tvd::g_stage_t, z, sizeof(z));
  }
  return 0;
#else
  (void)out128;
  (void)reset;
  return -1;
#endif
}

extern "C" int tvd_debug_pipe_phases(unsigned long long* out8, int reset) {
#ifdef TVD_PIPE_TIMING
  if (out8 && cudaMemcpyFromSymbol(out8, tvd::g_pipe_phase, 8 * sizeof(unsigned long long)) != cudaSuccess)
    return -1;
  if (reset) {
    unsigned long long z[8] = {};
    cudaMemcpyToSymbol(tvd::g_pipe_phase, z, sizeof(z));
  }
  return 0;
#else
  (void)out8;
  (void)reset;
  return -1;
#endif
}
