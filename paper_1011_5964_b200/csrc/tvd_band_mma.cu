// Banded 1D operator passes on the fp64 tensor cores (mma.sync m8n8k4 f64, SASS DMMA.884).
//
//   row pass     out[i][j] = sum_c B[j][c] in[i][c]        (GEMM  in * B^T)
//   column pass  out[i][j] = sum_r B[i][r] in[r][j] (+ fused normal-equation epilogue)
//
// B is the banded operator of tvd_stencil.h (half-width w, Toeplitz with symmetric taps in
// the interior, border rows from the table).  A warp owns T = 8 output tiles of 8 x 8 that
// are consecutive along the band direction.  For tile t and k-step s (4 input positions,
// starting KOFF = roundup(w, 4) before the tile) the operator fragment of a lane is
// B[o][o + d] with d = 4s - KOFF + (lane & 3) - (lane >> 2): it does not depend on the tile
// in the Toeplitz interior, so the CTA stages it once in shared memory, and the data
// fragment of (t, s) is data fragment 2t + s, so a warp issues 8 S DMMAs from
// S + 2 (T - 1) data-fragment loads (S = 2 + KOFF / 2).  Tiles that touch the first or
// last op.B outputs read their operator fragments from the border table.
//
// Reference semantics: H^T H p = G p G^T with G = H1^T H1 (src/pipeline.py:209-210,
// src/blur.py:197-326); the epilogue is tv.py:96-108 (L w) and pipeline.py:129-164 (s).
#include <cstdlib>

#include "tvd_stencil.h"

namespace tvd {
namespace {

constexpr int kBmT = 8;  // output tiles per warp along the band direction

__device__ __forceinline__ void bmma(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}
__device__ __forceinline__ void cp16(void* dst, const void* src, bool ok) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(src),
               "r"(ok ? 16 : 0));
}
__device__ __forceinline__ void cp_commit_wait() {
  asm volatile("cp.async.commit_group;\n" ::);
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
}

__device__ __forceinline__ void prefetch_l2(const double* p) {
  if (p) asm volatile("prefetch.global.L2 [%0];\n" ::"l"(p));
}
__device__ __forceinline__ void prefetch_l1(const double* p) {
  if (p) asm volatile("prefetch.global.L1 [%0];\n" ::"l"(p));
}

struct BandTaps {
  double t[64];  // t[k] = symmetric interior tap at offset +-k
};

__device__ __forceinline__ double coef_interior(const BandTaps& tp, int w, int d) {
  const int a = d < 0 ? -d : d;
  return a <= w ? tp.t[a] : 0.0;
}
// operator fragment of border tile p (host-built, tvd_capi.cu make_bandop)
__device__ __forceinline__ const double* border_frag(const BandOp& op, int p, int S) {
  const int np = (op.n + 7) / 8;
  const int idx = p < op.frag_l ? p : (p >= op.frag_r0 && p < np ? op.frag_l + p - op.frag_r0
                                                                  : op.frag_cnt);
  return op.frag + (size_t)idx * S * 32;
}

template <int KOFF, int TC = kBmT>
struct BmShape {
  static constexpr int S = 2 + KOFF / 2;  // k-steps per tile
  // row pass: 2 row blocks x 4 column strips of 8 T outputs
  static constexpr int RH = 16, CW = 32 * kBmT, WIDTH = CW + 2 * KOFF;
  static constexpr int RP = WIDTH + ((4 - WIDTH % 16) + 16) % 16;  // pitch = 4 (mod 16)
  // column pass: 4 row strips of 8 T outputs x 2 column tiles
  static constexpr int RW = 4 * 8 * TC, CC = 16, HEIGHT = RW + 2 * KOFF;  // TC tiles per warp
  static constexpr int CP = 24;  // pitch = 8 (mod 16): 4 rows x 8 columns in 2 wavefronts
  static size_t rows_smem() { return (size_t)(RH * RP + S * 32) * sizeof(double); }
  static size_t cols_smem() { return (size_t)(HEIGHT * CP + S * 32) * sizeof(double); }
};

template <int KOFF>
__device__ __forceinline__ void stage_fragments(double* fr, const BandTaps& tp, int w) {
  constexpr int S = BmShape<KOFF>::S;
  for (int e = threadIdx.x; e < S * 32; e += blockDim.x) {
    const int s = e >> 5, l = e & 31;
    fr[e] = coef_interior(tp, w, 4 * s - KOFF + (l & 3) - (l >> 2));
  }
}

// Fused CG direction update (PCG iterations >= 2): the pass reads z and the previous
// direction p_old, forms p = z + beta p_old (numpy rounding, k_pcg_update_p) for its tile
// including the halo columns, stores its interior columns to p_new (a different buffer:
// neighbouring CTAs still read p_old halos) and multiplies the formed tile -- the separate
// p-update pass and one read of p disappear.
struct PFuse {
  const double* z;     // nullptr: plain pass over `in`
  double* p_new;
  const PcgState* st;  // beta
};

template <int KOFF>
__global__ void __launch_bounds__(256, 2) k_bmma_rows(BandOp op, BandTaps tp,
                                                     const double* __restrict__ in,
                                                     double* __restrict__ out, const int* skip,
                                                     int row_lo, int row_hi, PFuse fz) {
  pdl_enter();
  if (skip && *skip) return;
  using SH = BmShape<KOFF>;
  constexpr int T = kBmT, S = SH::S, RP = SH::RP, W2 = SH::WIDTH / 2;
  const unsigned long long keep = l2_keep_policy();
  extern __shared__ __align__(16) double smb[];
  double* tile = smb;
  double* fr = smb + SH::RH * RP;
  double* tile2 = fr + S * 32;  // fused: p_old tile (tile holds z)
  const int n = op.n, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int i0 = row_lo + blockIdx.y * SH::RH, jb = blockIdx.x * SH::CW;
  const double* src = fz.z ? fz.z : in;
  for (int e = tid; e < SH::RH * W2; e += blockDim.x) {
    const int r = e / W2, c = 2 * (e - r * W2);
    const int row = i0 + r, col = jb - KOFF + c;
    const bool ok = row < row_hi && col >= 0 && col < n;
    cp16(tile + r * RP + c, ok ? src + (long)row * n + col : src + (long)i0 * n, ok);
    if (fz.z) cp16(tile2 + r * RP + c, ok ? in + (long)row * n + col : in + (long)i0 * n, ok);
  }
  stage_fragments<KOFF>(fr, tp, op.w);
  cp_commit_wait();
  __syncthreads();
  if (fz.z) {
    const double beta = fz.st->beta;
    for (int e = tid; e < SH::RH * W2; e += blockDim.x) {
      const int r = e / W2, c = 2 * (e - r * W2);
      const int row = i0 + r, col = jb - KOFF + c;
      double2* tz = reinterpret_cast<double2*>(tile + r * RP + c);
      const double2 po = *reinterpret_cast<const double2*>(tile2 + r * RP + c);
      const double2 zz = *tz;
      const double2 pv = make_double2(__dadd_rn(zz.x, __dmul_rn(beta, po.x)),
                                      __dadd_rn(zz.y, __dmul_rn(beta, po.y)));
      *tz = pv;  // zero-filled out-of-range elements stay zero
      if (row < row_hi && col >= jb && col < jb + SH::CW && col < n)
        st2_keep(fz.p_new + (long)row * n + col, pv.x, pv.y, keep);
    }
    __syncthreads();
  }
  const int rb = warp >> 2, cs = warp & 3;
  const int o0 = jb + cs * 8 * T;  // first output column of the warp
  const double* arow = tile + (rb * 8 + (lane >> 2)) * RP + cs * 8 * T + (lane & 3);
  double acc[T][2];
#pragma unroll
  for (int t = 0; t < T; ++t) acc[t][0] = acc[t][1] = 0.0;
  const int p0 = o0 >> 3;  // first 8-output tile of the warp
  if (p0 >= op.frag_l && p0 + T <= op.frag_r0) {
#pragma unroll
    for (int s = 0; s < S; ++s) {
      const double b = fr[s * 32 + lane];
#pragma unroll
      for (int t = 0; t < T; ++t) bmma(acc[t][0], acc[t][1], arow[4 * (2 * t + s)], b);
    }
  } else {
#pragma unroll
    for (int t = 0; t < T; ++t) {
      const int p = p0 + t;
      const double* bf = (p < op.frag_l || p >= op.frag_r0) ? border_frag(op, p, S) + lane
                                                            : fr + lane;
#pragma unroll
      for (int s = 0; s < S; ++s) bmma(acc[t][0], acc[t][1], arow[4 * (2 * t + s)], bf[s * 32]);
    }
  }
  const int row = i0 + rb * 8 + (lane >> 2);
  if (row < row_hi) {
#pragma unroll
    for (int t = 0; t < T; ++t) {
      const int col = o0 + 8 * t + 2 * (lane & 3);
      if (col < n)
        st2_keep(out + (long)row * n + col, acc[t][0], acc[t][1], keep);
    }
  }
}

template <int KOFF, int TC, int MINB>
__global__ void __launch_bounds__(256, MINB) k_bmma_cols(BandOp op, BandTaps tp,
                                                     const double* __restrict__ in,
                                                     double* __restrict__ out, Epilogue ep,
                                                     const int* skip, int row_lo, int row_hi) {
  pdl_enter();
  if (skip && *skip) return;
  using SH = BmShape<KOFF, TC>;
  constexpr int T = TC, S = SH::S, CP = SH::CP, C2 = SH::CC / 2;
  extern __shared__ __align__(16) double smb[];
  __shared__ double red[32];
  double* tile = smb;
  double* fr = smb + SH::HEIGHT * CP;
  const int n = op.n, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int ib = row_lo + blockIdx.y * SH::RW, j0 = blockIdx.x * SH::CC;
  // The epilogue's operands (a_h, a_v, lw and the extra streams) are read long after the
  // tile: option band_prefetch pulls their lines into L2 (1) or L1 (2) before the tile load.
  if (ep.prefetch) {
    auto pf = [&](const double* q) {
      if (ep.prefetch == 2) prefetch_l1(q);
      else prefetch_l2(q);
    };
    for (int i = tid; i < SH::RW + 2; i += blockDim.x) {
      const int row = ib - 1 + i;
      if (row < 0 || row >= n || row > row_hi) continue;
      const int c0 = j0 > 0 ? j0 - 1 : 0;
      pf(ep.lw ? ep.lw + (long)row * n + c0 : nullptr);
      pf(ep.lw ? ep.lw + (long)row * n + j0 : nullptr);
      pf(ep.lw ? ep.lw + (long)row * n + min(j0 + SH::CC, n - 1) : nullptr);
      if (row >= ib && row < row_hi) {
        pf(ep.a_h ? ep.a_h + (long)row * (n + 1) + j0 : nullptr);
        pf(ep.a_h ? ep.a_h + (long)row * (n + 1) + j0 + SH::CC : nullptr);
        pf(ep.a_v ? ep.a_v + (long)row * n + j0 : nullptr);
        pf(ep.a_v ? ep.a_v + (long)row * n + j0 + SH::CC - 1 : nullptr);
        if (ep.s) pf(ep.s + (long)row * n + j0);
        if (ep.dot_with && ep.dot_with != ep.lw) pf(ep.dot_with + (long)row * n + j0);
      }
      if (row == row_hi && ep.a_v) pf(ep.a_v + (long)row * n + j0);
    }
  }
  for (int e = tid; e < SH::HEIGHT * C2; e += blockDim.x) {
    const int r = e / C2, c = 2 * (e - r * C2);
    const int row = ib - KOFF + r, col = j0 + c;
    // rows outside [row_lo - KOFF, row_hi + KOFF) feed only outputs past row_hi, which are
    // dropped -- and a row slab's buffer ends there (a 128-row tile over a 64-row slab would
    // read past its halo): zero-fill them instead of reading
    const bool ok = row >= 0 && row < n && col < n && row >= row_lo - KOFF && row < row_hi + KOFF;
    cp16(tile + r * CP + c, ok ? in + (long)row * n + col : in + (long)ib * n, ok);
  }
  stage_fragments<KOFF>(fr, tp, op.w);
  cp_commit_wait();
  __syncthreads();
  const int rs = warp >> 1, ct = warp & 1;
  const int o0 = ib + rs * 8 * T;  // first output row of the warp
  const double* bcol = tile + (rs * 8 * T + (lane & 3)) * CP + ct * 8 + (lane >> 2);
  double acc[T][2];
#pragma unroll
  for (int t = 0; t < T; ++t) acc[t][0] = acc[t][1] = 0.0;
  const int p0 = o0 >> 3;  // first 8-output tile of the warp
  if (p0 >= op.frag_l && p0 + T <= op.frag_r0) {
#pragma unroll
    for (int s = 0; s < S; ++s) {
      const double a = fr[s * 32 + lane];
#pragma unroll
      for (int t = 0; t < T; ++t) bmma(acc[t][0], acc[t][1], a, bcol[4 * (2 * t + s) * CP]);
    }
  } else {
#pragma unroll
    for (int t = 0; t < T; ++t) {
      const int p = p0 + t;
      const double* af = (p < op.frag_l || p >= op.frag_r0) ? border_frag(op, p, S) + lane
                                                            : fr + lane;
#pragma unroll
      for (int s = 0; s < S; ++s) bmma(acc[t][0], acc[t][1], af[s * 32], bcol[4 * (2 * t + s) * CP]);
    }
  }
  // epilogue: q = [s *] (acc + alpha L(lw)), dot += dot_with . q (tv.py:96-108, pipeline.py:129-164).
  // Each lane owns the column pair (col, col + 1) of its T row tiles.  The zero-Neumann ghosts
  // are clamped indices rather than branches, so all operands of a group of TG tiles are in
  // flight before the first is used; per element the arithmetic is diffusion_at's, unfused.
  const double* __restrict__ a_h = ep.a_h;
  const double* __restrict__ a_v = ep.a_v;
  const double* __restrict__ lw = ep.lw;
  const double* __restrict__ sv = ep.s;
  const double* __restrict__ dw = ep.dot_with;
  const int col = j0 + ct * 8 + 2 * (lane & 3);
  const int cl = col > 0 ? col - 1 : 0, cr = col + 2 < n ? col + 2 : n - 1;
  auto ld2 = [](const double* p) { return __ldg(reinterpret_cast<const double2*>(p)); };
  constexpr int TG = 2;
  const unsigned long long keep_policy = l2_keep_policy();
  const bool ar = ep.bc_l == 1;  // anti-reflective ghosts 2 w_0 - w_1 at the image border
  double dot = 0.0, dself = 0.0;
  if (col < n) {
#pragma unroll
    for (int t0 = 0; t0 < T; t0 += TG) {
      double2 wc[TG], wu[TG], wd[TG], vu[TG], vd[TG], s2[TG], d2[TG];
      double wl[TG], wr[TG], h0[TG], h1[TG], h2[TG];
#pragma unroll
      for (int k = 0; k < TG; ++k) {
        const int i = min(o0 + 8 * (t0 + k) + (lane >> 2), row_hi - 1);
        const int iu = i > 0 ? i - 1 : 0, id = i < n - 1 ? i + 1 : n - 1;
        const long r = (long)i * n;
        if (a_h) {
          wc[k] = ld2(lw + r + col);
          wl[k] = __ldg(lw + r + cl);
          wr[k] = __ldg(lw + r + cr);
          wu[k] = ld2(lw + (long)iu * n + col);
          wd[k] = ld2(lw + (long)id * n + col);
          const long hb = (long)i * (n + 1) + col;
          h0[k] = __ldg(a_h + hb);
          h1[k] = __ldg(a_h + hb + 1);
          h2[k] = __ldg(a_h + hb + 2);
          vu[k] = ld2(a_v + r + col);
          vd[k] = ld2(a_v + r + n + col);
        }
        if (sv) s2[k] = ld2(sv + r + col);
        if (dw) d2[k] = ld2(dw + r + col);
      }
#pragma unroll
      for (int k = 0; k < TG; ++k) {
        const int i = o0 + 8 * (t0 + k) + (lane >> 2);
        if (i >= row_hi) continue;
        double x0 = acc[t0 + k][0], x1 = acc[t0 + k][1];
        if (a_h) {
          if (ar) {  // replace the clamped (zero-Neumann) ghosts by odd reflections
            if (col == 0) wl[k] = ar_ghost(wc[k].x, wc[k].y);
            if (col + 2 >= n) wr[k] = ar_ghost(wc[k].y, wc[k].x);
            if (i == 0) wu[k] = make_double2(ar_ghost(wc[k].x, wd[k].x), ar_ghost(wc[k].y, wd[k].y));
            if (i == n - 1) wd[k] = make_double2(ar_ghost(wc[k].x, wu[k].x), ar_ghost(wc[k].y, wu[k].y));
          }
          const double fl0 = __dmul_rn(h0[k], __dsub_rn(wc[k].x, wl[k]));
          const double fr0 = __dmul_rn(h1[k], __dsub_rn(wc[k].y, wc[k].x));
          const double fu0 = __dmul_rn(vu[k].x, __dsub_rn(wc[k].x, wu[k].x));
          const double fd0 = __dmul_rn(vd[k].x, __dsub_rn(wd[k].x, wc[k].x));
          const double fl1 = fr0;  // same edge: a_h[h0 + 1] * (w[col + 1] - w[col])
          const double fr1 = __dmul_rn(h2[k], __dsub_rn(wr[k], wc[k].y));
          const double fu1 = __dmul_rn(vu[k].y, __dsub_rn(wc[k].y, wu[k].y));
          const double fd1 = __dmul_rn(vd[k].y, __dsub_rn(wd[k].y, wc[k].y));
          const double l0 = __dmul_rn(-ep.inv_h2, __dadd_rn(__dsub_rn(fr0, fl0), __dsub_rn(fd0, fu0)));
          const double l1 = __dmul_rn(-ep.inv_h2, __dadd_rn(__dsub_rn(fr1, fl1), __dsub_rn(fd1, fu1)));
          x0 = __dadd_rn(x0, __dmul_rn(ep.alpha, l0));
          x1 = __dadd_rn(x1, __dmul_rn(ep.alpha, l1));
        }
        if (sv) {
          x0 = __dmul_rn(s2[k].x, x0);
          x1 = __dmul_rn(s2[k].y, x1);
        }
        // q is read once more, by the x / r update right after this pass: ask L2 to keep it
        st2_keep(out + (long)i * n + col, x0, x1, keep_policy);
        if (dw) {
          dot += d2[k].x * x0;
          dot += d2[k].y * x1;
        }
        dself += x0 * x0;
        dself += x1 * x1;
      }
    }
  }
  if (ep.partial) {
    const double s = block_sum(dot, red);
    if (tid == 0) ep.partial[blockIdx.y * gridDim.x + blockIdx.x] = s;
    if (ep.fin.s) pcg_fin_tail(ep.fin, ep.partial, gridDim.x * gridDim.y, red);
  }
  if (ep.partial_self) {
    const double s = block_sum(dself, red);
    if (tid == 0) ep.partial_self[blockIdx.y * gridDim.x + blockIdx.x] = s;
  }
}

bool make_taps(const BandOp& op, BandTaps* tp) {
  if (!op.taps_host || op.w > 63) return false;
  for (int k = 0; k <= op.w; ++k) tp->t[k] = op.taps_host[op.w + k];
  return true;
}

int koff_of(int w) {
  const int k = (w + 3) / 4 * 4;
  switch (k) {
    case 4: case 8: case 12: case 16: case 20: case 24: case 28: case 32: return k;
    default: return w > 32 && w <= 64 ? 64 : 0;
  }
}

// TVD_OPT_BAND_SLIDE selects the CUDA-core sliding-window kernels (comparison runs)
bool band_mma_enabled() { return option(kOptBandSlide) == 0; }

#define TVD_KOFFS(X) X(4) X(8) X(12) X(16) X(20) X(24) X(28) X(32) X(64)

}  // namespace

// Tiles are 256 outputs long along the band direction, so small grids keep the CUDA-core
// kernels (whose summation order the small-n iteration-count goldens were pinned with).
constexpr int kBandMmaMinN = 256;

bool band_mma_ok(const BandOp& op) {
  return band_mma_enabled() && op.n >= kBandMmaMinN && (op.n % 2) == 0 && op.taps_host &&
         op.frag && koff_of(op.w) != 0;
}

int band_mma_koff(int w) { return koff_of(w); }

// column-pass shape: 4 row tiles per warp (128-row CTAs), two CTAs per SM (matvec 81.5 us vs
// 87.7 us for 8 tiles / 256-row CTAs at 2048^2; three CTAs spill; 2 tiles: 88-96 us)
constexpr int kColsTiles = 4;
static int cols_tiles() { return kColsTiles; }
int band_mma_cols_grid(int n, int rows) {
  if (rows < 0) rows = n;
  const int rw = 32 * cols_tiles();
  return ((n + 15) / 16) * ((rows + rw - 1) / rw);
}
int band_mma_row_tile() { return 32 * cols_tiles(); }

cudaError_t launch_band_mma_rows(const BandOp& op, const double* in, double* out, const int* skip,
                                 cudaStream_t st, int row_lo, int row_hi) {
  return launch_band_mma_rows_fused(op, in, out, skip, st, nullptr, nullptr, nullptr, row_lo,
                                    row_hi);
}

cudaError_t launch_band_mma_rows_fused(const BandOp& op, const double* in, double* out,
                                       const int* skip, cudaStream_t st, const double* z,
                                       double* p_new, const PcgState* pst, int row_lo,
                                       int row_hi) {
  const PFuse fz{z, p_new, pst};
  BandTaps tp;
  if (!make_taps(op, &tp)) return cudaErrorInvalidValue;
  const int n = op.n;
  if (row_hi < 0) row_hi = n;
  if (row_lo < 0 || row_lo > row_hi || row_hi > n) return cudaErrorInvalidValue;
  const int nr = row_hi - row_lo;
  if (nr == 0) return cudaSuccess;
  switch (koff_of(op.w)) {
#define X(K)                                                                                 \
  case K: {                                                                                  \
    using SH = BmShape<K>;                                                                   \
    static bool attr = false;                                                                \
    if (!attr) {                                                                             \
      cudaFuncSetAttribute(k_bmma_rows<K>, cudaFuncAttributeMaxDynamicSharedMemorySize,      \
                           (int)(SH::rows_smem() + SH::RH * SH::RP * sizeof(double)));       \
      attr = true;                                                                           \
    }                                                                                        \
    dim3 grid((n + SH::CW - 1) / SH::CW, (nr + SH::RH - 1) / SH::RH);                        \
    const size_t sm = SH::rows_smem() + (z ? SH::RH * SH::RP * sizeof(double) : 0);           \
    return launch_pdl(k_bmma_rows<K>, grid, 256, sm, st, op, tp, in, out, skip, row_lo, row_hi, \
                      fz);                                                                   \
  }
    TVD_KOFFS(X)
#undef X
    default: return cudaErrorInvalidValue;
  }
}

template <int K, int TC, int MINB>
static cudaError_t launch_cols_t(const BandOp& op, const BandTaps& tp, const double* in,
                                 double* out, const Epilogue& ep, const int* skip, cudaStream_t st,
                                 int row_lo, int row_hi) {
  using SH = BmShape<K, TC>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_bmma_cols<K, TC, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)SH::cols_smem());
    attr = true;
  }
  const int n = op.n, nr = row_hi - row_lo;
  dim3 grid((n + SH::CC - 1) / SH::CC, (nr + SH::RW - 1) / SH::RW);
  return launch_pdl(k_bmma_cols<K, TC, MINB>, grid, 256, SH::cols_smem(), st, op, tp, in, out, ep,
                    skip, row_lo, row_hi);
}

cudaError_t launch_band_mma_cols(const BandOp& op, const double* in, double* out,
                                 const Epilogue& ep_in, const int* skip, cudaStream_t st, int row_lo,
                                 int row_hi) {
  BandTaps tp;
  if (!make_taps(op, &tp)) return cudaErrorInvalidValue;
  const int n = op.n;
  Epilogue ep = ep_in;
  ep.prefetch = option(kOptBandPrefetch);  // 1: L2 (measured slower, 96 vs 88 us), 2: L1
  if (row_hi < 0) row_hi = n;
  if (row_lo < 0 || row_lo > row_hi || row_hi > n) return cudaErrorInvalidValue;
  const int nr = row_hi - row_lo;
  if (nr == 0) return cudaSuccess;
  switch (koff_of(op.w)) {
#define X(K) \
  case K: return launch_cols_t<K, kColsTiles, 2>(op, tp, in, out, ep, skip, st, row_lo, row_hi);
    TVD_KOFFS(X)
#undef X
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace tvd
