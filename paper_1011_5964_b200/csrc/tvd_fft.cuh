// Shared-memory mixed-radix complex FFT for batches of lines (fp64).
//
// The DST-I / DCT passes of the preconditioner and the band-form projections
// of the preconditioner assembly all reduce to one complex FFT of length L per
// line (L = n-1 for the bordered sine family, L = n for the cosine family).
// The configs hit odd, prime-factor lengths (127, 511 = 7*73, 1023 = 3*11*31,
// 2047 = 23*89), so the engine is a Stockham autosort FFT with
//   * register codelets for radices 2,3,4,5,7,8 (twiddled inputs), and
//   * a shared-memory "pair" stage for every odd radix R >= 9: inputs are
//     folded into a_r = x_r + x_{R-r}, b_r = x_r - x_{R-r} in place, then each
//     work item accumulates KB output pairs (k, R-k) from real cos/sin
//     coefficients -- (R-1)^2/R real FMAs per point instead of R.
// Every stage is in place: a work item holds its outputs in registers across a
// __syncthreads(); lines are processed in rounds so that at most kFftSlots
// items per thread are live.  The host (tvd_plan.cpp) guarantees that one
// line's items fit in kFftSlots * blockDim.x.
#pragma once

#include "tvd_common.cuh"

namespace tvd {

constexpr int kFftMaxStages = 10;
constexpr int kFftKB = 4;     // output pairs per work item in odd stages
constexpr int kFftSlots = 2;  // register slots per thread per stage

enum : int { kStageReg = 0, kStageOdd = 1 };

struct FftStage {
  int radix;
  int kind;
  int ns;    // product of the radices of the previous stages
  int coef;  // odd stages: offset of (cos, sin)(2 pi t / R), t in [0, R)
};

struct FftPlan {
  int L;
  int nst;
  FftStage st[kFftMaxStages];
  const double2* tw;    // L entries exp(-2 pi i e / L)
  const double2* coef;  // odd-radix coefficient tables
};

// ---------------------------------------------------------------- codelets
template <int R>
__device__ __forceinline__ double2 odd_cs(int t);  // (cos, sin)(2 pi t / R)

template <>
__device__ __forceinline__ double2 odd_cs<3>(int t) {
  switch (t) {
    case 1: return make_double2(-0.5, 0.8660254037844386);
    case 2: return make_double2(-0.5, -0.8660254037844386);
    default: return make_double2(1.0, 0.0);
  }
}
template <>
__device__ __forceinline__ double2 odd_cs<5>(int t) {
  switch (t) {
    case 1: return make_double2(0.30901699437494745, 0.9510565162951535);
    case 2: return make_double2(-0.8090169943749475, 0.5877852522924731);
    case 3: return make_double2(-0.8090169943749475, -0.5877852522924731);
    case 4: return make_double2(0.30901699437494745, -0.9510565162951535);
    default: return make_double2(1.0, 0.0);
  }
}
template <>
__device__ __forceinline__ double2 odd_cs<7>(int t) {
  switch (t) {
    case 1: return make_double2(0.6234898018587336, 0.7818314824680298);
    case 2: return make_double2(-0.22252093395631434, 0.9749279121818236);
    case 3: return make_double2(-0.9009688679024191, 0.43388373911755823);
    case 4: return make_double2(-0.9009688679024191, -0.43388373911755823);
    case 5: return make_double2(-0.22252093395631434, -0.9749279121818236);
    case 6: return make_double2(0.6234898018587336, -0.7818314824680298);
    default: return make_double2(1.0, 0.0);
  }
}

template <>
__device__ __forceinline__ double2 odd_cs<13>(int t) {
  switch (t) {
    case 1: return make_double2(0.8854560256532099, 0.4647231720437685);
    case 2: return make_double2(0.5680647467311559, 0.8229838658936564);
    case 3: return make_double2(0.120536680255323, 0.992708874098054);
    case 4: return make_double2(-0.35460488704253545, 0.9350162426854148);
    case 5: return make_double2(-0.7485107481711012, 0.6631226582407952);
    case 6: return make_double2(-0.970941817426052, 0.23931566428755768);
    case 7: return make_double2(-0.9709418174260521, -0.23931566428755743);
    case 8: return make_double2(-0.7485107481711013, -0.663122658240795);
    case 9: return make_double2(-0.3546048870425359, -0.9350162426854147);
    case 10: return make_double2(0.1205366802553232, -0.992708874098054);
    case 11: return make_double2(0.5680647467311548, -0.822983865893657);
    case 12: return make_double2(0.88545602565321, -0.4647231720437684);
    default: return make_double2(1.0, 0.0);
  }
}

// Forward DFT (exp(-2 pi i jk / R)) of an odd-length register vector.
template <int R>
__device__ __forceinline__ void dft_odd_reg(double2 (&v)[R]) {
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
      const double2 w = odd_cs<R>((r * k) % R);
      A.x += a[r].x * w.x; A.y += a[r].y * w.x;
      B.x += b[r].x * w.y; B.y += b[r].y * w.y;
    }
    v[k] = make_double2(x0.x + A.x + B.y, x0.y + A.y - B.x);
    v[R - k] = make_double2(x0.x + A.x - B.y, x0.y + A.y + B.x);
  }
  v[0] = s0;
}

__device__ __forceinline__ void dft2(double2& a, double2& b) {
  const double2 t = a;
  a = cadd(t, b);
  b = csub(t, b);
}

// multiply by -i
__device__ __forceinline__ double2 mul_mi(double2 a) { return make_double2(a.y, -a.x); }

template <int R>
__device__ __forceinline__ void dft_reg(double2 (&v)[R]);

template <>
__device__ __forceinline__ void dft_reg<2>(double2 (&v)[2]) { dft2(v[0], v[1]); }

template <>
__device__ __forceinline__ void dft_reg<4>(double2 (&v)[4]) {
  dft2(v[0], v[2]);
  dft2(v[1], v[3]);
  v[3] = mul_mi(v[3]);
  dft2(v[0], v[1]);
  dft2(v[2], v[3]);
  // now v = X0, X2, X1, X3
  const double2 t = v[1];
  v[1] = v[2];
  v[2] = t;
}

template <>
__device__ __forceinline__ void dft_reg<8>(double2 (&v)[8]) {
  constexpr double c = 0.70710678118654752440;
  double2 e[4] = {v[0], v[2], v[4], v[6]};
  double2 o[4] = {v[1], v[3], v[5], v[7]};
  dft_reg<4>(e);
  dft_reg<4>(o);
  // twiddles W8^k, k = 0..3: 1, (c,-c), -i, (-c,-c)
  o[1] = make_double2(c * (o[1].x + o[1].y), c * (o[1].y - o[1].x));
  o[2] = mul_mi(o[2]);
  o[3] = make_double2(c * (o[3].y - o[3].x), -c * (o[3].x + o[3].y));
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    v[k] = cadd(e[k], o[k]);
    v[k + 4] = csub(e[k], o[k]);
  }
}

template <>
__device__ __forceinline__ void dft_reg<3>(double2 (&v)[3]) { dft_odd_reg<3>(v); }
template <>
__device__ __forceinline__ void dft_reg<5>(double2 (&v)[5]) { dft_odd_reg<5>(v); }
template <>
__device__ __forceinline__ void dft_reg<7>(double2 (&v)[7]) { dft_odd_reg<7>(v); }
template <>
__device__ __forceinline__ void dft_reg<13>(double2 (&v)[13]) { dft_odd_reg<13>(v); }

// ------------------------------------------------------------------ stages
// Line l occupies buf[l * LP, l * LP + L).
template <int R>
__device__ __forceinline__ void stage_reg(double2* buf, int LP, int nl, int L, int ns,
                                          const double2* __restrict__ tw) {
  const int tid = threadIdx.x, nth = blockDim.x;
  const int nb = L / R;
  const int tstride = L / (ns * R);
  int lpr = (kFftSlots * nth) / nb;
  if (lpr < 1) lpr = 1;
  for (int l0 = 0; l0 < nl; l0 += lpr) {
    const int items = min(lpr, nl - l0) * nb;
    double2 v[kFftSlots][R];
#pragma unroll
    for (int s = 0; s < kFftSlots; ++s) {
      const int i = tid + s * nth;
      if (i < items) {
        const int line = l0 + i / nb, j = i % nb, jm = j % ns;
        const double2* base = buf + line * LP;
        // one twiddle load per butterfly, the powers w^(r e0) by recurrence (~R ulp)
        const double2 w1 = ns > 1 ? __ldg(&tw[jm * tstride]) : make_double2(1.0, 0.0);
        double2 wr = w1;
#pragma unroll
        for (int r = 0; r < R; ++r) {
          double2 x = base[j + r * nb];
          if (r > 0 && ns > 1) {
            x = cmul(x, wr);
            if (r + 1 < R) wr = cmul(wr, w1);
          }
          v[s][r] = x;
        }
        dft_reg<R>(v[s]);
      }
    }
    __syncthreads();
#pragma unroll
    for (int s = 0; s < kFftSlots; ++s) {
      const int i = tid + s * nth;
      if (i < items) {
        const int line = l0 + i / nb, j = i % nb, jm = j % ns;
        double2* base = buf + line * LP;
        const int d = (j / ns) * ns * R + jm;
#pragma unroll
        for (int r = 0; r < R; ++r) base[d + r * ns] = v[s][r];
      }
    }
    __syncthreads();
  }
}

__device__ __forceinline__ void stage_odd(double2* buf, int LP, int nl, int L, int R, int ns,
                                          const double2* __restrict__ tw,
                                          const double2* __restrict__ cs) {
  const int tid = threadIdx.x, nth = blockDim.x;
  const int nb = L / R, H = (R - 1) / 2;
  const int tstride = L / (ns * R);
  // fold: twiddle, then (a_r, b_r) in place of (x_r, x_{R-r})
  const int nfold = nb * H;
  for (int i = tid; i < nl * nfold; i += nth) {
    const int line = i / nfold, rem = i - line * nfold;
    const int r = 1 + rem / nb, j = rem % nb;
    double2* base = buf + line * LP;
    double2 x1 = base[j + r * nb], x2 = base[j + (R - r) * nb];
    if (ns > 1) {
      const int jm = j % ns;
      x1 = cmul(x1, __ldg(&tw[r * jm * tstride]));
      x2 = cmul(x2, __ldg(&tw[(R - r) * jm * tstride]));
    }
    base[j + r * nb] = cadd(x1, x2);
    base[j + (R - r) * nb] = csub(x1, x2);
  }
  __syncthreads();
  const int nch = (H + kFftKB - 1) / kFftKB;
  const int ipl = nb * nch;
  int lpr = (kFftSlots * nth) / ipl;
  if (lpr < 1) lpr = 1;
  for (int l0 = 0; l0 < nl; l0 += lpr) {
    const int items = min(lpr, nl - l0) * ipl;
    double2 ok[kFftSlots][kFftKB], om[kFftSlots][kFftKB], o0[kFftSlots];
#pragma unroll
    for (int s = 0; s < kFftSlots; ++s) {
      const int i = tid + s * nth;
      if (i < items) {
        const int line = l0 + i / ipl, rem = i % ipl;
        const int c = rem / nb, j = rem % nb;
        const double2* base = buf + line * LP;
        const double2 x0 = base[j];
        double2 A[kFftKB], B[kFftKB];
        int t[kFftKB];
        const int k0 = 1 + c * kFftKB;
#pragma unroll
        for (int q = 0; q < kFftKB; ++q) {
          A[q] = make_double2(0.0, 0.0);
          B[q] = make_double2(0.0, 0.0);
          t[q] = 0;
        }
        double2 s0 = x0;
        for (int r = 1; r <= H; ++r) {
          const double2 a = base[j + r * nb], b = base[j + (R - r) * nb];
          s0 = cadd(s0, a);
#pragma unroll
          for (int q = 0; q < kFftKB; ++q) {
            t[q] += k0 + q;
            if (t[q] >= R) t[q] -= R;
            const double2 w = __ldg(&cs[t[q]]);
            A[q].x += a.x * w.x; A[q].y += a.y * w.x;
            B[q].x += b.x * w.y; B[q].y += b.y * w.y;
          }
        }
#pragma unroll
        for (int q = 0; q < kFftKB; ++q) {
          ok[s][q] = make_double2(x0.x + A[q].x + B[q].y, x0.y + A[q].y - B[q].x);
          om[s][q] = make_double2(x0.x + A[q].x - B[q].y, x0.y + A[q].y + B[q].x);
        }
        o0[s] = s0;
      }
    }
    __syncthreads();
#pragma unroll
    for (int s = 0; s < kFftSlots; ++s) {
      const int i = tid + s * nth;
      if (i < items) {
        const int line = l0 + i / ipl, rem = i % ipl;
        const int c = rem / nb, j = rem % nb, jm = j % ns;
        double2* base = buf + line * LP;
        const int d = (j / ns) * ns * R + jm;
        if (c == 0) base[d] = o0[s];
        const int k0 = 1 + c * kFftKB;
#pragma unroll
        for (int q = 0; q < kFftKB; ++q) {
          const int k = k0 + q;
          if (k <= H) {
            base[d + k * ns] = ok[s][q];
            base[d + (R - k) * ns] = om[s][q];
          }
        }
      }
    }
    __syncthreads();
  }
}

// Forward FFT of nl lines in place (natural order in and out).  Caller must
// __syncthreads() before (data written) -- the stages sync internally and at
// exit.
__device__ __forceinline__ void fft_lines(double2* buf, int LP, int nl, const FftPlan& P) {
  for (int s = 0; s < P.nst; ++s) {
    const FftStage st = P.st[s];
    if (st.kind == kStageOdd) {
      stage_odd(buf, LP, nl, P.L, st.radix, st.ns, P.tw, P.coef + st.coef);
    } else {
      switch (st.radix) {
        case 2: stage_reg<2>(buf, LP, nl, P.L, st.ns, P.tw); break;
        case 3: stage_reg<3>(buf, LP, nl, P.L, st.ns, P.tw); break;
        case 4: stage_reg<4>(buf, LP, nl, P.L, st.ns, P.tw); break;
        case 5: stage_reg<5>(buf, LP, nl, P.L, st.ns, P.tw); break;
        case 7: stage_reg<7>(buf, LP, nl, P.L, st.ns, P.tw); break;
        case 8: stage_reg<8>(buf, LP, nl, P.L, st.ns, P.tw); break;
        default: __trap();
      }
    }
  }
}

}  // namespace tvd
