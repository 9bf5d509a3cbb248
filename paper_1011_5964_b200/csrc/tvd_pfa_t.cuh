// Compile-time specialised odd-symmetric PFA DST engine (included by tvd_pfa.cu).
//
// Same algorithm as the runtime kernel in tvd_pfa.cu, with the factorization
// L = Q1 * Q2 * Q3 a template parameter: every stride, representative count,
// modular map and loop bound is a constant, the small-DFT loops unroll, and
// the data-independent index permutations (pack scatter, unpack gather,
// representative line bases) come from tables staged in shared memory.
#pragma once

// (included inside namespace tvd, after dmma884 / kMmaTiles)

constexpr int c_modinv(int a, int m) {
  int r = 1;
  for (int x = 1; x < m; ++x)
    if ((a * x) % m == 1) r = x;
  return r;
}

template <int Q1, int Q2, int Q3>
struct PfaShape {
  static constexpr int L = Q1 * Q2 * Q3;
  static constexpr int d = (Q1 > 1) + (Q2 > 1) + (Q3 > 1);
  static constexpr int q[3] = {Q1, Q2, Q3};
  static constexpr int stride[3] = {d == 2 ? pfa_row_pitch(Q2) : Q2 * Q3, Q3, 1};
  static constexpr int LP = Q1 * stride[0];  // padded line size (tvd_internal.h)
  static constexpr int h = (L - 1) / 2;
  static constexpr int N = L - 1;
};

// Stage along dimension S of the shape.
template <class SH, int S>
struct PfaStageC {
  static constexpr int q = SH::q[S];
  static constexpr int H = (q - 1) / 2;
  static constexpr int st = SH::stride[S];
  // other dims in order; D1 = 1 when only one other dim
  static constexpr int o0 = S == 0 ? 1 : 0;
  static constexpr int o1 = S == 2 ? 1 : 2;
  static constexpr int D1 = SH::d == 3 ? SH::q[o0] : 1;
  static constexpr int S1 = SH::d == 3 ? SH::stride[o0] : 0;
  static constexpr int D2 = SH::d == 3 ? SH::q[o1] : (SH::d == 2 ? SH::q[o0] : 1);
  static constexpr int S2 = SH::d == 3 ? SH::stride[o1] : (SH::d == 2 ? SH::stride[o0] : 0);
  static constexpr int Rcnt = (D1 * D2 + 1) / 2;
  static constexpr int h2 = (D2 + 1) / 2;
  static constexpr int KP = (H + 1 + 7) / 8 * 8;
  static constexpr int RP = (H + 3) / 4 * 4;
  static constexpr bool mma = H >= 8;
  static constexpr int LPc = SH::LP;
  static constexpr bool gen = false;  // odd input: one DFT per {tau, -tau} pair
};

// The same stage for a general (not odd) complex input: every other-index tuple is its own
// DFT line (greps), outputs never mirrored to a negated partner.
template <class SH, int S>
struct PfaStageG : PfaStageC<SH, S> {
  static constexpr int Rcnt = PfaStageC<SH, S>::D1 * PfaStageC<SH, S>::D2;
  static constexpr bool gen = true;
};

template <class ST>
__device__ __forceinline__ void rep_ab(int t, int& a, int& b) {
  if (t < ST::h2) {
    a = 0;
    b = t;
  } else {
    const int u = t - ST::h2;
    a = 1 + u / ST::D2;
    b = u - (a - 1) * ST::D2;
  }
}

// fold + DFT of one stage.  `reps` holds (base | neg << 16) of every representative line
// (line 0); line l adds l * LP.  OOP: read `src`, write `dst` (a different buffer), so
// outputs go out as soon as they are formed and the stage needs a single closing barrier;
// otherwise src == dst and every round holds its outputs across an in-place barrier.
template <class ST, int NL, int MT = 4, int NW = 0, int TPWc = 3, bool OOP = false>
__device__ __forceinline__ void pfa_stage_c(const double2* src, double2* dst, const unsigned* reps,
                                            const double* Cm, const double* Sm,
                                            const double* __restrict__ Cf = nullptr,
                                            const double* __restrict__ Sf = nullptr) {
  double2* buf = dst;  // in-place paths (src == dst)
  constexpr int kMmaTiles = MT;  // output tiles a warp holds across the in-place barrier
  constexpr int q = ST::q, H = ST::H, st = ST::st, LP = ST::LPc;
  const int tid = threadIdx.x, nth = blockDim.x;
  constexpr int ndft = NL * ST::Rcnt;
  if constexpr (ST::mma && NW > 0) {
    // A-stationary tensor-core stage: warp -> fixed k-tile (its cos/sin fragments for every
    // r stay in registers) x TPW column tiles per round, sized so one round normally covers
    // every tile.  The fold a/b is fused into the B-fragment load (no fold sweep).  The
    // r-steps run outermost, so a warp keeps 2 TPW independent accumulator chains in flight
    // and issues each step's loads together; padded r (> H) and clamped columns read
    // in-range data against zero coefficients / dropped outputs, so nothing is predicated.
    constexpr int nkt = ST::KP / 8, nct = (2 * ndft + 7) / 8, nrs = ST::RP / 4;
    constexpr int G = NW / nkt >= 1 ? NW / nkt : 1;  // warps sharing one k-tile
    constexpr int TPWn = (nct + G - 1) / G;          // tiles per warp for a single round
    constexpr int TPW = TPWn < TPWc ? TPWn : TPWc;   // column tiles per warp per round
    constexpr int ROUND = G * TPW;
    const int lane = tid & 31, warp = tid >> 5;
    const int kt = warp % nkt, g = warp / nkt;
    const bool wact = warp < nkt * G;
    const int krow = kt * 8 + (lane >> 2);
    double ca[nrs], sa[nrs];
#pragma unroll
    for (int rs = 0; rs < nrs; ++rs) {  // fragment-ordered tables: coalesced 256-byte reads
      ca[rs] = __ldg(Cf + (kt * nrs + rs) * 32 + lane);
      sa[rs] = __ldg(Sf + (kt * nrs + rs) * 32 + lane);
    }
#ifdef TVD_PIPE_TIMING
    const long long ts_ = clock64();
#endif
    const double* bufd = reinterpret_cast<const double*>(src);
    for (int ct0 = 0; ct0 < nct; ct0 += ROUND) {
      double acc[TPW][4];
      const double* pb[TPW];
#pragma unroll
      for (int j = 0; j < TPW; ++j) {
        acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.0;
        const int ct = min(ct0 + g + j * G, nct - 1);
        const int dB = min((ct * 8 + (lane >> 2)) >> 1, ndft - 1);
        const int lB = dB / ST::Rcnt, tB = dB - lB * ST::Rcnt;
        pb[j] = bufd + 2 * (lB * LP + (reps[tB] & 0xffffu)) + ((lane >> 2) & 1);
      }
#ifdef TVD_PIPE_TIMING
      const long long tl0_ = clock64();
#endif
      if (wact) {
#pragma unroll
        for (int rs = 0; rs < nrs; ++rs) {
          const int r = 1 + rs * 4 + (lane & 3);
          double x1[TPW], x2[TPW];
#pragma unroll
          for (int j = 0; j < TPW; ++j) {
            x1[j] = pb[j][2 * r * st];
            x2[j] = pb[j][2 * (q - r) * st];
          }
#pragma unroll
          for (int j = 0; j < TPW; ++j) {
            dmma884(acc[j][0], acc[j][1], ca[rs], x1[j] + x2[j]);
            dmma884(acc[j][2], acc[j][3], sa[rs], x1[j] - x2[j]);
          }
        }
      }
#ifdef TVD_PIPE_TIMING
      long long tle_ = 0;
      {
        double z_ = 0.0;  // make the accumulators' completion part of the timed region
#pragma unroll
        for (int j = 0; j < TPW; ++j) z_ += acc[j][0] + acc[j][3];
        if (z_ == 12345.678) buf[0].x = z_;
        tle_ = clock64();
      }
#endif
      double2 vk[TPW], vm[TPW];
      unsigned ob[TPW];
      int oflag[TPW];
#pragma unroll
      for (int j = 0; j < TPW; ++j) {
        oflag[j] = 0;
        const int ct = ct0 + g + j * G;
        const int dO = ct * 4 + (lane & 3);
        if (wact && ct < nct && krow <= H && dO < ndft) {
          const int lO = dO / ST::Rcnt, tO = dO - lO * ST::Rcnt;
          const unsigned rp = reps[tO] + (unsigned)(lO * LP) * 0x10001u;
          const double2 x0 = src[rp & 0xffffu];
          const double a0 = acc[j][0], a1 = acc[j][1], b0 = acc[j][2], b1 = acc[j][3];
          vk[j] = make_double2(x0.x + a0 + b1, x0.y + a1 - b0);
          vm[j] = make_double2(x0.x + a0 - b1, x0.y + a1 + b0);
          ob[j] = rp;
          oflag[j] = 1 | ((ST::gen || tO == 0) ? 2 : 0);
        }
      }
      if constexpr (!OOP) __syncthreads();
#pragma unroll
      for (int j = 0; j < TPW; ++j) {
        if (oflag[j]) {
          const int k = krow;
          double2* p = buf + (ob[j] & 0xffffu);
          double2* pn = buf + (ob[j] >> 16);
          const bool self = oflag[j] & 2;
          if (k == 0) {
            p[0] = vk[j];
            if (!self) pn[0] = make_double2(-vk[j].x, -vk[j].y);
          } else {
            p[k * st] = vk[j];
            p[(q - k) * st] = vm[j];
            if (!self) {
              pn[(q - k) * st] = make_double2(-vk[j].x, -vk[j].y);
              pn[k * st] = make_double2(-vm[j].x, -vm[j].y);
            }
          }
        }
      }
      if constexpr (!OOP) __syncthreads();
#ifdef TVD_PIPE_TIMING
      if (OOP && lane == 0 && warp < 16) {
        const long long tep_ = clock64();
        unsigned long long* slot = g_stage_t + ((q == 89 ? 0 : 1) * 16 + warp) * 4;
        atomicAdd(slot + 0, (unsigned long long)(tl0_ - ts_));
        atomicAdd(slot + 1, (unsigned long long)(tle_ - tl0_));
        atomicAdd(slot + 2, (unsigned long long)(tep_ - tle_));
      }
#endif
    }
#ifdef TVD_PIPE_TIMING
    const long long tb0_ = clock64();
#endif
    if constexpr (OOP) __syncthreads();
#ifdef TVD_PIPE_TIMING
    if (OOP && lane == 0 && warp < 16)
      atomicAdd(g_stage_t + ((q == 89 ? 0 : 1) * 16 + warp) * 4 + 3,
                (unsigned long long)(clock64() - tb0_));
#endif
    return;
  }
  if constexpr (OOP && !(ST::mma && NW > 0)) {
    // small radix, out of place: one thread per representative DFT, fold in registers
    static_assert(!ST::mma, "out-of-place stages use the A-stationary tensor-core path");
    for (int d0 = 0; d0 < ndft; d0 += nth) {
      const int dft = d0 + tid;
      if (dft < ndft) {
        const int l = dft / ST::Rcnt, t = dft - l * ST::Rcnt;
        const unsigned rp = reps[t] + (unsigned)(l * LP) * 0x10001u;
        const bool self = ST::gen || t == 0;
        const double2* p = src + (rp & 0xffffu);
        const double2 x0 = p[0];
        double2 A[H + 1], Bv[H + 1];
#pragma unroll
        for (int r = 1; r <= H; ++r) {
          const double2 x1 = p[r * st], x2 = p[(q - r) * st];
          A[r] = cadd(x1, x2);
          Bv[r] = csub(x1, x2);
        }
        double2 v[q];
        double2 s0 = x0;
#pragma unroll
        for (int r = 1; r <= H; ++r) s0 = cadd(s0, A[r]);
        v[0] = s0;
#pragma unroll
        for (int k = 1; k <= H; ++k) {
          double2 a = make_double2(0.0, 0.0), b = make_double2(0.0, 0.0);
#pragma unroll
          for (int r = 1; r <= H; ++r) {
            const double c = Cm[k * ST::RP + r - 1], sn = Sm[k * ST::RP + r - 1];
            a.x += A[r].x * c; a.y += A[r].y * c;
            b.x += Bv[r].x * sn; b.y += Bv[r].y * sn;
          }
          v[k] = make_double2(x0.x + a.x + b.y, x0.y + a.y - b.x);
          v[q - k] = make_double2(x0.x + a.x - b.y, x0.y + a.y + b.x);
        }
        double2* o = dst + (rp & 0xffffu);
        double2* on = dst + (rp >> 16);
#pragma unroll
        for (int k = 0; k < q; ++k) {
          o[k * st] = v[k];
          if (!self) on[((q - k) % q) * st] = make_double2(-v[k].x, -v[k].y);
        }
      }
    }
    __syncthreads();
    return;
  }
  // fold (scalar and legacy tensor-core paths)
  constexpr int nfold = NL * ST::Rcnt * H;
  for (int i = tid; i < nfold; i += nth) {
    const int t = i % ST::Rcnt;
    const int rest = i / ST::Rcnt;
    const int line = rest / H;
    const int r = 1 + rest - line * H;
    double2* p = buf + line * LP + (reps[t] & 0xffffu);
    const double2 x1 = p[r * st], x2 = p[(q - r) * st];
    p[r * st] = cadd(x1, x2);
    p[(q - r) * st] = csub(x1, x2);
  }
  __syncthreads();
  if constexpr (ST::mma) {
    const int lane = tid & 31, warp = tid >> 5, nw = nth >> 5;
    constexpr int nkt = ST::KP / 8, nct = (2 * ndft + 7) / 8, nrs = ST::RP / 4;
    const int ctr = max(1, (nw * kMmaTiles) / nkt);
    const double* bufd = reinterpret_cast<const double*>(buf);
    for (int ct0 = 0; ct0 < nct; ct0 += ctr) {
      const int ntile = nkt * min(ctr, nct - ct0);
      double2 vk[kMmaTiles], vm[kMmaTiles];
      unsigned ob[kMmaTiles];
      int oflag[kMmaTiles];
#pragma unroll
      for (int s = 0; s < kMmaTiles; ++s) {
        oflag[s] = 0;
        const int tile = warp + s * nw;
        if (tile < ntile) {
          const int ct = ct0 + tile / nkt, kt = tile - (tile / nkt) * nkt;
          double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
          const int colB = ct * 8 + (lane >> 2);
          const int dB = colB >> 1;
          const bool vB = dB < ndft;
          const int lB = vB ? dB / ST::Rcnt : 0;
          const int tB = vB ? dB - lB * ST::Rcnt : 0;
          const double* pb = bufd + 2 * (lB * LP + (reps[tB] & 0xffffu)) + (colB & 1);
          const int krow = kt * 8 + (lane >> 2);
          const double* cm = Cm + krow * ST::RP + (lane & 3);
          const double* sm = Sm + krow * ST::RP + (lane & 3);
#pragma unroll
          for (int rs = 0; rs < nrs; ++rs) {
            const int r = 1 + rs * 4 + (lane & 3);
            double xa = 0.0, xb = 0.0;
            if (vB && (rs * 4 + 4 <= H || r <= H)) {
              xa = pb[2 * r * st];
              xb = pb[2 * (q - r) * st];
            }
            dmma884(a0, a1, cm[rs * 4], xa);
            dmma884(b0, b1, sm[rs * 4], xb);
          }
          const int dO = ct * 4 + (lane & 3);
          if (krow <= H && dO < ndft) {
            const int lO = dO / ST::Rcnt, tO = dO - lO * ST::Rcnt;
            const unsigned rp = reps[tO] + (unsigned)(lO * LP) * 0x10001u;
            const double2 x0 = buf[rp & 0xffffu];
            vk[s] = make_double2(x0.x + a0 + b1, x0.y + a1 - b0);
            vm[s] = make_double2(x0.x + a0 - b1, x0.y + a1 + b0);
            ob[s] = rp;
            oflag[s] = 1 | ((ST::gen || tO == 0) ? 2 : 0);
          }
        }
      }
      __syncthreads();
#pragma unroll
      for (int s = 0; s < kMmaTiles; ++s) {
        if (oflag[s]) {
          const int tile = warp + s * nw;
          const int k = (tile - (tile / nkt) * nkt) * 8 + (lane >> 2);
          double2* p = buf + (ob[s] & 0xffffu);
          double2* pn = buf + (ob[s] >> 16);
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
  } else {
    // small radix: one thread per representative DFT, fully unrolled in registers
    for (int d0 = 0; d0 < ndft; d0 += nth) {
      const int dft = d0 + tid;
      const bool act = dft < ndft;
      double2 v[q];
      unsigned rp = 0;
      bool self = false;
      if (act) {
        const int l = dft / ST::Rcnt, t = dft - l * ST::Rcnt;
        rp = reps[t] + (unsigned)(l * LP) * 0x10001u;
        self = ST::gen || t == 0;
        const double2* p = buf + (rp & 0xffffu);
        const double2 x0 = p[0];
        double2 A[H + 1], B[H + 1];
#pragma unroll
        for (int r = 1; r <= H; ++r) {
          A[r] = p[r * st];
          B[r] = p[(q - r) * st];
        }
        double2 s0 = x0;
#pragma unroll
        for (int r = 1; r <= H; ++r) s0 = cadd(s0, A[r]);
        v[0] = s0;
#pragma unroll
        for (int k = 1; k <= H; ++k) {
          double2 a = make_double2(0.0, 0.0), b = make_double2(0.0, 0.0);
#pragma unroll
          for (int r = 1; r <= H; ++r) {
            const double c = Cm[k * ST::RP + r - 1], sn = Sm[k * ST::RP + r - 1];
            a.x += A[r].x * c; a.y += A[r].y * c;
            b.x += B[r].x * sn; b.y += B[r].y * sn;
          }
          v[k] = make_double2(x0.x + a.x + b.y, x0.y + a.y - b.x);
          v[q - k] = make_double2(x0.x + a.x - b.y, x0.y + a.y + b.x);
        }
      }
      __syncthreads();
      if (act) {
        double2* p = buf + (rp & 0xffffu);
        double2* pn = buf + (rp >> 16);
#pragma unroll
        for (int k = 0; k < q; ++k) {
          p[k * st] = v[k];
          if (!self) pn[((q - k) % q) * st] = make_double2(-v[k].x, -v[k].y);
        }
      }
      __syncthreads();
    }
  }
}


// ---------------------------------------------------------------- half-line layout
// Two-factor lengths L = Q0 * Q1.  c' is odd, so the Good-Thomas grid value at (a, b) is
// -(value at (-a, -b)) and only b <= H1 = (Q1 - 1) / 2 is stored, row pitch P1h (= 4 mod 8,
// which makes the q = Q0 stage's operand loads and output stores bank-conflict-free), plus
// one zero pad element per line.  Stage 0 (along a, q = Q0) transforms the stored columns
// b = 0..H1 and needs no partner lines; stage 1 (along b, q = Q1) transforms row a together
// with its partner row -a: inputs x_r = S[a][r], x_{q-r} = -S[-a][r]; outputs V_k -> S[a][k],
// V_{q-k} -> S[-a][k] = -V_{q-k}.  Every DFT reads and writes only its own positions, so
// both stages stay in place, and no partner line is ever materialised.
template <int Q0_, int Q1_>
struct HalfShape {
  static constexpr int Q0 = Q0_, Q1 = Q1_;
  static constexpr int L = Q0 * Q1, N = L - 1;
  static constexpr int H0 = (Q0 - 1) / 2, H1 = (Q1 - 1) / 2;
  static constexpr int P1h = H1 + 1 + ((4 - (H1 + 1) % 8) + 8) % 8;  // tvd_capi.cu build_pfa
  static constexpr int PADI = Q0 * P1h;  // the zero pad element read by stage 1's padded r
  // line pitch: past the pad element, rounded up to 4 (mod 8) double2 so that the two lines of
  // a batch sit 16 words apart modulo the 32 banks and the unpack / mid gathers of a quarter
  // warp (four consecutive t of both lines, 16 bytes each) touch 32 distinct banks
  static constexpr int LPh = PADI + 1 + ((4 - (PADI + 1) % 8) + 8) % 8;
};

template <class SH, int S>
struct HalfStage {
  static constexpr bool partnered = S == 1;
  static constexpr int q = S == 0 ? SH::Q0 : SH::Q1;
  static constexpr int H = (q - 1) / 2;
  static constexpr int st = S == 0 ? SH::P1h : 1;
  static constexpr int Rcnt = S == 0 ? SH::H1 + 1 : SH::H0 + 1;
  static constexpr int KP = (H + 1 + 7) / 8 * 8;
  static constexpr int RP = (H + 3) / 4 * 4;
  static constexpr bool mma = H >= 8;
  static constexpr int LP = SH::LPh;
  __device__ static int base(int t) { return S == 0 ? t : t * SH::P1h; }
  __device__ static int partner(int t) { return S == 0 ? t : ((SH::Q0 - t) % SH::Q0) * SH::P1h; }
};

// CSM: Cm / Sm point to shared-memory copies and the A fragments are read per r-step
// (frees the 2 nrs registers of the stationary fragments)
// OOP: read `buf`, write `dst` (a second line buffer): no in-place hazard, so the warps run
// their rounds back to back without the two barriers per round, one barrier at the end.
// CO: column-owner tensor-core stage (out of place only).  A warp owns one column tile (8
// columns = 4 DFTs x re / im) and accumulates EVERY k-tile of it: per r-step it loads the data
// fragment once, folds it, and issues 2 nkt DMMAs on nkt independent accumulator pairs with
// the cos / sin fragments read through L1 -- the accumulator chains of a warp are independent,
// so the DMMA latency (29 cycles) is hidden by the warp itself instead of by more warps, at
// ~60 registers.  Every output's DMMA sequence (fragments, k-step order) is the k-tile-owner
// stage's, so the results are bit-identical.
// One column tile `ct` of the column-owner stage, k-tiles kt0 .. kt0 + NK - 1.
template <class ST, int NL, int NK, bool SMC = false>
__device__ __forceinline__ void co_tile(const double2* buf, const double* __restrict__ Cf,
                                        const double* __restrict__ Sf, double2* out, int ct,
                                        int kt0) {
  constexpr int q = ST::q, H = ST::H, st = ST::st, LP = ST::LP;
  constexpr bool PT = ST::partnered;
  constexpr int ndft = NL * ST::Rcnt;
  constexpr int nrs = ST::RP / 4;
  const int lane = threadIdx.x & 31;
  const double* bufd = reinterpret_cast<const double*>(buf);
  const int dB = min((ct * 8 + (lane >> 2)) >> 1, ndft - 1);
  const int lB = dB / ST::Rcnt, tB = dB - lB * ST::Rcnt;
  const double* p1 = bufd + 2 * (lB * LP + ST::base(tB)) + ((lane >> 2) & 1);
  const double* p2 = bufd + 2 * (lB * LP + ST::partner(tB)) + ((lane >> 2) & 1);
  const double* __restrict__ cf = Cf + kt0 * nrs * 32 + lane;  // A-fragment order (PfaStage::Cf)
  const double* __restrict__ sf = Sf + kt0 * nrs * 32 + lane;
  double acc[NK][4];
#pragma unroll
  for (int kt = 0; kt < NK; ++kt) acc[kt][0] = acc[kt][1] = acc[kt][2] = acc[kt][3] = 0.0;
#pragma unroll
  for (int rs = 0; rs < nrs; ++rs) {
    const int r = 1 + rs * 4 + (lane & 3);
    const double x1 = p1[2 * r * st];
    const double x2 = PT ? p2[2 * r * st] : p1[2 * (q - r) * st];
    const double fa = PT ? x1 - x2 : x1 + x2;
    const double fb = PT ? x1 + x2 : x1 - x2;
#pragma unroll
    for (int kt = 0; kt < NK; ++kt) {
      const int o = (kt * nrs + rs) * 32;
      // SMC: the tables are a shared-memory copy (plain loads), else global through L1
      dmma884(acc[kt][0], acc[kt][1], SMC ? cf[o] : __ldg(cf + o), fa);
      dmma884(acc[kt][2], acc[kt][3], SMC ? sf[o] : __ldg(sf + o), fb);
    }
  }
  const int dO = ct * 4 + (lane & 3);
  if (dO < ndft) {
    const int lO = dO / ST::Rcnt, tO = dO - lO * ST::Rcnt;
    const int ob = lO * LP + ST::base(tO), on = lO * LP + ST::partner(tO);
    const bool self = tO == 0;
    const double2 x0 = buf[ob];
    double2* p = out + ob;
    double2* pn = out + on;
#pragma unroll
    for (int kt = 0; kt < NK; ++kt) {
      const int k = (kt0 + kt) * 8 + (lane >> 2);
      if (k <= H) {
        const double a0 = acc[kt][0], a1 = acc[kt][1], b0 = acc[kt][2], b1 = acc[kt][3];
        const double2 vk = make_double2(x0.x + a0 + b1, x0.y + a1 - b0);
        const double2 vm = make_double2(x0.x + a0 - b1, x0.y + a1 + b0);
        if (!PT) {
          if (k == 0) {
            p[0] = vk;
          } else {
            p[k * st] = vk;
            p[(q - k) * st] = vm;
          }
        } else {
          p[k] = vk;
          if (!self) pn[k] = k == 0 ? make_double2(-vk.x, -vk.y) : make_double2(-vm.x, -vm.y);
        }
      }
    }
  }
}

template <class ST, int NL, int NW, bool SMC = false>
__device__ __forceinline__ void half_stage_co(const double2* buf, const double* __restrict__ Cf,
                                              const double* __restrict__ Sf, double2* out) {
  constexpr int ndft = NL * ST::Rcnt;
  constexpr int nkt = ST::KP / 8, nct = (2 * ndft + 7) / 8;
  const int warp = threadIdx.x >> 5;
  for (int ct = warp; ct < nct; ct += NW) co_tile<ST, NL, nkt, SMC>(buf, Cf, Sf, out, ct, 0);
  __syncthreads();
}

// Stage S of a two-factor shape in the FULL Good-Thomas layout (row pitch stride[0]) for a
// general, not odd, complex input: every column (S = 0) / row (S = 1) is a DFT line of its
// own, outputs V_k and V_{q-k} both stored.  Same members as HalfStage, so the column-owner
// stage (half_stage_co / co_tile) runs it unchanged (the assembly's band projections).
template <class SH, int S>
struct FullStage {
  using Shape = SH;
  static constexpr bool partnered = false;
  static constexpr int q = S == 0 ? SH::q[0] : SH::q[1];
  static constexpr int H = (q - 1) / 2;
  static constexpr int P1 = SH::stride[0];
  static constexpr int st = S == 0 ? P1 : 1;
  static constexpr int Rcnt = S == 0 ? SH::q[1] : SH::q[0];
  static constexpr int KP = (H + 1 + 7) / 8 * 8;
  static constexpr int RP = (H + 3) / 4 * 4;
  static constexpr bool mma = H >= 8;
  static constexpr int LP = SH::LP;
  __device__ static int base(int t) { return S == 0 ? t : t * P1; }
  __device__ static int partner(int t) { return base(t); }
};

template <class ST, int NL, int NW, int TPWc, bool CSM = false, bool OOP = false, bool CO = false>
__device__ __forceinline__ void half_stage(double2* buf, const double* Cm, const double* Sm,
                                           double2* dst = nullptr,
                                           const double* __restrict__ Cf = nullptr,
                                           const double* __restrict__ Sf = nullptr) {
  constexpr int q = ST::q, H = ST::H, st = ST::st, LP = ST::LP;
  constexpr bool PT = ST::partnered;
  const int tid = threadIdx.x, nth = blockDim.x;
  constexpr int ndft = NL * ST::Rcnt;
  double2* const out = OOP ? dst : buf;
  if constexpr (ST::mma && CO && OOP) {
    half_stage_co<ST, NL, NW, CSM>(buf, Cf, Sf, dst);
    return;
  }
  if constexpr (ST::mma) {
    // A-stationary tensor-core stage (see pfa_stage_c): warp -> one k-tile x TPW column tiles
    constexpr int nkt = ST::KP / 8, nct = (2 * ndft + 7) / 8, nrs = ST::RP / 4;
    constexpr int G = NW / nkt >= 1 ? NW / nkt : 1;
    constexpr int TPWn = (nct + G - 1) / G;
    constexpr int TPW = TPWn < TPWc ? TPWn : TPWc;
    constexpr int ROUND = G * TPW;
    const int lane = tid & 31, warp = tid >> 5;
    const int kt = warp % nkt, g = warp / nkt;
    const bool wact = warp < nkt * G;
    const int krow = kt * 8 + (lane >> 2);
    constexpr int nra = CSM ? 1 : nrs;
    double ca[nra], sa[nra];
    const double* cmk = Cf + kt * nrs * 32 + lane;  // CSM: shared copy, read per r-step
    const double* smk = Sf + kt * nrs * 32 + lane;
    if constexpr (!CSM) {
#pragma unroll
      for (int rs = 0; rs < nrs; ++rs) {  // fragment-ordered tables: coalesced 256-byte reads
        ca[rs] = __ldg(Cf + (kt * nrs + rs) * 32 + lane);
        sa[rs] = __ldg(Sf + (kt * nrs + rs) * 32 + lane);
      }
    }
#ifdef TVD_PIPE_TIMING
    const long long ts_ = clock64();
    long long tl0_ = 0, tle_ = 0, tep_ = 0;
#endif
    const double* bufd = reinterpret_cast<const double*>(buf);
    for (int ct0 = 0; ct0 < nct; ct0 += ROUND) {
      double acc[TPW][4];
      const double* p1[TPW];
      const double* p2[TPW];
#pragma unroll
      for (int j = 0; j < TPW; ++j) {
        acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.0;
        const int ct = min(ct0 + g + j * G, nct - 1);
        const int dB = min((ct * 8 + (lane >> 2)) >> 1, ndft - 1);
        const int lB = dB / ST::Rcnt, tB = dB - lB * ST::Rcnt;
        p1[j] = bufd + 2 * (lB * LP + ST::base(tB)) + ((lane >> 2) & 1);
        p2[j] = bufd + 2 * (lB * LP + ST::partner(tB)) + ((lane >> 2) & 1);
      }
#ifdef TVD_PIPE_TIMING
      tl0_ = clock64();
#endif
      if (wact) {
#pragma unroll
        for (int rs = 0; rs < nrs; ++rs) {
          const int r = 1 + rs * 4 + (lane & 3);
          double x1[TPW], x2[TPW];
#pragma unroll
          for (int j = 0; j < TPW; ++j) {
            x1[j] = p1[j][2 * r * st];
            x2[j] = PT ? p2[j][2 * r * st] : p1[j][2 * (q - r) * st];
          }
          const double car = CSM ? cmk[rs * 32] : ca[CSM ? 0 : rs];
          const double sar = CSM ? smk[rs * 32] : sa[CSM ? 0 : rs];
#pragma unroll
          for (int j = 0; j < TPW; ++j) {
            // fold: a = x_r + x_{q-r}, b = x_r - x_{q-r}; partnered x_{q-r} = -S[-a][r]
            const double fa = PT ? x1[j] - x2[j] : x1[j] + x2[j];
            const double fb = PT ? x1[j] + x2[j] : x1[j] - x2[j];
            dmma884(acc[j][0], acc[j][1], car, fa);
            dmma884(acc[j][2], acc[j][3], sar, fb);
          }
        }
      }
#ifdef TVD_PIPE_TIMING
      {
        double z_ = 0.0;
#pragma unroll
        for (int j = 0; j < TPW; ++j) z_ += acc[j][0] + acc[j][3];
        if (z_ == 12345.678) buf[0].x = z_;
        tle_ = clock64();
      }
#endif
      double2 vk[TPW], vm[TPW];
      int ob[TPW], on[TPW], oflag[TPW];
#pragma unroll
      for (int j = 0; j < TPW; ++j) {
        oflag[j] = 0;
        const int ct = ct0 + g + j * G;
        const int dO = ct * 4 + (lane & 3);
        if (wact && ct < nct && krow <= H && dO < ndft) {
          const int lO = dO / ST::Rcnt, tO = dO - lO * ST::Rcnt;
          ob[j] = lO * LP + ST::base(tO);
          on[j] = lO * LP + ST::partner(tO);
          const double2 x0 = buf[ob[j]];
          const double a0 = acc[j][0], a1 = acc[j][1], b0 = acc[j][2], b1 = acc[j][3];
          vk[j] = make_double2(x0.x + a0 + b1, x0.y + a1 - b0);
          vm[j] = make_double2(x0.x + a0 - b1, x0.y + a1 + b0);
          oflag[j] = 1 | (tO == 0 ? 2 : 0);
        }
      }
      if constexpr (!OOP) __syncthreads();
#pragma unroll
      for (int j = 0; j < TPW; ++j) {
        if (oflag[j]) {
          const int k = krow;
          double2* p = out + ob[j];
          if (!PT) {
            if (k == 0) {
              p[0] = vk[j];
            } else {
              p[k * st] = vk[j];
              p[(q - k) * st] = vm[j];
            }
          } else {
            double2* pn = out + on[j];
            const bool self = oflag[j] & 2;
            p[k] = vk[j];
            if (!self) pn[k] = k == 0 ? make_double2(-vk[j].x, -vk[j].y)
                                      : make_double2(-vm[j].x, -vm[j].y);
          }
        }
      }
#ifdef TVD_PIPE_TIMING
      tep_ = clock64();
#endif
      if constexpr (!OOP) __syncthreads();
    }
    if constexpr (OOP) __syncthreads();
#ifdef TVD_PIPE_TIMING
    if (lane == 0 && warp < 16) {
      unsigned long long* slot = g_stage_t + ((PT ? 1 : 0) * 16 + warp) * 4;
      atomicAdd(slot + 0, (unsigned long long)(tl0_ - ts_));
      atomicAdd(slot + 1, (unsigned long long)(tle_ - tl0_));
      atomicAdd(slot + 2, (unsigned long long)(tep_ - tle_));
      atomicAdd(slot + 3, (unsigned long long)(clock64() - tep_));
    }
#endif
  } else {
    // small radix: one thread per representative DFT, fully unrolled in registers
    for (int d0 = 0; d0 < ndft; d0 += nth) {
      const int dft = d0 + tid;
      const bool act = dft < ndft;
      double2 v[q];
      int obs = 0, ons = 0;
      bool self = false;
      if (act) {
        const int l = dft / ST::Rcnt, t = dft - l * ST::Rcnt;
        obs = l * LP + ST::base(t);
        ons = l * LP + ST::partner(t);
        self = t == 0;
        const double2 x0 = buf[obs];
        double2 A[H + 1], Bv[H + 1];
#pragma unroll
        for (int r = 1; r <= H; ++r) {
          const double2 x1 = buf[obs + r * st];
          const double2 x2 = PT ? make_double2(-buf[ons + r * st].x, -buf[ons + r * st].y)
                                : buf[obs + (q - r) * st];
          A[r] = cadd(x1, x2);
          Bv[r] = csub(x1, x2);
        }
        double2 s0 = x0;
#pragma unroll
        for (int r = 1; r <= H; ++r) s0 = cadd(s0, A[r]);
        v[0] = s0;
#pragma unroll
        for (int k = 1; k <= H; ++k) {
          double2 a = make_double2(0.0, 0.0), b = make_double2(0.0, 0.0);
#pragma unroll
          for (int r = 1; r <= H; ++r) {
            const double c = Cm[k * ST::RP + r - 1], sn = Sm[k * ST::RP + r - 1];
            a.x += A[r].x * c; a.y += A[r].y * c;
            b.x += Bv[r].x * sn; b.y += Bv[r].y * sn;
          }
          v[k] = make_double2(x0.x + a.x + b.y, x0.y + a.y - b.x);
          v[q - k] = make_double2(x0.x + a.x - b.y, x0.y + a.y + b.x);
        }
      }
      __syncthreads();
      if (act) {
        if (!PT) {
#pragma unroll
          for (int k = 0; k < q; ++k) out[obs + k * st] = v[k];
        } else {
#pragma unroll
          for (int k = 0; k <= H; ++k) out[obs + k] = v[k];
          if (!self) {
            out[ons] = make_double2(-v[0].x, -v[0].y);
#pragma unroll
            for (int k = 1; k <= H; ++k) out[ons + k] = make_double2(-v[q - k].x, -v[q - k].y);
          }
        }
      }
      __syncthreads();
    }
  }
}

// shared-memory coefficient tables of the CSM variant: [Cm0][Sm0][Cm1][Sm1], KP x RP each
template <class SH>
struct HalfCoef {
  using S0 = HalfStage<SH, 0>;
  using S1 = HalfStage<SH, 1>;
  static constexpr int n0 = S0::KP * S0::RP, n1 = S1::KP * S1::RP;
  static constexpr int total = 2 * (n0 + n1);
};

// CO: 0 = k-tile-owner tensor-core stages, 1 = column-owner wide stage (q = Q0), 2 = both
template <int Q0, int Q1, int NL, int NW, int TPW, bool CSM = false, bool OOP = false, int CO = 0>
__device__ __forceinline__ void half_transform(double2* buf, const PfaPlan& pl, int stages,
                                               const double* cs = nullptr,
                                               double2* buf2 = nullptr) {
  using SH = HalfShape<Q0, Q1>;
  using HC = HalfCoef<SH>;
  // stage 0 (the wide radix) reads its fragment-ordered tables from the shared copy when CSM
  const double* c0 = CSM ? cs : pl.st[0].Cf;
  const double* s0 = CSM ? cs + HC::n0 : pl.st[0].Sf;
  // OOP: stage 0 buf -> buf2, stage 1 buf2 -> buf (the result lands in buf either way)
  if (stages >= 1)
    half_stage<HalfStage<SH, 0>, NL, NW, TPW, CSM, OOP, (CO >= 1)>(buf, pl.st[0].Cm, pl.st[0].Sm,
                                                                   buf2, c0, s0);
  if (stages >= 2) {
    if constexpr (OOP)
      half_stage<HalfStage<SH, 1>, NL, NW, TPW, false, true, (CO >= 2)>(
          buf2, pl.st[1].Cm, pl.st[1].Sm, buf, pl.st[1].Cf, pl.st[1].Sf);
    else
      half_stage<HalfStage<SH, 1>, NL, NW, TPW>(buf, pl.st[1].Cm, pl.st[1].Sm, nullptr, pl.st[1].Cf,
                                                pl.st[1].Sf);
  }
}
