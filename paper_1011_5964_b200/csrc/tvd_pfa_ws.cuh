// Warp-specialised DST-I row pass for the two-factor half-line shapes (included by
// tvd_pfa.cu after k_dst_pipe; same semantics as k_dst_pipe without the AR transform hooks).
//
// k_dst_pipe runs every phase of a batch with all warps in lock step: pack (table-driven
// scatter of the TMA-staged rows), the two Good-Thomas DFT stages (fp64 tensor cores), the
// unpack (gather, scaling, stores, dot).  Pack / unpack are load-store and latency bound, the
// stages DMMA and barrier bound, so they leave each other's units idle.  Here NP producer
// warps own the global side (TMA issue, pack, unpack, stores, dot partials) and NC consumer
// warps own the transforms, on two line buffers: while the consumers transform batch j in
// buffer j & 1, the producers unpack batch j - 1 from the other buffer and pack batch j + 1
// into it.  Hand-off uses named barriers (bar.arrive by the signalling group, bar.sync by the
// waiting one: FULL[b] "buffer b packed", DONE[b] "buffer b transformed"); each group syncs
// internally on its own named barrier.  The sandwich pass's middle step (x lambda^-1 and the
// re-pack) runs on the consumers between their two transforms.
#pragma once

namespace ws {

__device__ __forceinline__ void bar_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void bar_arrive(int id, int count) {
  asm volatile("bar.arrive %0, %1;\n" ::"r"(id), "r"(count) : "memory");
}

// barrier ids (0 is __syncthreads)
constexpr int kFull0 = 1, kDone0 = 3, kCons = 5, kProd = 6;

// half_stage (tvd_pfa_t.cuh) for a thread group: tid / NW warps of the group, group barrier
template <class ST, int NL, int NW, int TPWc>
__device__ __forceinline__ void stage_grp(double2* buf, const double* Cm, const double* Sm,
                                          const int tid) {
  constexpr int q = ST::q, H = ST::H, st = ST::st, LP = ST::LP;
  constexpr bool PT = ST::partnered;
  constexpr int nth = NW * 32;
  constexpr int ndft = NL * ST::Rcnt;
  if constexpr (ST::mma) {
    constexpr int nkt = ST::KP / 8, nct = (2 * ndft + 7) / 8, nrs = ST::RP / 4;
    constexpr int G = NW / nkt >= 1 ? NW / nkt : 1;
    constexpr int TPWn = (nct + G - 1) / G;
    constexpr int TPW = TPWn < TPWc ? TPWn : TPWc;
    constexpr int ROUND = G * TPW;
    static_assert(NW >= nkt, "every k-tile needs a warp");
    const int lane = tid & 31, warp = tid >> 5;
    const int kt = warp % nkt, g = warp / nkt;
    const bool wact = warp < nkt * G;
    const int krow = kt * 8 + (lane >> 2);
    double ca[nrs], sa[nrs];
    const double* cmk = Cm + krow * ST::RP + (lane & 3);
    const double* smk = Sm + krow * ST::RP + (lane & 3);
#pragma unroll
    for (int rs = 0; rs < nrs; ++rs) {
      ca[rs] = cmk[rs * 4];
      sa[rs] = smk[rs * 4];
    }
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
#pragma unroll
          for (int j = 0; j < TPW; ++j) {
            const double fa = PT ? x1[j] - x2[j] : x1[j] + x2[j];
            const double fb = PT ? x1[j] + x2[j] : x1[j] - x2[j];
            dmma884(acc[j][0], acc[j][1], ca[rs], fa);
            dmma884(acc[j][2], acc[j][3], sa[rs], fb);
          }
        }
      }
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
      bar_sync(kCons, nth);
#pragma unroll
      for (int j = 0; j < TPW; ++j) {
        if (oflag[j]) {
          const int k = krow;
          double2* p = buf + ob[j];
          if (!PT) {
            if (k == 0) {
              p[0] = vk[j];
            } else {
              p[k * st] = vk[j];
              p[(q - k) * st] = vm[j];
            }
          } else {
            double2* pn = buf + on[j];
            const bool self = oflag[j] & 2;
            p[k] = vk[j];
            if (!self) pn[k] = k == 0 ? make_double2(-vk[j].x, -vk[j].y)
                                      : make_double2(-vm[j].x, -vm[j].y);
          }
        }
      }
      bar_sync(kCons, nth);
    }
  } else {
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
      bar_sync(kCons, nth);
      if (act) {
        if (!PT) {
#pragma unroll
          for (int k = 0; k < q; ++k) buf[obs + k * st] = v[k];
        } else {
#pragma unroll
          for (int k = 0; k <= H; ++k) buf[obs + k] = v[k];
          if (!self) {
            buf[ons] = make_double2(-v[0].x, -v[0].y);
#pragma unroll
            for (int k = 1; k <= H; ++k) buf[ons + k] = make_double2(-v[q - k].x, -v[q - k].y);
          }
        }
      }
      bar_sync(kCons, nth);
    }
  }
}

template <int Q0, int Q1, int NL, int NW, int TPW>
__device__ __forceinline__ void transform_grp(double2* buf, const PfaPlan& pl, int tid) {
  using SH = HalfShape<Q0, Q1>;
  stage_grp<HalfStage<SH, 0>, NL, NW, TPW>(buf, pl.st[0].Cm, pl.st[0].Sm, tid);
  stage_grp<HalfStage<SH, 1>, NL, NW, TPW>(buf, pl.st[1].Cm, pl.st[1].Sm, tid);
}

}  // namespace ws

// NP producer warps + NC consumer warps, B = 2 lines per batch, two line buffers.
template <int Q1, int Q2, int NP, int NC, int TPW, int MINB = 1>
__global__ void __launch_bounds__((NP + NC) * 32, MINB) k_dst_ws(const PipeK p) {
  using SH = PfaShape<Q1, Q2, 1>;
  using HS = HalfShape<Q1, Q2>;
  constexpr int B = 2, LP = HS::LPh, N = SH::N;
  constexpr int NPT = NP * 32, NCT = NC * 32, ALL = NPT + NCT;
  constexpr int kTp = (N + NPT - 1) / NPT;  // t-values per producer thread per line
  constexpr int kTc = (N + NCT - 1) / NCT;  // t-values per consumer thread (sandwich)
  if (p.skip && *p.skip) return;
  extern __shared__ __align__(16) unsigned char smraw[];
  __shared__ double red[32];
  __shared__ double bord[2][B][2];
  __shared__ __align__(8) unsigned long long mbar;
  const int tid = threadIdx.x, n = p.n;
  const bool producer = tid < NPT;
  double2* const buf0 = reinterpret_cast<double2*>(smraw);  // line buffer b at buf0 + b B LP
  double* stage = reinterpret_cast<double*>(buf0 + 2 * B * LP);
  const unsigned* __restrict__ scat = p.pl.hscat;
  const unsigned* __restrict__ gath = p.pl.hgath;
  // the balanced batch schedule of k_dst_pipe
  const int G = gridDim.x, c = blockIdx.x;
  const int F = p.nlines / (B * G), rem = p.nlines - F * B * G;
  const int tl0 = F * B * G + (int)((long)c * rem / G);
  const int tl1 = F * B * G + (int)((long)(c + 1) * rem / G);
  const int nb = F + (tl1 > tl0 ? 1 : 0);
  auto first_of = [&](int j) { return j < F ? (j * G + c) * B : tl0; };
  auto rows_of = [&](int j) { return j < F ? B : tl1 - tl0; };
  auto issue = [&](int j) {
    const int first = first_of(j), rows = rows_of(j);
    mbar_expect_tx(&mbar, (unsigned)(rows * n * 8));
    for (int l = 0; l < rows; ++l) {
      const long r = (long)(first + l) * n;
      if (p.in_seg) {
        const long base = (long)(first + l) * p.in_seg;
        for (int s0 = 0; s0 < n; s0 += p.in_seg)
          bulk_g2s(stage + l * n + s0, p.in + (s0 / p.in_seg) * p.in_seg_stride + base,
                   (unsigned)(p.in_seg * 8), &mbar);
      } else {
        bulk_g2s(stage + l * n, p.in + r, (unsigned)(n * 8), &mbar);
      }
      if (p.pre) bulk_prefetch_l2(p.pre + r, (unsigned)(n * 8));
      if (p.mid) bulk_prefetch_l2(p.mid + r, (unsigned)(n * 8));
      if (!p.transposed) {
        if (p.post) bulk_prefetch_l2(p.post + r, (unsigned)(n * 8));
        if (p.dot_with) bulk_prefetch_l2(p.dot_with + r, (unsigned)(n * 8));
      }
    }
  };
  if (tid == 0) {
    mbar_init(&mbar, 1);
    if (nb > 0) issue(0);
  }
  __syncthreads();
  auto unpack_at = [&](const double2* res, int l, unsigned gi, int k) {
    double2 C = res[l * LP + (gi & 0x7fffu)];
    if (gi & 0x8000u) C = make_double2(-C.x, -C.y);
    return ((k & 1) ? -(C.y + C.x) : -(C.y - C.x)) * p.scale;
  };
  auto scatter = [&](double* bl, int t, unsigned e, double x) {
    double* b = bl + (t & 1);
    b[2 * (e & 0x7fffu)] = (e & 0x8000u) ? -x : x;
    if (e >> 31) b[2 * ((e >> 16) & 0x7fffu)] = -x;
  };
  const long nl_out = p.nlines;
  double acc = 0.0;
  if (producer) {
    unsigned phase = 0;
    // unpack + store batch j from buffer j & 1 (k_dst_pipe's unpack, producer threads)
    auto unpack_batch = [&](int j) {
      const double2* res = buf0 + (j & 1) * B * LP;
      const int line0 = first_of(j), nlv = rows_of(j);
      if (p.transposed) {
        const int l = tid & (B - 1);
        constexpr int TS = NPT / B;
        constexpr int JT = (N + TS - 1) / TS;
        constexpr int JG = 8;
        if (l < nlv) {
          const long cb = (long)(p.off - 1) * nl_out + line0 + l;
          double* __restrict__ ocol = p.out + cb;
          const double* __restrict__ dcol = p.dot_with ? p.dot_with + cb : nullptr;
          const double* __restrict__ qcol = p.post ? p.post + cb : nullptr;
          const int t0 = 1 + tid / B;
#pragma unroll
          for (int j0 = 0; j0 < JT; j0 += JG) {
            unsigned gg[JG];
            double y[JG], q[JG], dv[JG];
#pragma unroll
            for (int jj = 0; jj < JG; ++jj) {
              const int t = t0 + (j0 + jj) * TS;
              const bool ok = j0 + jj < JT && t <= N;
              gg[jj] = ok ? __ldg(gath + t - 1) : 0u;
              q[jj] = (qcol && ok) ? qcol[(long)t * nl_out] : 1.0;
              dv[jj] = (dcol && ok) ? dcol[(long)t * nl_out] : 0.0;
            }
#pragma unroll
            for (int jj = 0; jj < JG; ++jj) {
              const int t = t0 + (j0 + jj) * TS;
              if (j0 + jj < JT && t <= N) {
                double y = unpack_at(res, l, gg[jj], t);
                if (qcol) y = p.post_mul ? y * q[jj] : y / q[jj];
                ocol[(long)t * nl_out] = y;
                acc += y * dv[jj];
              }
            }
            (void)y;
          }
        }
      } else {
        unsigned g[kTp];
#pragma unroll
        for (int k = 0; k < kTp; ++k) {
          const int t = 1 + tid + k * NPT;
          g[k] = (k < kTp - 1 || t <= N) ? __ldg(gath + t - 1) : 0u;
        }
        for (int l = 0; l < nlv; ++l) {
          const long rowb = (long)(line0 + l) * n + p.off - 1;
          double* __restrict__ orow = p.out + rowb;
          const double* __restrict__ drow = p.dot_with ? p.dot_with + rowb : nullptr;
          const double* __restrict__ qrow = p.post ? p.post + rowb : nullptr;
          double q[kTp], dv[kTp];
#pragma unroll
          for (int k = 0; k < kTp; ++k) {
            const int t = 1 + tid + k * NPT;
            const bool ok = k < kTp - 1 || t <= N;
            q[k] = (qrow && ok) ? qrow[t] : 1.0;
            dv[k] = (drow && ok) ? drow[t] : 0.0;
          }
#pragma unroll
          for (int k = 0; k < kTp; ++k) {
            const int t = 1 + tid + k * NPT;
            if (k < kTp - 1 || t <= N) {
              double y = unpack_at(res, l, g[k], t);
              if (qrow) y = p.post_mul ? y * q[k] : y / q[k];
              orow[t] = y;
              acc += y * dv[k];
            }
          }
        }
      }
      if (p.off && tid < 2 * nlv) {  // Shat borders pass through (x mid, then post)
        const int l = tid >> 1, e = (tid & 1) ? n - 1 : 0;
        double y = bord[j & 1][l][tid & 1];
        if (p.mid) y *= p.mid[(long)(line0 + l) * n + e];
        const long gidx = p.transposed ? (long)e * nl_out + line0 + l : (long)(line0 + l) * n + e;
        if (p.post) y = p.post_mul ? y * p.post[gidx] : y / p.post[gidx];
        p.out[gidx] = y;
        if (p.dot_with) acc += y * p.dot_with[gidx];
      }
    };
    for (int j = 0; j < nb; ++j) {
      const int bi = j & 1;
      double2* buf = buf0 + bi * B * LP;
      const int line0 = first_of(j), nlv = rows_of(j);
      unsigned e[kTp];
#pragma unroll
      for (int k = 0; k < kTp; ++k) {
        const int t = 1 + tid + k * NPT;
        e[k] = (k < kTp - 1 || t <= N) ? __ldg(scat + t - 1) : 0u;
      }
      // buffer bi held batch j - 2, unpacked at iteration j - 1 by every producer thread:
      // free once all of them are past that unpack.  Zero its pads.
      if (j >= 1) ws::bar_sync(ws::kProd, NPT);
      for (int i = tid; i < B; i += NPT) {
        buf[i * LP] = make_double2(0.0, 0.0);
        buf[i * LP + LP - 1] = make_double2(0.0, 0.0);
      }
      for (int i = tid; i < (B - nlv) * LP; i += NPT) buf[nlv * LP + i] = make_double2(0.0, 0.0);
      mbar_wait(&mbar, phase);
      phase ^= 1u;
      for (int l = 0; l < nlv; ++l) {
        const double* srow = stage + l * n + p.off - 1;
        double x[kTp];
#pragma unroll
        for (int k = 0; k < kTp; ++k) {
          const int t = 1 + tid + k * NPT;
          x[k] = (k < kTp - 1 || t <= N) ? srow[t] : 0.0;
        }
        if (p.pre) {
          const double* __restrict__ prow = p.pre + (long)(line0 + l) * n + p.off - 1;
          double q[kTp];
#pragma unroll
          for (int k = 0; k < kTp; ++k) {
            const int t = 1 + tid + k * NPT;
            q[k] = (k < kTp - 1 || t <= N) ? prow[t] : 1.0;
          }
#pragma unroll
          for (int k = 0; k < kTp; ++k) x[k] = p.pre_mul ? x[k] * q[k] : x[k] / q[k];
        }
        double* bl = reinterpret_cast<double*>(buf + l * LP);
#pragma unroll
        for (int k = 0; k < kTp; ++k) {
          const int t = 1 + tid + k * NPT;
          if (k < kTp - 1 || t <= N) scatter(bl, t, e[k], x[k]);
        }
      }
      if (p.off && tid < 2 * nlv) {
        const int l = tid >> 1, ee = (tid & 1) ? n - 1 : 0;
        double x = stage[l * n + ee];
        if (p.pre) {
          const double q = p.pre[(long)(line0 + l) * n + ee];
          x = p.pre_mul ? x * q : x / q;
        }
        bord[bi][l][tid & 1] = x;
      }
      ws::bar_sync(ws::kProd, NPT);  // staging fully read, buffer fully written
      if (tid == 0 && j + 1 < nb) {
        fence_proxy_async();
        issue(j + 1);
      }
      ws::bar_arrive(ws::kFull0 + bi, ALL);
      if (j >= 1) {
        ws::bar_sync(ws::kDone0 + (bi ^ 1), ALL);
        unpack_batch(j - 1);
      }
    }
    if (nb > 0) {
      ws::bar_sync(ws::kDone0 + ((nb - 1) & 1), ALL);
      unpack_batch(nb - 1);
    }
  } else {
    const int ctid = tid - NPT;
    for (int j = 0; j < nb; ++j) {
      const int bi = j & 1;
      double2* buf = buf0 + bi * B * LP;
      ws::bar_sync(ws::kFull0 + bi, ALL);
      ws::transform_grp<Q1, Q2, B, NC, TPW>(buf, p.pl, ctid);
      if (p.mid) {  // sandwich: x lambda^-1 (row of the transposed grid), re-pack, transform
        const int line0 = first_of(j), nlv = rows_of(j);
        double v[B][kTc];
#pragma unroll
        for (int l = 0; l < B; ++l) {
          const double* __restrict__ mrow = p.mid + (long)(line0 + min(l, nlv - 1)) * n + p.off - 1;
#pragma unroll
          for (int k = 0; k < kTc; ++k) {
            const int t = 1 + ctid + k * NCT;
            v[l][k] = (l < nlv && t <= N) ? mrow[t] : 0.0;
          }
        }
#pragma unroll
        for (int l = 0; l < B; ++l)
#pragma unroll
          for (int k = 0; k < kTc; ++k) {
            const int t = 1 + ctid + k * NCT;
            if (l < nlv && t <= N) v[l][k] *= unpack_at(buf, l, __ldg(gath + t - 1), t);
          }
        ws::bar_sync(ws::kCons, NCT);
#pragma unroll
        for (int l = 0; l < B; ++l) {
          double* bl = reinterpret_cast<double*>(buf + l * LP);
#pragma unroll
          for (int k = 0; k < kTc; ++k) {
            const int t = 1 + ctid + k * NCT;
            if (l < nlv && t <= N) scatter(bl, t, __ldg(scat + t - 1), v[l][k]);
          }
        }
        for (int i = ctid; i < B; i += NCT) {
          buf[i * LP] = make_double2(0.0, 0.0);
          buf[i * LP + LP - 1] = make_double2(0.0, 0.0);
        }
        ws::bar_sync(ws::kCons, NCT);
        ws::transform_grp<Q1, Q2, B, NC, TPW>(buf, p.pl, ctid);
      }
      ws::bar_arrive(ws::kDone0 + bi, ALL);
    }
  }
  if (p.partial) {
    const double s = block_sum(acc, red);
    if (tid == 0) p.partial[blockIdx.x] = s;
    if (p.fin.s) pcg_fin_tail(p.fin, p.partial, gridDim.x, red);
  }
}
