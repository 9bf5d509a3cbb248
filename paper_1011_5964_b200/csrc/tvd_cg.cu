// PCG state machine + vector kernels.  The recurrence, its check order and its
// error semantics follow krylov.py:82-116 exactly; vector updates use explicit
// round-to-nearest ops so they match numpy's `x += step * p` bit for bit.
// Reductions are deterministic: fixed grids write per-CTA partials, one
// 512-thread CTA sums them in a fixed order.
#include <cmath>

#include "tvd_cg.h"

namespace tvd {

constexpr int kVecThreads = 256;
int vec_blocks() { return kRedBlocks; }

__device__ __forceinline__ double sum_partials_block(const double* partial, int nb) {
  __shared__ double red[32];
  double v = 0.0;
  for (int i = threadIdx.x; i < nb; i += blockDim.x) v += partial[i];
  return block_sum(v, red);
}

__global__ void k_sum_partials(const double* partial, int nb, double* out) {
  const double s = sum_partials_block(partial, nb);
  if (threadIdx.x == 0) *out = s;
}

__global__ void k_residual_init(const double* __restrict__ b, const double* __restrict__ q,
                                double* __restrict__ r, long N, double* partial) {
  __shared__ double red[32];
  double acc = 0.0;
  for (long g = blockIdx.x * (long)blockDim.x + threadIdx.x; g < N; g += (long)gridDim.x * blockDim.x) {
    const double v = __dsub_rn(b[g], q[g]);
    r[g] = v;
    acc += v * v;
  }
  const double s = block_sum(acc, red);
  if (threadIdx.x == 0) partial[blockIdx.x] = s;
}

__global__ void k_pcg_start(PcgState* s, const double* partial, int nb) {
  const double rr = sum_partials_block(partial, nb);
  if (threadIdx.x == 0) {
    s->r0 = sqrt(rr);
    s->k = 1;
    s->status = kOk;
    s->err_iter = 0;
    s->err_val = 0.0;
    s->converged = 0;
    s->iters = 0;
    s->done = 0;
    s->x_pending = 0;
    if (s->r0 == 0.0) {
      s->done = 1;
      s->iters = 0;
      s->converged = 1;
    }
  }
}

__global__ void k_pcg_rz0(PcgState* s, const double* partial, int nb) {
  if (s->done) return;
  const double rz = sum_partials_block(partial, nb);
  if (threadIdx.x == 0) s->rz = rz;
}

__global__ void k_copy(const double* __restrict__ src, double* __restrict__ dst, long N, const int* skip) {
  if (skip && *skip) return;
  for (long g = blockIdx.x * (long)blockDim.x + threadIdx.x; g < N; g += (long)gridDim.x * blockDim.x)
    dst[g] = src[g];
}

__global__ void k_pcg_gamma(PcgState* s, const double* partial, int nb) {
  pdl_enter();
  if (s->done) return;
  const double gamma = sum_partials_block(partial, nb);
  if (threadIdx.x == 0) pcg_fin_gamma(s, gamma);
}

// x += step p ; r -= step q ; partial = |r|^2.  128-bit accesses, two pairs per thread in
// flight; odd N leaves one tail element to thread 0.
__global__ void k_pcg_update_xr(const PcgState* s, double* __restrict__ x, double* __restrict__ r,
                                const double* __restrict__ p, const double* __restrict__ q, long N,
                                double* partial, PcgFin fin) {
  pdl_enter();
  if (s->done) return;
  __shared__ double red[32];
  const double step = s->step;
  const long N2 = N >> 1, stride = (long)gridDim.x * blockDim.x;
  double2* __restrict__ x2 = reinterpret_cast<double2*>(x);
  double2* __restrict__ r2 = reinterpret_cast<double2*>(r);
  const double2* __restrict__ p2 = reinterpret_cast<const double2*>(p);
  const double2* __restrict__ q2 = reinterpret_cast<const double2*>(q);
  double acc = 0.0;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < N2; i += 2 * stride) {
    const long j = i + stride;
    const bool two = j < N2;
    const double2 xa = x2[i], pa = p2[i], ra = r2[i], qa = q2[i];
    double2 xb = make_double2(0.0, 0.0), pb = xb, rb = xb, qb = xb;
    if (two) {
      xb = x2[j];
      pb = p2[j];
      rb = r2[j];
      qb = q2[j];
    }
    x2[i] = make_double2(__dadd_rn(xa.x, __dmul_rn(step, pa.x)), __dadd_rn(xa.y, __dmul_rn(step, pa.y)));
    const double2 va = make_double2(__dsub_rn(ra.x, __dmul_rn(step, qa.x)),
                                    __dsub_rn(ra.y, __dmul_rn(step, qa.y)));
    r2[i] = va;
    acc += va.x * va.x;
    acc += va.y * va.y;
    if (two) {
      x2[j] = make_double2(__dadd_rn(xb.x, __dmul_rn(step, pb.x)), __dadd_rn(xb.y, __dmul_rn(step, pb.y)));
      const double2 vb = make_double2(__dsub_rn(rb.x, __dmul_rn(step, qb.x)),
                                      __dsub_rn(rb.y, __dmul_rn(step, qb.y)));
      r2[j] = vb;
      acc += vb.x * vb.x;
      acc += vb.y * vb.y;
    }
  }
  if ((N & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
    const long g = N - 1;
    x[g] = __dadd_rn(x[g], __dmul_rn(step, p[g]));
    const double v = __dsub_rn(r[g], __dmul_rn(step, q[g]));
    r[g] = v;
    acc += v * v;
  }
  const double t = block_sum(acc, red);
  if (threadIdx.x == 0) partial[blockIdx.x] = t;
  if (fin.s) pcg_fin_tail(fin, partial, gridDim.x, red);  // stop test in the last CTA
}

__global__ void k_pcg_update_r(const PcgState* s, double* __restrict__ r,
                               const double* __restrict__ q, long N, double* partial, PcgFin fin) {
  pdl_enter();
  if (s->done) return;
  __shared__ double red[32];
  const double step = s->step;
  const long N2 = N >> 1, stride = (long)gridDim.x * blockDim.x;
  double2* __restrict__ r2 = reinterpret_cast<double2*>(r);
  const double2* __restrict__ q2 = reinterpret_cast<const double2*>(q);
  double acc = 0.0;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < N2; i += 2 * stride) {
    const long j = i + stride;
    const bool two = j < N2;
    const double2 ra = r2[i], qa = q2[i];
    double2 rb = make_double2(0.0, 0.0), qb = rb;
    if (two) {
      rb = r2[j];
      qb = q2[j];
    }
    const double2 va = make_double2(__dsub_rn(ra.x, __dmul_rn(step, qa.x)),
                                    __dsub_rn(ra.y, __dmul_rn(step, qa.y)));
    r2[i] = va;
    acc += va.x * va.x;
    acc += va.y * va.y;
    if (two) {
      const double2 vb = make_double2(__dsub_rn(rb.x, __dmul_rn(step, qb.x)),
                                      __dsub_rn(rb.y, __dmul_rn(step, qb.y)));
      r2[j] = vb;
      acc += vb.x * vb.x;
      acc += vb.y * vb.y;
    }
  }
  if ((N & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
    const long g = N - 1;
    const double v = __dsub_rn(r[g], __dmul_rn(step, q[g]));
    r[g] = v;
    acc += v * v;
  }
  const double t = block_sum(acc, red);
  if (threadIdx.x == 0) partial[blockIdx.x] = t;
  if (fin.s) pcg_fin_tail(fin, partial, gridDim.x, red);  // stop test in the last CTA
}

__global__ void k_pcg_update_x(PcgState* s, double* __restrict__ x, const double* __restrict__ p,
                               long N, unsigned* counter) {
  pdl_enter();
  if (!s->x_pending) return;
  const double step = s->step;
  const long N2 = N >> 1, stride = (long)gridDim.x * blockDim.x;
  double2* __restrict__ x2 = reinterpret_cast<double2*>(x);
  const double2* __restrict__ p2 = reinterpret_cast<const double2*>(p);
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < N2; i += 2 * stride) {
    const long j = i + stride;
    const bool two = j < N2;
    const double2 xa = x2[i], pa = p2[i];
    double2 xb = make_double2(0.0, 0.0), pb = xb;
    if (two) {
      xb = x2[j];
      pb = p2[j];
    }
    x2[i] = make_double2(__dadd_rn(xa.x, __dmul_rn(step, pa.x)), __dadd_rn(xa.y, __dmul_rn(step, pa.y)));
    if (two)
      x2[j] = make_double2(__dadd_rn(xb.x, __dmul_rn(step, pb.x)), __dadd_rn(xb.y, __dmul_rn(step, pb.y)));
  }
  if ((N & 1) && blockIdx.x == 0 && threadIdx.x == 0) x[N - 1] = __dadd_rn(x[N - 1], __dmul_rn(step, p[N - 1]));
  // the last CTA to finish (every CTA has read x_pending) clears it
  __shared__ int last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(counter, 1u) == gridDim.x - 1;
  __syncthreads();
  if (last && threadIdx.x == 0) {
    s->x_pending = 0;
    *counter = 0u;
  }
}

__global__ void k_pcg_rel(PcgState* s, const double* partial, int nb, double tol, double* hist) {
  pdl_enter();
  if (s->done) return;
  const double rr = sum_partials_block(partial, nb);
  if (threadIdx.x == 0) pcg_fin_rel(s, rr, tol, hist);
}

__global__ void k_pcg_beta(PcgState* s, const double* partial, int nb, int max_it) {
  pdl_enter();
  if (s->done) return;
  const double rz_next = sum_partials_block(partial, nb);
  if (threadIdx.x == 0) pcg_fin_beta(s, rz_next, max_it);
}

// p = z + beta p (numpy rounding); 128-bit accesses, two pairs per thread in flight.
__global__ void k_pcg_update_p(const PcgState* s, double* __restrict__ p, const double* __restrict__ z,
                               long N) {
  pdl_enter();
  if (s->done) return;
  const double beta = s->beta;
  const long N2 = N >> 1, stride = (long)gridDim.x * blockDim.x;
  double2* __restrict__ p2 = reinterpret_cast<double2*>(p);
  const double2* __restrict__ z2 = reinterpret_cast<const double2*>(z);
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < N2; i += 2 * stride) {
    const long j = i + stride;
    const bool two = j < N2;
    const double2 pa = p2[i], za = z2[i];
    double2 pb = make_double2(0.0, 0.0), zb = pb;
    if (two) {
      pb = p2[j];
      zb = z2[j];
    }
    p2[i] = make_double2(__dadd_rn(za.x, __dmul_rn(beta, pa.x)), __dadd_rn(za.y, __dmul_rn(beta, pa.y)));
    if (two)
      p2[j] = make_double2(__dadd_rn(zb.x, __dmul_rn(beta, pb.x)), __dadd_rn(zb.y, __dmul_rn(beta, pb.y)));
  }
  if ((N & 1) && blockIdx.x == 0 && threadIdx.x == 0) p[N - 1] = __dadd_rn(z[N - 1], __dmul_rn(beta, p[N - 1]));
}

__global__ void k_diag_solve(const double* __restrict__ r, const double* __restrict__ d,
                             double* __restrict__ z, long N, double* partial, const int* skip) {
  if (skip && *skip) return;
  __shared__ double red[32];
  double acc = 0.0;
  for (long g = blockIdx.x * (long)blockDim.x + threadIdx.x; g < N; g += (long)gridDim.x * blockDim.x) {
    const double v = __ddiv_rn(r[g], d[g]);
    z[g] = v;
    acc += r[g] * v;
  }
  const double t = block_sum(acc, red);
  if (threadIdx.x == 0 && partial) partial[blockIdx.x] = t;
}

__global__ void k_dot_partials(const double* __restrict__ x, const double* __restrict__ y, long N,
                               double* partial, const int* skip) {
  if (skip && *skip) return;
  __shared__ double red[32];
  double acc = 0.0;
  for (long g = blockIdx.x * (long)blockDim.x + threadIdx.x; g < N; g += (long)gridDim.x * blockDim.x)
    acc += x[g] * y[g];
  const double t = block_sum(acc, red);
  if (threadIdx.x == 0) partial[blockIdx.x] = t;
}

__global__ void k_axpby(double a, const double* __restrict__ x, double b, const double* __restrict__ y,
                        double* __restrict__ out, long N) {
  for (long g = blockIdx.x * (long)blockDim.x + threadIdx.x; g < N; g += (long)gridDim.x * blockDim.x) {
    const double u = a == 1.0 ? x[g] : __dmul_rn(a, x[g]);
    const double v = b == 1.0 ? y[g] : __dmul_rn(b, y[g]);
    out[g] = __dadd_rn(u, v);
  }
}

__global__ void k_mul(const double* __restrict__ x, const double* __restrict__ y, double* __restrict__ out,
                      long N) {
  for (long g = blockIdx.x * (long)blockDim.x + threadIdx.x; g < N; g += (long)gridDim.x * blockDim.x)
    out[g] = __dmul_rn(x[g], y[g]);
}

__global__ void k_div(const double* __restrict__ x, const double* __restrict__ y, double* __restrict__ out,
                      long N) {
  for (long g = blockIdx.x * (long)blockDim.x + threadIdx.x; g < N; g += (long)gridDim.x * blockDim.x)
    out[g] = __ddiv_rn(x[g], y[g]);
}

__global__ void k_scaling(const double* __restrict__ diag, double alpha, double* d, double* dsq,
                          double* s, long N, double* partial_min) {
  __shared__ double red[32];
  double mn = 1.0 / 0.0;
  for (long g = blockIdx.x * (long)blockDim.x + threadIdx.x; g < N; g += (long)gridDim.x * blockDim.x) {
    const double v = __dadd_rn(1.0, __dmul_rn(alpha, diag[g]));
    if (d) d[g] = v;
    if (dsq) dsq[g] = __dsqrt_rn(v);
    if (s) s[g] = pow(v, -0.5);
    mn = fmin(mn, v);
  }
  for (int o = 16; o > 0; o >>= 1) mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) red[wid] = mn;
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = red[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) m = fmin(m, red[w]);
    partial_min[blockIdx.x] = m;
  }
}

__global__ void k_scale_bands(const double* __restrict__ diag, const double* __restrict__ inner,
                              const double* __restrict__ block, const double* __restrict__ s, int n,
                              double* diag_s, double* inner_s, double* block_s) {
  const long N = (long)n * n;
  for (long g = blockIdx.x * (long)blockDim.x + threadIdx.x; g < N; g += (long)gridDim.x * blockDim.x) {
    const int i = (int)(g / n), j = (int)(g % n);
    diag_s[g] = __dmul_rn(__dmul_rn(diag[g], s[g]), s[g]);
    if (j < n - 1) {
      const long h = (long)i * (n - 1) + j;
      inner_s[h] = __dmul_rn(__dmul_rn(inner[h], s[g]), s[g + 1]);
    }
    if (i < n - 1) block_s[g] = __dmul_rn(__dmul_rn(block[g], s[g]), s[g + n]);
  }
}

__global__ void k_invert_eigs(const double* __restrict__ lam, double floor, double* __restrict__ inv,
                              long N, double* partial) {
  __shared__ double red[32];
  double cnt = 0.0;
  for (long g = blockIdx.x * (long)blockDim.x + threadIdx.x; g < N; g += (long)gridDim.x * blockDim.x) {
    const double v = lam[g];
    if (v < floor) cnt += 1.0;
    inv[g] = __ddiv_rn(1.0, fmax(v, floor));
  }
  const double t = block_sum(cnt, red);
  if (threadIdx.x == 0) partial[blockIdx.x] = t;
}

// device-side checks of the deferred assembly (tvd_precond_assemble_async): the scaling
// diagonal's minimum, the eigenvalues' min / max (per-CTA pairs), the clamp floor read back
// from device memory, and the clamp count
__global__ void k_reduce_min(const double* partial_min, int nb, double* out) {
  __shared__ double red[32];
  double mn = 1.0 / 0.0;
  for (int i = threadIdx.x; i < nb; i += blockDim.x) mn = fmin(mn, partial_min[i]);
  for (int o = 16; o > 0; o >>= 1) mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mn;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) mn = fmin(mn, red[w]);
    *out = mn;
  }
}
__global__ void k_reduce_minmax(const double* partial_mm, int nb, double* out_min, double* out_max) {
  __shared__ double rmn[32], rmx[32];
  double mn = 1.0 / 0.0, mx = -1.0 / 0.0;
  for (int i = threadIdx.x; i < nb; i += blockDim.x) {
    mn = fmin(mn, partial_mm[2 * i]);
    mx = fmax(mx, partial_mm[2 * i + 1]);
  }
  for (int o = 16; o > 0; o >>= 1) {
    mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  if ((threadIdx.x & 31) == 0) {
    rmn[threadIdx.x >> 5] = mn;
    rmx[threadIdx.x >> 5] = mx;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
      mn = fmin(mn, rmn[w]);
      mx = fmax(mx, rmx[w]);
    }
    *out_min = mn;
    *out_max = mx;
  }
}
__global__ void k_invert_eigs_dev(const double* __restrict__ lam, const double* max_lam,
                                  double* __restrict__ inv, long N, double* partial) {
  __shared__ double red[32];
  const double floor = 1e-14 * *max_lam;  // precond.py:442 (same rounding as the host's)
  double cnt = 0.0;
  for (long g = blockIdx.x * (long)blockDim.x + threadIdx.x; g < N; g += (long)gridDim.x * blockDim.x) {
    const double v = lam[g];
    if (v < floor) cnt += 1.0;
    inv[g] = __ddiv_rn(1.0, fmax(v, floor));
  }
  const double t = block_sum(cnt, red);
  if (threadIdx.x == 0) partial[blockIdx.x] = t;
}

// ------------------------------------------------------------- launchers
#define TVD_VEC_GRID kRedBlocks, kVecThreads, 0, st

cudaError_t launch_sum_partials(const double* partial, int nb, double* out, cudaStream_t st) {
  k_sum_partials<<<1, 512, 0, st>>>(partial, nb, out);
  return cudaGetLastError();
}
cudaError_t launch_residual_init(const double* b, const double* q, double* r, long N, double* partial,
                                 int, cudaStream_t st) {
  k_residual_init<<<TVD_VEC_GRID>>>(b, q, r, N, partial);
  return cudaGetLastError();
}
cudaError_t launch_pcg_start(PcgState* s, const double* partial, int nb, cudaStream_t st) {
  k_pcg_start<<<1, 512, 0, st>>>(s, partial, nb);
  return cudaGetLastError();
}
cudaError_t launch_pcg_rz0(PcgState* s, const double* partial, int nb, cudaStream_t st) {
  k_pcg_rz0<<<1, 512, 0, st>>>(s, partial, nb);
  return cudaGetLastError();
}
cudaError_t launch_copy(const double* src, double* dst, long N, const int* skip, cudaStream_t st) {
  k_copy<<<TVD_VEC_GRID>>>(src, dst, N, skip);
  return cudaGetLastError();
}
cudaError_t launch_pcg_gamma(PcgState* s, const double* partial, int nb, cudaStream_t st) {
  return launch_pdl(k_pcg_gamma, 1, 512, 0, st, s, partial, nb);
}
cudaError_t launch_pcg_update_xr(PcgState* s, double* x, double* r, const double* p, const double* q,
                                 long N, double* partial, int, cudaStream_t st, const PcgFin* fin) {
  return launch_pdl(k_pcg_update_xr, kRedBlocks, kVecThreads, 0, st, s, x, r, p, q, N, partial,
                    fin ? *fin : PcgFin{});
}
cudaError_t launch_pcg_update_r(PcgState* s, double* r, const double* q, long N, double* partial,
                                cudaStream_t st, const PcgFin* fin) {
  return launch_pdl(k_pcg_update_r, kRedBlocks, kVecThreads, 0, st, s, r, q, N, partial,
                    fin ? *fin : PcgFin{});
}
cudaError_t launch_pcg_update_x(PcgState* s, double* x, const double* p, long N, unsigned* counter,
                                cudaStream_t st) {
  return launch_pdl(k_pcg_update_x, kRedBlocks, kVecThreads, 0, st, s, x, p, N, counter);
}
cudaError_t launch_pcg_rel(PcgState* s, const double* partial, int nb, double tol, double* hist,
                           cudaStream_t st) {
  return launch_pdl(k_pcg_rel, 1, 512, 0, st, s, partial, nb, tol, hist);
}
cudaError_t launch_pcg_beta(PcgState* s, const double* partial, int nb, int max_it, cudaStream_t st) {
  return launch_pdl(k_pcg_beta, 1, 512, 0, st, s, partial, nb, max_it);
}
cudaError_t launch_pcg_update_p(PcgState* s, double* p, const double* z, long N, cudaStream_t st) {
  return launch_pdl(k_pcg_update_p, kRedBlocks, kVecThreads, 0, st, s, p, z, N);
}
cudaError_t launch_diag_solve(const double* r, const double* d, double* z, long N, double* partial, int,
                              const int* skip, cudaStream_t st) {
  k_diag_solve<<<TVD_VEC_GRID>>>(r, d, z, N, partial, skip);
  return cudaGetLastError();
}
cudaError_t launch_dot_partials(const double* x, const double* y, long N, double* partial, int,
                                const int* skip, cudaStream_t st) {
  k_dot_partials<<<TVD_VEC_GRID>>>(x, y, N, partial, skip);
  return cudaGetLastError();
}
cudaError_t launch_axpby(double a, const double* x, double b, const double* y, double* out, long N,
                         cudaStream_t st) {
  k_axpby<<<TVD_VEC_GRID>>>(a, x, b, y, out, N);
  return cudaGetLastError();
}
cudaError_t launch_mul(const double* x, const double* y, double* out, long N, cudaStream_t st) {
  k_mul<<<TVD_VEC_GRID>>>(x, y, out, N);
  return cudaGetLastError();
}
cudaError_t launch_div(const double* x, const double* y, double* out, long N, cudaStream_t st) {
  k_div<<<TVD_VEC_GRID>>>(x, y, out, N);
  return cudaGetLastError();
}
cudaError_t launch_scaling(const double* diag, double alpha, double* d, double* dsq, double* s, long N,
                           double* partial_min, int, cudaStream_t st) {
  k_scaling<<<TVD_VEC_GRID>>>(diag, alpha, d, dsq, s, N, partial_min);
  return cudaGetLastError();
}
cudaError_t launch_scale_bands(const double* diag, const double* inner, const double* block,
                               const double* s, int n, double* diag_s, double* inner_s,
                               double* block_s, cudaStream_t st) {
  k_scale_bands<<<TVD_VEC_GRID>>>(diag, inner, block, s, n, diag_s, inner_s, block_s);
  return cudaGetLastError();
}
cudaError_t launch_invert_eigs(const double* lam, double floor, double* inv, long N, double* partial,
                               int, cudaStream_t st) {
  k_invert_eigs<<<TVD_VEC_GRID>>>(lam, floor, inv, N, partial);
  return cudaGetLastError();
}
cudaError_t launch_invert_eigs_dev(const double* lam, const double* max_lam, double* inv, long N,
                                   double* partial, cudaStream_t st) {
  k_invert_eigs_dev<<<TVD_VEC_GRID>>>(lam, max_lam, inv, N, partial);
  return cudaGetLastError();
}
cudaError_t launch_reduce_min(const double* partial_min, int nb, double* out, cudaStream_t st) {
  k_reduce_min<<<1, 512, 0, st>>>(partial_min, nb, out);
  return cudaGetLastError();
}
cudaError_t launch_reduce_minmax(const double* partial_mm, int nb, double* out_min, double* out_max,
                                 cudaStream_t st) {
  k_reduce_minmax<<<1, 512, 0, st>>>(partial_mm, nb, out_min, out_max);
  return cudaGetLastError();
}

// ------------------------------------------------------------ BiCGstab (krylov.py:119-174)
__device__ __forceinline__ void bicg_fail(BicgState* s, int status, double val) {
  s->status = status;
  s->err_iter = s->k;
  s->err_val = val;
  s->done = 1;
  s->halt = 1;
}

__global__ void k_bicg_start(BicgState* s, const double* partial, int nb) {
  const double rr = sum_partials_block(partial, nb);
  if (threadIdx.x == 0) {
    s->r0 = sqrt(rr);
    s->rho = s->alpha = s->omega = 1.0;
    s->k = 1;
    s->status = kOk;
    s->err_iter = 0;
    s->err_val = 0.0;
    s->converged = 0;
    s->iters = 0;
    s->early = 0;
    s->done = s->halt = 0;
    if (s->r0 == 0.0) {
      s->done = s->halt = 1;
      s->converged = 1;
    }
  }
}

// rho_next = rs . r ; beta
__global__ void k_bicg_rho(BicgState* s, const double* partial, int nb) {
  if (s->halt) return;
  const double rho_next = sum_partials_block(partial, nb);
  if (threadIdx.x == 0) {
    s->rho_next = rho_next;
    if (fabs(rho_next) < 1e-30 * s->r0 * s->r0) {
      bicg_fail(s, kErrBreakdown, 1.0);  // "rho vanished"
      return;
    }
    s->beta = (rho_next / s->rho) * (s->alpha / s->omega);
  }
}

// p = r + beta (p - omega v)
__global__ void k_bicg_update_p(const BicgState* s, double* __restrict__ p,
                                const double* __restrict__ r, const double* __restrict__ v,
                                long N) {
  if (s->halt) return;
  const double beta = s->beta, omega = s->omega;
  for (long g = blockIdx.x * (long)blockDim.x + threadIdx.x; g < N; g += (long)gridDim.x * blockDim.x)
    p[g] = __dadd_rn(r[g], __dmul_rn(beta, __dsub_rn(p[g], __dmul_rn(omega, v[g]))));
}

// alpha = rho_next / (rs . v)
__global__ void k_bicg_alpha(BicgState* s, const double* partial, int nb) {
  if (s->halt) return;
  const double denom = sum_partials_block(partial, nb);
  if (threadIdx.x == 0) {
    if (fabs(denom) < 1e-300) {
      bicg_fail(s, kErrBreakdown, 2.0);  // "shadow angle vanished"
      return;
    }
    s->alpha = s->rho_next / denom;
  }
}

// s = r - alpha v ; partial |s|^2
__global__ void k_bicg_s(const BicgState* st, double* __restrict__ sv, const double* __restrict__ r,
                         const double* __restrict__ v, long N, double* partial) {
  if (st->halt) return;
  __shared__ double red[32];
  const double alpha = st->alpha;
  double acc = 0.0;
  for (long g = blockIdx.x * (long)blockDim.x + threadIdx.x; g < N; g += (long)gridDim.x * blockDim.x) {
    const double x = __dsub_rn(r[g], __dmul_rn(alpha, v[g]));
    sv[g] = x;
    acc += x * x;
  }
  const double t = block_sum(acc, red);
  if (threadIdx.x == 0) partial[blockIdx.x] = t;
}

// rel = |s| / r0: divergence check, early convergence (x += alpha p_hat follows)
__global__ void k_bicg_srel(BicgState* s, const double* partial, int nb, double tol) {
  if (s->halt) return;
  const double ss = sum_partials_block(partial, nb);
  if (threadIdx.x == 0) {
    const double rel = sqrt(ss) / s->r0;
    s->rel = rel;
    if (!isfinite(rel)) {
      bicg_fail(s, kErrDiverged, 0.0);
      return;
    }
    if (rel < tol) {
      s->early = 1;
      s->halt = 1;
    }
  }
}

// omega = (t . s) / (t . t)
__global__ void k_bicg_omega(BicgState* s, const double* p_ts, int nb_ts, const double* p_tt,
                             int nb_tt) {
  if (s->halt) return;
  const double ts = sum_partials_block(p_ts, nb_ts);
  __syncthreads();
  const double tt = sum_partials_block(p_tt, nb_tt);
  if (threadIdx.x == 0) {
    if (tt == 0.0) {
      bicg_fail(s, kErrBreakdown, 3.0);  // "stabilizer direction vanished"
      return;
    }
    const double omega = ts / tt;
    if (fabs(omega) < 1e-300) {
      bicg_fail(s, kErrBreakdown, 4.0);  // "omega vanished"
      return;
    }
    s->omega = omega;
  }
}

// early: x += alpha p_hat ; else x += alpha p_hat + omega s_hat, r = s - omega t, |r|^2
__global__ void k_bicg_update_xr(const BicgState* st, double* __restrict__ x, double* __restrict__ r,
                                 const double* __restrict__ ph, const double* __restrict__ sh,
                                 const double* __restrict__ sv, const double* __restrict__ t,
                                 long N, double* partial) {
  if (st->done) return;
  __shared__ double red[32];
  const double alpha = st->alpha, omega = st->omega;
  const bool early = st->early;
  double acc = 0.0;
  for (long g = blockIdx.x * (long)blockDim.x + threadIdx.x; g < N; g += (long)gridDim.x * blockDim.x) {
    if (early) {
      x[g] = __dadd_rn(x[g], __dmul_rn(alpha, ph[g]));
    } else {
      x[g] = __dadd_rn(x[g], __dadd_rn(__dmul_rn(alpha, ph[g]), __dmul_rn(omega, sh[g])));
      const double v = __dsub_rn(sv[g], __dmul_rn(omega, t[g]));
      r[g] = v;
      acc += v * v;
    }
  }
  const double tot = block_sum(acc, red);
  if (threadIdx.x == 0) partial[blockIdx.x] = tot;
}

// end of iteration k: history, convergence / exhaustion, rho <- rho_next
__global__ void k_bicg_rel(BicgState* s, const double* partial, int nb, double tol, double* hist,
                           int max_it) {
  if (s->done) return;
  const double rr = sum_partials_block(partial, nb);
  if (threadIdx.x == 0) {
    if (s->early) {  // converged on the s residual
      if (hist) hist[s->k - 1] = s->rel;
      s->iters = s->k;
      s->converged = 1;
      s->done = s->halt = 1;
      return;
    }
    const double rel = sqrt(rr) / s->r0;
    s->rel = rel;
    if (!isfinite(rel)) {
      bicg_fail(s, kErrDiverged, 0.0);
      return;
    }
    if (hist) hist[s->k - 1] = rel;
    if (rel < tol) {
      s->iters = s->k;
      s->converged = 1;
      s->done = s->halt = 1;
      return;
    }
    s->rho = s->rho_next;
    s->k += 1;
    if (s->k > max_it) {
      s->iters = max_it;
      s->converged = 0;
      s->done = s->halt = 1;
    }
  }
}

cudaError_t launch_bicg_start(BicgState* s, const double* partial, int nb, cudaStream_t st) {
  k_bicg_start<<<1, 512, 0, st>>>(s, partial, nb);
  return cudaGetLastError();
}
cudaError_t launch_bicg_rho(BicgState* s, const double* partial, int nb, cudaStream_t st) {
  k_bicg_rho<<<1, 512, 0, st>>>(s, partial, nb);
  return cudaGetLastError();
}
cudaError_t launch_bicg_update_p(BicgState* s, double* p, const double* r, const double* v, long N,
                                 cudaStream_t st) {
  k_bicg_update_p<<<kRedBlocks, kVecThreads, 0, st>>>(s, p, r, v, N);
  return cudaGetLastError();
}
cudaError_t launch_bicg_alpha(BicgState* s, const double* partial, int nb, cudaStream_t st) {
  k_bicg_alpha<<<1, 512, 0, st>>>(s, partial, nb);
  return cudaGetLastError();
}
cudaError_t launch_bicg_s(BicgState* s, double* sv, const double* r, const double* v, long N,
                          double* partial, cudaStream_t st) {
  k_bicg_s<<<kRedBlocks, kVecThreads, 0, st>>>(s, sv, r, v, N, partial);
  return cudaGetLastError();
}
cudaError_t launch_bicg_srel(BicgState* s, const double* partial, double tol, cudaStream_t st) {
  k_bicg_srel<<<1, 512, 0, st>>>(s, partial, kRedBlocks, tol);
  return cudaGetLastError();
}
cudaError_t launch_bicg_omega(BicgState* s, const double* p_ts, int nb_ts, const double* p_tt,
                              int nb_tt, cudaStream_t st) {
  k_bicg_omega<<<1, 512, 0, st>>>(s, p_ts, nb_ts, p_tt, nb_tt);
  return cudaGetLastError();
}
cudaError_t launch_bicg_update_xr(BicgState* s, double* x, double* r, const double* p_hat,
                                  const double* s_hat, const double* sv, const double* t, long N,
                                  double* partial, cudaStream_t st) {
  k_bicg_update_xr<<<kRedBlocks, kVecThreads, 0, st>>>(s, x, r, p_hat, s_hat, sv, t, N, partial);
  return cudaGetLastError();
}
cudaError_t launch_bicg_rel(BicgState* s, const double* partial, double tol, double* hist,
                            int max_it, cudaStream_t st) {
  k_bicg_rel<<<1, 512, 0, st>>>(s, partial, kRedBlocks, tol, hist, max_it);
  return cudaGetLastError();
}

}  // namespace tvd
