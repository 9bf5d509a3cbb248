// Row-slab decomposition of one large PCG solve over several ranks.
// Included at the end of tvd_capi.cu (it uses the context, plan and launch helpers there).
//
// Rank rho of P owns the global rows [rho R, rho R + R), R = n / P, of every n x n array.
// One PCG iteration (krylov.py:99-116) is a fixed schedule of kernel phases run here and
// collectives run by the caller (paper_1011_5964_b200/slab.py) on the buffers exposed by
// tvd_slab_buffer:
//
//   MATVEC_ROWS   t = p G_1^T on the slab rows, into the interior of t_ext
//   halo          t_ext: KOFF rows to / from each neighbour; p_ext: 1 row (the L stencil)
//   MATVEC_COLS   q = G_0 t + alpha L p on the slab rows (global-row band / border fragments,
//                 AR or zero-Neumann ghosts at the image border only), contrib = local p.q
//   allgather     contrib -> gather[P]; every rank sums it in rank order (bit-identical
//                 scalars on every rank, so every rank takes the same branch)
//   GAMMA_UPDATE  gamma / step; x += step p, r -= step q, contrib = local r.r
//   allgather ; REL (stop test)
//   PREC_ROWS     row DST of r (/ d) written transposed: block j of `send` = the columns of
//                 rank j (R x R, [column][row])
//   all-to-all    send -> recv: recv[i] = rank i's rows of my columns
//   PREC_COLS     every local column is one line of P all-to-all segments (TMA bulk copy per
//                 segment): DST, x lambda^-1 (transposed-eigenvalue slab), DST, written
//                 transposed: block i of `send` = rank i's rows of my columns
//   all-to-all    send -> recv: recv[j] = my rows of rank j's columns
//   PREC_FINAL    row DST of the segmented rows (/ d), z, contrib = local r.z
//   allgather ; BETA_P (beta, p = z + beta p)
//
// With P = 1 the schedule is the single-GPU algorithm with row-major segments.

struct tvd_slab {
  tvd_ctx* ctx = nullptr;
  tvd_system sys{};
  tvd_precond pre{};
  int n = 0, R = 0, P = 1, rank = 0, row_lo = 0, khalo = 0;
  const TrigPlan* plan = nullptr;
  bool rader = false;
  bool loop = false;  // false until RZ0: the init matvec must not skip on a stale done flag
  const double* b = nullptr;
  double tol = 0.0;
  int max_it = 0;
  double* hist = nullptr;
  double *x = nullptr, *r = nullptr, *z = nullptr, *q = nullptr, *p_ext = nullptr,
         *t_ext = nullptr, *send = nullptr, *recv = nullptr, *tmp = nullptr, *partial = nullptr,
         *contrib = nullptr, *gather = nullptr;
  size_t partial_cap = 0;
  PcgState* S = nullptr;
  PcgState* hS = nullptr;
  std::vector<void*> owned;
};

static int slab_alloc(tvd_slab* s, size_t count, double** out) {
  void* p = nullptr;
  if (cudaMalloc(&p, count * sizeof(double)) != cudaSuccess)
    return fail(TVD_ERR_CUDA, "slab buffer allocation failed");
  s->owned.push_back(p);
  *out = static_cast<double*>(p);
  return TVD_OK;
}

// p (global-row indexed): p_ext holds the slab rows at row 1, one halo row on each side
static inline double* slab_p(const tvd_slab* s) { return s->p_ext + s->n; }

static int slab_local_sum(tvd_slab* s, int nb) {
  TVD_LAUNCH(s->ctx, kCatFin, 1, launch_sum_partials(s->partial, nb, s->contrib, s->ctx->stream));
  return TVD_OK;
}

static int slab_matvec_rows(tvd_slab* s) {
  tvd_ctx* c = s->ctx;
  const int n = s->n;
  const int* skip = s->loop ? &s->S->done : nullptr;
  const BandOp& g1 = s->sys.blur->g[1];
  const double* in = slab_p(s) - (long)s->row_lo * n;                   // global-row view of p
  double* out = s->t_ext + (long)s->khalo * n - (long)s->row_lo * n;  // global-row view of t
  TVD_LAUNCH(c, kCatBandRows, 1,
             launch_band_mma_rows(g1, in, out, skip, c->stream, s->row_lo, s->row_lo + s->R));
  return TVD_OK;
}

static int slab_matvec_cols(tvd_slab* s) {
  tvd_ctx* c = s->ctx;
  const int n = s->n;
  const long lo = s->row_lo;
  const int* skip = s->loop ? &s->S->done : nullptr;
  const BandOp& g0 = s->sys.blur->g[0];
  Epilogue ep{};
  const double* pv = slab_p(s) - lo * n;
  if (s->sys.a_h) {
    ep.a_h = s->sys.a_h - lo * (n + 1);
    ep.a_v = s->sys.a_v - lo * n;
    ep.lw = pv;
    ep.alpha = s->sys.alpha;
    ep.inv_h2 = 1.0 / (s->sys.spacing * s->sys.spacing);
  }
  ep.dot_with = pv;
  ep.partial = s->partial;
  ep.bc_l = s->sys.bc_l;
  const double* tv = s->t_ext + (long)s->khalo * n - lo * n;
  TVD_LAUNCH(c, kCatBandCols, 1,
             launch_band_mma_cols(g0, tv, s->q - lo * n, ep, skip, c->stream, s->row_lo,
                                  s->row_lo + s->R));
  return slab_local_sum(s, band_mma_cols_grid(n, s->R));
}

// one row pass of the slab's DST engine: `lines` lines of length n
static int slab_dst_pass(tvd_slab* s, const LineIO& io, bool transposed, int* nb) {
  tvd_ctx* c = s->ctx;
  const int fam = s->pre.family == TVD_TRANSFORM_DST1 ? kFamDst1 : kFamSineHat;
  const int cat = io.mid_mul ? kCatTrigCols : kCatTrigRows;
  if (!s->rader) {
    TVD_LAUNCH(c, cat, 1, launch_pipe(s->plan->pfa, fam, s->n, s->R, transposed ? 1 : 0, io, nb,
                                      c->stream));
    return TVD_OK;
  }
  // Rader engine: one line per CTA, row-major output, then an explicit rectangular transpose
  LineIO a = io;
  if (transposed) a.out = s->tmp;
  TVD_LAUNCH(c, cat, 1, launch_rader_rows(s->plan->rader, fam, s->n, s->R, a, nb, c->stream));
  if (transposed)
    TVD_LAUNCH(c, kCatVec, 1,
               launch_transpose_rect(s->tmp, io.out, s->R, s->n, io.skip, c->stream));
  return TVD_OK;
}

static int slab_phase(tvd_slab* s, int phase) {
  tvd_ctx* c = s->ctx;
  cudaStream_t st = c->stream;
  const long NL = (long)s->R * s->n;
  const int* skip = &s->S->done;
  const bool transform = s->pre.kind == TVD_PRECOND_TRANSFORM;
  switch (phase) {
    case TVD_SLAB_MATVEC_ROWS: return slab_matvec_rows(s);
    case TVD_SLAB_MATVEC_COLS: return slab_matvec_cols(s);
    case TVD_SLAB_RESIDUAL:
      TVD_LAUNCH(c, kCatVec, 1, launch_residual_init(s->b, s->q, s->r, NL, s->partial, vec_blocks(), st));
      return slab_local_sum(s, vec_blocks());
    case TVD_SLAB_START:
      TVD_LAUNCH(c, kCatFin, 1, launch_pcg_start(s->S, s->gather, s->P, st));
      return TVD_OK;
    case TVD_SLAB_GAMMA_UPDATE:
      TVD_LAUNCH(c, kCatFin, 1, launch_pcg_gamma(s->S, s->gather, s->P, st));
      TVD_LAUNCH(c, kCatVec, 1, launch_pcg_update_xr(s->S, s->x, s->r, slab_p(s), s->q, NL,
                                                     s->partial, vec_blocks(), st));
      return slab_local_sum(s, vec_blocks());
    case TVD_SLAB_REL:
      TVD_LAUNCH(c, kCatFin, 1, launch_pcg_rel(s->S, s->gather, s->P, s->tol, s->hist, st));
      return TVD_OK;
    case TVD_SLAB_PREC_ROWS: {
      if (!transform) {  // identity / diagonal: z and r.z locally, no exchange
        if (s->pre.kind == TVD_PRECOND_DIAG) {
          TVD_LAUNCH(c, kCatVec, 1, launch_diag_solve(s->r, s->pre.d, s->z, NL, s->partial,
                                                      vec_blocks(), skip, st));
        } else {
          TVD_LAUNCH(c, kCatVec, 1, launch_copy(s->r, s->z, NL, skip, st));
          TVD_LAUNCH(c, kCatVec, 1, launch_dot_partials(s->r, s->r, NL, s->partial, vec_blocks(),
                                                        skip, st));
        }
        return slab_local_sum(s, vec_blocks());
      }
      LineIO a{};
      a.in = s->r;
      a.out = s->send;
      a.pre = s->pre.d;
      a.skip = skip;
      int nb;
      return slab_dst_pass(s, a, true, &nb);
    }
    case TVD_SLAB_PREC_COLS: {
      if (!transform) return fail(TVD_ERR_INVALID, "PREC_COLS without a transform preconditioner");
      LineIO b{};
      b.in = s->recv;
      b.in_seg = s->R;
      b.in_seg_stride = (long)s->R * s->R;
      b.out = s->send;
      b.mid_mul = s->pre.inv_eig;
      b.skip = skip;
      int nb;
      return slab_dst_pass(s, b, true, &nb);
    }
    case TVD_SLAB_PREC_FINAL: {
      if (!transform) return fail(TVD_ERR_INVALID, "PREC_FINAL without a transform preconditioner");
      LineIO z{};
      z.in = s->recv;
      z.in_seg = s->R;
      z.in_seg_stride = (long)s->R * s->R;
      z.out = s->z;
      z.post = s->pre.d;
      z.dot_with = s->r;
      z.partial = s->partial;
      z.skip = skip;
      int nb = 0;
      int rc = slab_dst_pass(s, z, false, &nb);
      if (rc) return rc;
      return slab_local_sum(s, nb);
    }
    case TVD_SLAB_RZ0:
      TVD_LAUNCH(c, kCatFin, 1, launch_pcg_rz0(s->S, s->gather, s->P, st));
      TVD_LAUNCH(c, kCatVec, 1, launch_copy(s->z, slab_p(s), NL, skip, st));
      s->loop = true;
      return TVD_OK;
    case TVD_SLAB_BETA_P:
      TVD_LAUNCH(c, kCatFin, 1, launch_pcg_beta(s->S, s->gather, s->P, s->max_it, st));
      TVD_LAUNCH(c, kCatVec, 1, launch_pcg_update_p(s->S, slab_p(s), s->z, NL, st));
      return TVD_OK;
    default: return fail(TVD_ERR_INVALID, "unknown slab phase");
  }
}

extern "C" {

int tvd_slab_create(tvd_ctx* c, const tvd_system* sys, const tvd_precond* pre, int nranks,
                    int rank, tvd_slab** out) {
  if (!c || !out) return fail(TVD_ERR_INVALID, "null argument");
  *out = nullptr;
  int rc = check_system(sys);
  if (rc) return rc;
  tvd_blur* b = sys->blur;
  const int n = b->n;
  if (nranks < 1 || rank < 0 || rank >= nranks) return fail(TVD_ERR_INVALID, "bad rank / nranks");
  if (n % nranks) return fail(TVD_ERR_INVALID, "n must be divisible by the number of ranks");
  const int R = n / nranks;
  if (R % 8) return fail(TVD_ERR_INVALID, "slab height n / nranks must be a multiple of 8");
  if (sys->s || sys->reblur)
    return fail(TVD_ERR_INVALID, "slab solves support the X / D_X systems H^T H + alpha L");
  if (!b->separable || !band_mma_ok(b->g[0]) || !band_mma_ok(b->g[1]))
    return fail(TVD_ERR_INVALID,
                "slab solves need a separable PSF on the tensor-core band passes (n >= 256)");
  const int K = band_mma_koff(b->g[0].w);
  if (R < K) return fail(TVD_ERR_INVALID, "slab height is below the band halo");
  const TrigPlan* P = nullptr;
  bool rader = false;
  if (pre && pre->kind == TVD_PRECOND_TRANSFORM) {
    if (pre->family != TVD_TRANSFORM_SINE_HAT && pre->family != TVD_TRANSFORM_DST1)
      return fail(TVD_ERR_INVALID, "slab solves support the DST-I / Shat (M) family");
    if (!pre->inv_eig) return fail(TVD_ERR_INVALID, "transform preconditioner needs inverse eigenvalues");
    const int fam = pre->family == TVD_TRANSFORM_DST1 ? kFamDst1 : kFamSineHat;
    if (!pipe_ok(c, fam, n, &P)) {
      if (!rader_ok(c, fam, n, &P))
        return fail(TVD_ERR_INVALID, "no row-pass DST engine (PFA pipeline / Rader) for this n");
      rader = true;
    }
    if (R % 2) return fail(TVD_ERR_INVALID, "slab height must be even (16-byte segments)");
  } else if (pre && pre->kind == TVD_PRECOND_DIAG && !pre->d) {
    return fail(TVD_ERR_INVALID, "diagonal preconditioner needs d");
  } else if (pre && pre->kind != TVD_PRECOND_NONE && pre->kind != TVD_PRECOND_DIAG) {
    return fail(TVD_ERR_INVALID, "unknown preconditioner kind");
  }
  DeviceGuard g(c->device);
  auto s = std::make_unique<tvd_slab>();
  s->ctx = c;
  s->sys = *sys;
  if (pre) s->pre = *pre;
  else s->pre.kind = TVD_PRECOND_NONE;
  s->n = n;
  s->R = R;
  s->P = nranks;
  s->rank = rank;
  s->row_lo = rank * R;
  s->khalo = K;
  s->plan = P;
  s->rader = rader;
  const long NL = (long)R * n;
  s->partial_cap = std::max<size_t>({(size_t)band_mma_cols_grid(n, R), (size_t)vec_blocks(),
                                     (size_t)n + 64});
#define SLAB_ALLOC(field, count)                   \
  do {                                             \
    int rc_ = slab_alloc(s.get(), (count), &field); \
    if (rc_) {                                     \
      for (void* p_ : s->owned) cudaFree(p_);      \
      return rc_;                                  \
    }                                              \
  } while (0)
  SLAB_ALLOC(s->x, NL);
  SLAB_ALLOC(s->r, NL);
  SLAB_ALLOC(s->z, NL);
  SLAB_ALLOC(s->q, NL);
  SLAB_ALLOC(s->p_ext, NL + 2L * n);
  SLAB_ALLOC(s->t_ext, NL + 2L * K * n);
  SLAB_ALLOC(s->send, NL);
  SLAB_ALLOC(s->recv, NL);
  if (rader) SLAB_ALLOC(s->tmp, NL);
  SLAB_ALLOC(s->partial, s->partial_cap);
  SLAB_ALLOC(s->contrib, 8);
  SLAB_ALLOC(s->gather, (size_t)nranks + 8);
#undef SLAB_ALLOC
  // halo rows that lie outside the image are never read, but keep them finite
  TVD_CUDA(cudaMemsetAsync(s->p_ext, 0, (NL + 2L * n) * sizeof(double), c->stream));
  TVD_CUDA(cudaMemsetAsync(s->t_ext, 0, (NL + 2L * K * n) * sizeof(double), c->stream));
  void* st = nullptr;
  if (cudaMalloc(&st, sizeof(PcgState)) != cudaSuccess) {
    for (void* p : s->owned) cudaFree(p);
    return fail(TVD_ERR_CUDA, "slab state allocation failed");
  }
  s->owned.push_back(st);
  s->S = static_cast<PcgState*>(st);
  TVD_CUDA(cudaMemsetAsync(s->S, 0, sizeof(PcgState), c->stream));
  if (cudaMallocHost(&s->hS, sizeof(PcgState)) != cudaSuccess) {
    for (void* p : s->owned) cudaFree(p);
    return fail(TVD_ERR_CUDA, "slab host state allocation failed");
  }
  *out = s.release();
  return TVD_OK;
}

int tvd_slab_destroy(tvd_slab* s) {
  if (!s) return TVD_OK;
  DeviceGuard g(s->ctx->device);
  cudaStreamSynchronize(s->ctx->stream);
  for (void* p : s->owned) cudaFree(p);
  cudaFreeHost(s->hS);
  delete s;
  return TVD_OK;
}

int tvd_slab_info(tvd_slab* s, int* info) {
  if (!s || !info) return fail(TVD_ERR_INVALID, "null argument");
  info[0] = s->n;
  info[1] = s->R;
  info[2] = s->row_lo;
  info[3] = s->khalo;
  info[4] = 1;  // p halo rows
  info[5] = s->P;
  info[6] = s->rank;
  info[7] = s->pre.kind == TVD_PRECOND_TRANSFORM ? 1 : 0;  // the preconditioner exchanges
  return TVD_OK;
}

int tvd_slab_buffer(tvd_slab* s, int which, double** ptr, long long* count) {
  if (!s || !ptr || !count) return fail(TVD_ERR_INVALID, "null argument");
  const long long NL = (long long)s->R * s->n;
  switch (which) {
    case TVD_SLAB_BUF_X: *ptr = s->x; *count = NL; break;
    case TVD_SLAB_BUF_R: *ptr = s->r; *count = NL; break;
    case TVD_SLAB_BUF_Z: *ptr = s->z; *count = NL; break;
    case TVD_SLAB_BUF_Q: *ptr = s->q; *count = NL; break;
    case TVD_SLAB_BUF_P_EXT: *ptr = s->p_ext; *count = NL + 2LL * s->n; break;
    case TVD_SLAB_BUF_T_EXT: *ptr = s->t_ext; *count = NL + 2LL * s->khalo * s->n; break;
    case TVD_SLAB_BUF_SEND: *ptr = s->send; *count = NL; break;
    case TVD_SLAB_BUF_RECV: *ptr = s->recv; *count = NL; break;
    case TVD_SLAB_BUF_CONTRIB: *ptr = s->contrib; *count = 1; break;
    case TVD_SLAB_BUF_GATHER: *ptr = s->gather; *count = s->P; break;
    default: return fail(TVD_ERR_INVALID, "unknown slab buffer");
  }
  return TVD_OK;
}

int tvd_slab_start(tvd_slab* s, const double* b, const double* x0, double tol, int max_iterations,
                   double* history) {
  if (!s || !b || !x0) return fail(TVD_ERR_INVALID, "null argument");
  if (!(tol > 0)) return fail(TVD_ERR_INVALID, "tol must be positive");
  if (max_iterations < 1) return fail(TVD_ERR_INVALID, "max_iterations must be at least 1");
  DeviceGuard g(s->ctx->device);
  const size_t bytes = (size_t)s->R * s->n * sizeof(double);
  s->b = b;
  s->tol = tol;
  s->max_it = max_iterations;
  s->hist = history;
  s->loop = false;
  TVD_CUDA(cudaMemcpyAsync(s->x, x0, bytes, cudaMemcpyDeviceToDevice, s->ctx->stream));
  TVD_CUDA(cudaMemcpyAsync(slab_p(s), x0, bytes, cudaMemcpyDeviceToDevice, s->ctx->stream));
  return TVD_OK;
}

int tvd_slab_phase(tvd_slab* s, int phase) {
  if (!s) return fail(TVD_ERR_INVALID, "null slab");
  if (!s->b) return fail(TVD_ERR_INVALID, "tvd_slab_start was not called");
  DeviceGuard g(s->ctx->device);
  return slab_phase(s, phase);
}

int tvd_slab_status(tvd_slab* s, int* done, int* iterations, int* converged, int* err_iteration,
                    double* err_value) {
  if (!s) return fail(TVD_ERR_INVALID, "null slab");
  DeviceGuard g(s->ctx->device);
  TVD_CUDA(cudaMemcpyAsync(s->hS, s->S, sizeof(PcgState), cudaMemcpyDeviceToHost, s->ctx->stream));
  TVD_CUDA(cudaStreamSynchronize(s->ctx->stream));
  const PcgState& h = *s->hS;
  if (done) *done = h.done;
  if (iterations) *iterations = h.iters;
  if (converged) *converged = h.converged;
  if (err_iteration) *err_iteration = h.err_iter;
  if (err_value) *err_value = h.err_val;
  if (!h.done) return TVD_OK;
  if (h.status == kErrDiverged) return fail(TVD_ERR_DIVERGED, "pcg produced non-finite values");
  if (h.status == kErrIndefinite) return fail(TVD_ERR_INDEFINITE, "pcg met nonpositive curvature");
  return TVD_OK;
}

}  // extern "C"
