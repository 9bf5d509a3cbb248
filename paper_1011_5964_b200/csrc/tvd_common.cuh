// Common helpers for the tvdeblur B200 kernels (fp64 throughout).
#pragma once

#include <cuda_runtime.h>
#include <cstdint>
#include <cstdlib>
#include <utility>

namespace tvd {

constexpr int kSMs = 148;          // B200 SM count (grid sizing)
constexpr int kRedBlocks = 592;    // fixed partial-sum grid = 4 x 148 (deterministic reductions)

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cscale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
__device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }

// Warp + block sum in a fixed order (deterministic for a fixed launch shape).
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Stores with an L2 evict_last policy for arrays the next kernels read again: the band passes
// write t, p and q that way, so the column pass and the HBM-bound x / r update find them in
// the 126 MB L2 (x / r update 30.5 -> 27.8 us, c3 2911 -> 2951 PCG it/s).  The same hint on r
// and on the M^-1 intermediates measured no further gain (the pinned set then competes with
// q: the update went back to 29.3 us), so only the band passes use it.
__device__ __forceinline__ unsigned long long l2_keep_policy() {
  unsigned long long pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void st2_keep(double* p, double x, double y, unsigned long long pol) {
  asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;\n" ::"l"(p), "d"(x), "d"(y), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void st1_keep(double* p, double x, unsigned long long pol) {
  asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;\n" ::"l"(p), "d"(x), "l"(pol) : "memory");
}

// Sum over the block; result valid in thread 0.  `scratch` >= 32 doubles.
__device__ __forceinline__ double block_sum(double v, double* scratch) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int nw = (blockDim.x + 31) >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) scratch[wid] = v;
  __syncthreads();
  double t = 0.0;
  if (wid == 0) {
    t = lane < nw ? scratch[lane] : 0.0;
    t = warp_sum(t);
  }
  return t;
}

// Programmatic dependent launch (PDL).  The PCG iteration kernels (DST / Rader / generic line
// passes, both band passes, the vector updates and finalizers) are launched with the
// programmatic-stream-serialization attribute (`launch_pdl`): a kernel's grid is launched as
// soon as every CTA of the previous one has exited, before that grid's completion and memory
// flush, so the launch latency overlaps the previous kernel's drain.  Every kernel launched
// that way calls `pdl_enter()` FIRST, unconditionally (also before its done / skip test, which
// reads state the previous kernel wrote): griddepcontrol.wait blocks until the previous grid
// has completed and its memory is visible, so completion stays transitive along the stream.
// An explicit early trigger (griddepcontrol.launch_dependents right after the wait, so the
// next grid's CTAs become resident during this one's last wave) measured 8 % SLOWER on c3
// (2330 vs 2532 it/s) and is off by default (-DTVD_PDL_EARLY_TRIGGER=1 builds it).  Both
// instructions are no-ops for a grid launched without the attribute.  Wait-only PDL: neutral
// at c3 (2787 vs 2782 it/s), and +17 / +31 / +24 / +20 % on single-stream c1 / c2a / c2b / c4
// solves (round 2, tools/pcg_ab.py pdl 0,1 CONFIG), whose short kernels leave the launch
// latency exposed; on by default, option TVD_OPT_PDL.
// A LATE trigger (launch_dependents when a CTA of a single-wave grid -- the persistent DST
// passes, the x / r update -- enters its last batch, with every kernel's wait moved behind its
// constant-table prologue) measured +0.5 % on c3 and -8 % on the four-stream c4 batch, where
// dependents parked on drained SMs starve the other streams' kernels: no kernel triggers.
#ifndef TVD_PDL_EARLY_TRIGGER
#define TVD_PDL_EARLY_TRIGGER 0
#endif
__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (TVD_PDL_EARLY_TRIGGER) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// Process-wide switches set through tvd_ctx_set_option (include/tvdeblur_b200.h TVD_OPT_*);
// every default is the measured production configuration.
enum TvdOpt : int {
  kOptGenericFft = 1, kOptSolverGraph, kOptPdl, kOptBandGeneric, kOptBandSlide, kOptFinFusion,
  kOptPFusion, kOptPfaStages, kOptGeneralBlur, kOptBandPrefetch, kOptSplitX, kOptGuardSlots, kOptCount
};
int option(int id);  // tvd_capi.cu

inline bool pdl_enabled() { return option(kOptPdl) != 0; }

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

}  // namespace tvd
