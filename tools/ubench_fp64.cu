// Microbenchmark: FP64 DMMA (mma.sync m8n8k4 f64) and DFMA latency / throughput on B200.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench_fp64 tools/ubench_fp64.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

template <int CH>
__global__ void k_dmma(double* out, int iters, double a, double b) {
  double d[CH][2];
#pragma unroll
  for (int c = 0; c < CH; ++c) d[c][0] = d[c][1] = threadIdx.x * 1e-3 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) dmma(d[c][0], d[c][1], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += d[c][0] + d[c][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int CH>
__global__ void k_dfma(double* out, int iters, double a, double b) {
  double d[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) d[c] = threadIdx.x * 1e-3 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) d[c] = fma(d[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += d[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// DMMA and DFMA chains interleaved in one warp: do the two fp64 paths add up?
template <int CH, int CF>
__global__ void k_mixed(double* out, int iters, double a, double b) {
  double d[CH][2], f[CF];
#pragma unroll
  for (int c = 0; c < CH; ++c) d[c][0] = d[c][1] = threadIdx.x * 1e-3 + c;
#pragma unroll
  for (int c = 0; c < CF; ++c) f[c] = threadIdx.x * 1e-3 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) dmma(d[c][0], d[c][1], a, b);
#pragma unroll
    for (int c = 0; c < CF; ++c) f[c] = fma(f[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += d[c][0] + d[c][1];
#pragma unroll
  for (int c = 0; c < CF; ++c) s += f[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <class F>
float timeit(F f) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  f();
  cudaEventRecord(e0);
  f();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms;
}

int main() {
  double* out;
  cudaMalloc(&out, 1 << 26);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int iters = 4096;
  // latency: 1 warp, 1 chain
  float ms = timeit([&] { k_dmma<1><<<1, 32>>>(out, iters, 1.0, 1e-9); });
  printf("DMMA latency  : %.1f cycles (at %d MHz)\n", ms * 1e-3 * clk * 1e3 / iters, clk / 1000);
  ms = timeit([&] { k_dfma<1><<<1, 32>>>(out, iters, 1.0, 1e-9); });
  printf("DFMA latency  : %.1f cycles\n", ms * 1e-3 * clk * 1e3 / iters);
  // throughput: full GPU
  for (int w : {4, 8, 16, 32}) {
    ms = timeit([&] { k_dmma<8><<<148 * 4, 32 * w / 4>>>(out, iters, 1.0, 1e-9); });
    const double fma = 148.0 * 4 * (32.0 * w / 4 / 32) * iters * 8 * 256;
    printf("DMMA thru (%2d warps/SM, 8 chains): %.2f TFLOP/s\n", w, 2 * fma / (ms * 1e-3) / 1e12);
  }
  for (int w : {4, 8, 16, 32}) {
    ms = timeit([&] { k_dfma<8><<<148 * 4, 32 * w / 4>>>(out, iters, 1.0, 1e-9); });
    const double fma = 148.0 * 4 * (32.0 * w / 4) * iters * 8;
    printf("DFMA thru (%2d warps/SM, 8 chains): %.2f TFLOP/s\n", w, 2 * fma / (ms * 1e-3) / 1e12);
  }
  // mixed: 8 DMMA chains + CF DFMA chains per thread, 16 warps / SM
  for (int w : {16}) {
    const int blocks = 148 * 4, threads = 32 * w / 4;
    ms = timeit([&] { k_mixed<8, 8><<<blocks, threads>>>(out, iters, 1.0, 1e-9); });
    double dm = 2.0 * blocks * (threads / 32) * (double)iters * 8 * 256;
    double df = 2.0 * blocks * threads * (double)iters * 8;
    printf("mixed 8 DMMA + 8 DFMA chains: %.2f TFLOP/s total (%.2f DMMA + %.2f DFMA)\n",
           (dm + df) / (ms * 1e-3) / 1e12, dm / (ms * 1e-3) / 1e12, df / (ms * 1e-3) / 1e12);
    ms = timeit([&] { k_mixed<8, 32><<<blocks, threads>>>(out, iters, 1.0, 1e-9); });
    df = 2.0 * blocks * threads * (double)iters * 32;
    printf("mixed 8 DMMA + 32 DFMA chains: %.2f TFLOP/s total (%.2f DMMA + %.2f DFMA)\n",
           (dm + df) / (ms * 1e-3) / 1e12, dm / (ms * 1e-3) / 1e12, df / (ms * 1e-3) / 1e12);
  }
  return 0;
}
