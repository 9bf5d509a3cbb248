// Microbenchmark: the access patterns of a transposed DST pass at 2048^2 fp64.
//  (a) "col16w": each CTA writes 2 lines as 16-byte column segments (current transposed store)
//  (b) "row_w" : each CTA writes 2 lines as contiguous rows (row-major store)
//  (c) "blk32r": each CTA reads one 32-byte segment per 2-line block (pair-blocked layout)
//  (d) "row_r" : each CTA reads 2 contiguous rows
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ub_tr tools/ubench_transpose.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int N = 2048;

__global__ void k_col16w(double* out, int nb) {  // batches of 2 lines, 2 CTAs/SM-like grid
  for (int b = blockIdx.x; b < nb; b += gridDim.x) {
    const int line0 = 2 * b;
    for (int i = threadIdx.x; i < 2 * N; i += blockDim.x) {
      const int l = i & 1, t = i >> 1;
      out[(long)t * N + line0 + l] = t * 1e-3 + l;
    }
  }
}
__global__ void k_roww(double* out, int nb) {
  for (int b = blockIdx.x; b < nb; b += gridDim.x) {
    const int line0 = 2 * b;
    for (int i = threadIdx.x; i < 2 * N; i += blockDim.x) {
      const int l = i / N, t = i - l * N;
      out[(long)(line0 + l) * N + t] = t * 1e-3 + l;
    }
  }
}
// pair-blocked layout: block p = lines (2p, 2p+1) stored [p][t][2]; a batch of 2 "columns"
// (t, t+1) of the blocked array reads, for every p, the 32 contiguous bytes [p][t..t+1][0..1]
__global__ void k_blk32r(const double* in, double* sink, int nb) {
  double acc = 0.0;
  for (int b = blockIdx.x; b < nb; b += gridDim.x) {
    const int t = 2 * b;
    for (int p = threadIdx.x; p < N / 2; p += blockDim.x) {
      const double4 v = *reinterpret_cast<const double4*>(in + ((long)p * N + t) * 2);
      acc += v.x + v.y + v.z + v.w;
    }
  }
  if (acc == 1.2345) sink[0] = acc;
}
__global__ void k_rowr(const double* in, double* sink, int nb) {
  double acc = 0.0;
  for (int b = blockIdx.x; b < nb; b += gridDim.x) {
    for (int i = threadIdx.x; i < N; i += blockDim.x) {  // 2 lines as N double2
      const double2 v = reinterpret_cast<const double2*>(in + (long)2 * b * N)[i];
      acc += v.x + v.y;
    }
  }
  if (acc == 1.2345) sink[0] = acc;
}

template <class F>
float timeit(F f) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  f();
  cudaEventRecord(e0);
  for (int i = 0; i < 20; ++i) f();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms / 20 * 1e3;
}

int main() {
  double *a, *b, *sink;
  cudaMalloc(&a, (size_t)N * N * 8);
  cudaMalloc(&b, (size_t)N * N * 8);
  cudaMalloc(&sink, 64);
  cudaMemset(a, 0, (size_t)N * N * 8);
  const int nb = N / 2, grid = 296, nt = 192;
  printf("col16w %.1f us\n", timeit([&] { k_col16w<<<grid, nt>>>(a, nb); }));
  printf("row_w  %.1f us\n", timeit([&] { k_roww<<<grid, nt>>>(a, nb); }));
  printf("blk32r %.1f us\n", timeit([&] { k_blk32r<<<grid, nt>>>(a, sink, nb); }));
  printf("row_r  %.1f us\n", timeit([&] { k_rowr<<<grid, nt>>>(a, sink, nb); }));
  return 0;
}
