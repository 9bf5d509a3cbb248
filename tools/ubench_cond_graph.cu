// Feasibility check (not product): a CUDA-graph WHILE conditional node whose body is stream-captured;
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o ub tools/ubench_cond_graph.cu && ./ub  (B200: 49 us for 5
// trips of 3 dependent one-warp kernels, i.e. 3.3 us per dependent kernel inside the loop)
#include <cstdio>
#include <cuda_runtime.h>
__global__ void body(int* k) { if (threadIdx.x == 0) *k += 1; }
__global__ void cond(int* k, cudaGraphConditionalHandle h) {
  if (threadIdx.x == 0) cudaGraphSetConditional(h, *k < 10 ? 1u : 0u);
}
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s -> %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)
int main() {
  int* k; CK(cudaMalloc(&k, 4)); CK(cudaMemset(k, 0, 4));
  cudaStream_t st; CK(cudaStreamCreate(&st));
  cudaGraph_t g; CK(cudaGraphCreate(&g, 0));
  cudaGraphConditionalHandle h;
  CK(cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault));
  cudaGraphNodeParams p = {};
  p.type = cudaGraphNodeTypeConditional;
  p.conditional.handle = h;
  p.conditional.type = cudaGraphCondTypeWhile;
  p.conditional.size = 1;
  cudaGraphNode_t node;
  CK(cudaGraphAddNode(&node, g, nullptr, 0, &p));
  cudaGraph_t bodyg = p.conditional.phGraph_out[0];
  CK(cudaStreamBeginCaptureToGraph(st, bodyg, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
  body<<<1, 32, 0, st>>>(k);
  body<<<1, 32, 0, st>>>(k);
  cond<<<1, 32, 0, st>>>(k, h);
  cudaGraph_t tmp; CK(cudaStreamEndCapture(st, &tmp));
  cudaGraphExec_t ex; CK(cudaGraphInstantiate(&ex, g, 0));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int rep = 0; rep < 3; ++rep) {
    CK(cudaMemset(k, 0, 4));
    cudaEventRecord(e0, st);
    CK(cudaGraphLaunch(ex, st));
    cudaEventRecord(e1, st);
    CK(cudaStreamSynchronize(st));
    int hk; CK(cudaMemcpy(&hk, k, 4, cudaMemcpyDeviceToHost));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("k = %d (expect 10), %.1f us for 5 loop trips of 3 kernels\n", hk, ms * 1e3);
  }
  return 0;
}
