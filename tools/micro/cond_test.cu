// conditional WHILE node with a nested IF, built by stream capture (probe for the level loop)
#include <cuda_runtime.h>
#include <cstdio>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)
__global__ void k_init(int *c) { c[0] = 0; c[1] = 0; c[2] = 0; }
__global__ void k_body(int *c) { c[0]++; }
__global__ void k_end(int *c, cudaGraphConditionalHandle hw, cudaGraphConditionalHandle hi) {
  cudaGraphSetConditional(hw, c[0] < 7 ? 1 : 0);
  cudaGraphSetConditional(hi, (c[0] % 3) == 0 ? 1 : 0);
}
__global__ void k_if(int *c) { c[1]++; }
__global__ void k_after(int *c) { c[2] = 100 + c[0]; }
static cudaGraphNode_t add_cond(cudaStream_t s, cudaGraphConditionalHandle h, cudaGraphConditionalNodeType t, cudaGraph_t *body) {
  cudaStreamCaptureStatus st; cudaGraph_t cg; const cudaGraphNode_t *deps; size_t nd;
  cudaStreamGetCaptureInfo(s, &st, nullptr, &cg, &deps, &nd);
  cudaGraphNodeParams p = {}; p.type = cudaGraphNodeTypeConditional; p.conditional.handle = h; p.conditional.type = t; p.conditional.size = 1;
  cudaGraphNode_t n; cudaError_t e = cudaGraphAddNode(&n, cg, deps, nd, &p);
  if (e != cudaSuccess) printf("add node: %s\n", cudaGetErrorString(e));
  *body = p.conditional.phGraph_out[0];
  cudaStreamUpdateCaptureDependencies(s, &n, 1, cudaStreamSetCaptureDependencies);
  return n;
}
int main() {
  int *c; CK(cudaMalloc(&c, 16));
  cudaStream_t s, s2; CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking)); CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
  cudaGraph_t g; CK(cudaGraphCreate(&g, 0));
  cudaGraphConditionalHandle hw; CK(cudaGraphConditionalHandleCreate(&hw, g, 1, cudaGraphCondAssignDefault));
  CK(cudaStreamBeginCaptureToGraph(s, g, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
  k_init<<<1,1,0,s>>>(c);
  cudaGraph_t body; add_cond(s, hw, cudaGraphCondTypeWhile, &body);
  cudaGraphConditionalHandle hi; CK(cudaGraphConditionalHandleCreate(&hi, body, 0, cudaGraphCondAssignDefault));
  CK(cudaStreamBeginCaptureToGraph(s2, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
  k_body<<<1,1,0,s2>>>(c);
  k_end<<<1,1,0,s2>>>(c, hw, hi);
  cudaGraph_t ib; add_cond(s2, hi, cudaGraphCondTypeIf, &ib);
  cudaStream_t s3; CK(cudaStreamCreateWithFlags(&s3, cudaStreamNonBlocking));
  CK(cudaStreamBeginCaptureToGraph(s3, ib, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
  k_if<<<1,1,0,s3>>>(c);
  cudaGraph_t tmp; CK(cudaStreamEndCapture(s3, &tmp));
  CK(cudaStreamEndCapture(s2, &tmp));
  k_after<<<1,1,0,s>>>(c);
  CK(cudaStreamEndCapture(s, &g));
  cudaGraphExec_t ex; CK(cudaGraphInstantiate(&ex, g, 0));
  for (int it = 0; it < 3; it++) {
    CK(cudaGraphLaunch(ex, s)); CK(cudaStreamSynchronize(s));
    int h[3]; CK(cudaMemcpy(h, c, 12, cudaMemcpyDeviceToHost));
    printf("iter %d: body=%d if=%d after=%d\n", it, h[0], h[1], h[2]);
  }
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0, s); for (int i = 0; i < 100; i++) cudaGraphLaunch(ex, s); cudaEventRecord(e1, s); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1); printf("per launch %.2f us (7 iterations, ~17 kernels)\n", ms * 10);
  return 0;
}
