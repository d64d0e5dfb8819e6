#include <cstdio>
#include <cuda_runtime.h>
__global__ void body(int* counter, cudaGraphConditionalHandle h, int limit) {
  int c = ++(*counter);
  if (c >= limit) cudaGraphSetConditional(h, 0);
}
__global__ void work(double* x) { x[threadIdx.x] += 1.0; }
int main() {
  int* cnt; double* x;
  cudaMalloc(&cnt, 4); cudaMalloc(&x, 256 * 8);
  cudaMemset(cnt, 0, 4); cudaMemset(x, 0, 256 * 8);
  cudaGraph_t g; cudaGraphCreate(&g, 0);
  cudaGraphConditionalHandle h;
  cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault);
  cudaGraphNodeParams cp = {};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = h;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t node;
  cudaError_t e = cudaGraphAddNode(&node, g, nullptr, 0, &cp);
  printf("add node %s\n", cudaGetErrorString(e));
  cudaGraph_t bodyg = cp.conditional.phGraph_out[0];
  cudaStream_t s; cudaStreamCreate(&s);
  e = cudaStreamBeginCaptureToGraph(s, bodyg, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed);
  printf("begin capture %s\n", cudaGetErrorString(e));
  work<<<1, 256, 0, s>>>(x);
  body<<<1, 1, 0, s>>>(cnt, h, 5);
  e = cudaStreamEndCapture(s, &bodyg);
  printf("end capture %s\n", cudaGetErrorString(e));
  cudaGraphExec_t ge;
  e = cudaGraphInstantiate(&ge, g, 0);
  printf("instantiate %s\n", cudaGetErrorString(e));
  for (int rep = 0; rep < 3; ++rep) {
    cudaMemsetAsync(cnt, 0, 4, s);
    e = cudaGraphLaunch(ge, s);
    cudaStreamSynchronize(s);
    double hx; int hc;
    cudaMemcpy(&hx, x, 8, cudaMemcpyDeviceToHost); cudaMemcpy(&hc, cnt, 4, cudaMemcpyDeviceToHost);
    printf("launch %s count %d x %g\n", cudaGetErrorString(e), hc, hx);
  }
  return 0;
}
