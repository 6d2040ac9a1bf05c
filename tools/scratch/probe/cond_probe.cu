// Probe: WHILE node whose body holds two IF nodes (handles created on the
// body graph) and a kernel that sets all three handles for the next
// iteration.  Prints the sequence of branches taken.
#include <cstdio>
#include <cuda_runtime.h>

__device__ int g_iter;
__device__ int g_log[64];

__global__ void k_a(int* log) { int i = g_iter; log[i] = 1; }
__global__ void k_b(int* log) { int i = g_iter; log[i] = 2; }
__global__ void k_book(cudaGraphConditionalHandle hw, cudaGraphConditionalHandle ha, cudaGraphConditionalHandle hb) {
  int i = ++g_iter;
  bool more = i < 6;
  bool use_a = (i % 2) == 0;
  cudaGraphSetConditional(hw, more ? 1u : 0u);
  cudaGraphSetConditional(ha, use_a ? 1u : 0u);
  cudaGraphSetConditional(hb, use_a ? 0u : 1u);
}
__global__ void k_init(cudaGraphConditionalHandle ha, cudaGraphConditionalHandle hb) {
  g_iter = 0;
  cudaGraphSetConditional(ha, 1u);
  cudaGraphSetConditional(hb, 0u);
}

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

int main() {
  int* log;
  CK(cudaMalloc(&log, 64 * sizeof(int)));
  CK(cudaMemset(log, 0, 64 * sizeof(int)));
  cudaGraph_t g;
  CK(cudaGraphCreate(&g, 0));
  cudaGraphConditionalHandle hw;
  CK(cudaGraphConditionalHandleCreate(&hw, g, 1, cudaGraphCondAssignDefault));
  cudaGraphNodeParams wp = {};
  wp.type = cudaGraphNodeTypeConditional;
  wp.conditional.handle = hw;
  wp.conditional.type = cudaGraphCondTypeWhile;
  wp.conditional.size = 1;
  cudaGraphNode_t wnode;
  // body
  CK(cudaGraphAddNode(&wnode, g, nullptr, 0, &wp));
  cudaGraph_t body = wp.conditional.phGraph_out[0];
  cudaGraphConditionalHandle ha, hb;
  CK(cudaGraphConditionalHandleCreate(&ha, body, 0, 0));
  CK(cudaGraphConditionalHandleCreate(&hb, body, 0, 0));
  cudaStream_t s;
  CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  // IF a
  cudaGraphNodeParams ip = {};
  ip.type = cudaGraphNodeTypeConditional;
  ip.conditional.handle = ha;
  ip.conditional.type = cudaGraphCondTypeIf;
  ip.conditional.size = 1;
  cudaGraphNode_t ia;
  CK(cudaGraphAddNode(&ia, body, nullptr, 0, &ip));
  CK(cudaStreamBeginCaptureToGraph(s, ip.conditional.phGraph_out[0], nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
  k_a<<<1, 1, 0, s>>>(log);
  cudaGraph_t tmp;
  CK(cudaStreamEndCapture(s, &tmp));
  cudaGraphNodeParams ip2 = {};
  ip2.type = cudaGraphNodeTypeConditional;
  ip2.conditional.handle = hb;
  ip2.conditional.type = cudaGraphCondTypeIf;
  ip2.conditional.size = 1;
  cudaGraphNode_t ib;
  CK(cudaGraphAddNode(&ib, body, &ia, 1, &ip2));
  CK(cudaStreamBeginCaptureToGraph(s, ip2.conditional.phGraph_out[0], nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
  k_b<<<1, 1, 0, s>>>(log);
  CK(cudaStreamEndCapture(s, &tmp));
  // book in the body after ib
  CK(cudaStreamBeginCaptureToGraph(s, body, &ib, nullptr, 1, cudaStreamCaptureModeThreadLocal));
  k_book<<<1, 1, 0, s>>>(hw, ha, hb);
  CK(cudaStreamEndCapture(s, &tmp));
  // init before the while node: set the IF handles from the parent graph
  cudaGraph_t pre;
  CK(cudaGraphCreate(&pre, 0));
  cudaGraphNode_t initnode;
  cudaKernelNodeParams kp = {};
  void* args[2] = {&ha, &hb};
  kp.func = (void*)k_init;
  kp.gridDim = dim3(1);
  kp.blockDim = dim3(1);
  kp.kernelParams = args;
  cudaError_t e1 = cudaGraphAddKernelNode(&initnode, g, nullptr, 0, &kp);
  printf("add init node in parent graph: %s\n", cudaGetErrorString(e1));
  if (e1 == cudaSuccess) CK(cudaGraphAddDependencies(g, &initnode, &wnode, 1));
  cudaGraphExec_t ex;
  cudaError_t e2 = cudaGraphInstantiate(&ex, g, 0);
  printf("instantiate: %s\n", cudaGetErrorString(e2));
  if (e2 != cudaSuccess) return 1;
  for (int rep = 0; rep < 2; rep++) {
    CK(cudaMemset(log, 0, 64 * sizeof(int)));
    CK(cudaGraphLaunch(ex, s));
    CK(cudaStreamSynchronize(s));
    int h[64];
    CK(cudaMemcpy(h, log, sizeof(h), cudaMemcpyDeviceToHost));
    printf("run %d:", rep);
    for (int i = 0; i < 8; i++) printf(" %d", h[i]);
    printf("\n");
  }
  return 0;
}
