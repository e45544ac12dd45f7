// Feasibility probe: a conditional WHILE graph node whose body is captured
// from a stream (kernels + a PDL launch), the loop condition set on the
// device. nvcc -gencode arch=compute_100a,code=sm_100a tools/cond_while_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_work(int* c) { atomicAdd(c, 1); }
__global__ void k_cond(cudaGraphConditionalHandle h, int* c, int limit) {
  cudaGraphSetConditional(h, *c < limit ? 1 : 0);
}

int main() {
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  int* c;
  cudaMalloc(&c, sizeof(int));
  cudaMemset(c, 0, sizeof(int));
  cudaGraph_t parent;
  cudaGraphCreate(&parent, 0);
  cudaGraphConditionalHandle h;
  if (cudaGraphConditionalHandleCreate(&h, parent, 1, cudaGraphCondAssignDefault) != cudaSuccess) { printf("handle fail\n"); return 1; }
  cudaGraphNodeParams cp = {};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = h;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t node;
  if (cudaGraphAddNode(&node, parent, nullptr, 0, &cp) != cudaSuccess) { printf("add fail\n"); return 1; }
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  if (cudaStreamBeginCaptureToGraph(st, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal) != cudaSuccess) { printf("cap fail\n"); return 1; }
  k_work<<<1, 1, 0, st>>>(c);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(1); cfg.blockDim = dim3(1); cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at; cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k_work, c);
  k_cond<<<1, 1, 0, st>>>(h, c, 100);
  cudaGraph_t out;
  cudaError_t e = cudaStreamEndCapture(st, &out);
  printf("end capture: %s\n", cudaGetErrorString(e));
  cudaGraphExec_t ex;
  e = cudaGraphInstantiate(&ex, parent, 0);
  printf("instantiate: %s\n", cudaGetErrorString(e));
  for (int rep = 0; rep < 2; ++rep) {
    cudaMemsetAsync(c, 0, sizeof(int), st);
    e = cudaGraphLaunch(ex, st);
    cudaStreamSynchronize(st);
    int hc = 0;
    cudaMemcpy(&hc, c, sizeof(int), cudaMemcpyDeviceToHost);
    printf("launch %d: %s, counter %d (expect 100)\n", rep, cudaGetErrorString(e), hc);
  }
  return 0;
}
