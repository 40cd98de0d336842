// Per-step floor of a chain of dependent launches on this GPU: K empty (or
// near-empty) kernels captured in one CUDA graph, with and without
// programmatic dependent launch, timed over graph replays.  The decode step
// (one launch per step) cannot be faster than this.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/pdl_floor tools/pdl_floor.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void step_kernel(int* buf, int grid_work) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0) asm volatile("griddepcontrol.launch_dependents;");
  if (grid_work && threadIdx.x == 0) atomicAdd(buf + blockIdx.x, 1);
}

static float run(int blocks, int threads, bool pdl, int K, int* buf) {
  cudaStream_t s;
  cudaStreamCreate(&s);
  cudaGraph_t g;
  cudaGraphExec_t ge;
  cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
  for (int k = 0; k < K; ++k) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(blocks);
    cfg.blockDim = dim3(threads);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    cudaLaunchKernelEx(&cfg, step_kernel, buf, 1);
  }
  cudaStreamEndCapture(s, &g);
  cudaGraphInstantiate(&ge, g, 0);
  for (int i = 0; i < 5; ++i) cudaGraphLaunch(ge, s);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a, s);
  const int R = 50;
  for (int i = 0; i < R; ++i) cudaGraphLaunch(ge, s);
  cudaEventRecord(b, s);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  cudaGraphExecDestroy(ge);
  cudaGraphDestroy(g);
  cudaStreamDestroy(s);
  return ms * 1e3f / (R * K);
}

int main() {
  int* buf;
  cudaMalloc(&buf, 1 << 20);
  for (int blocks : {1, 72, 144})
    for (int pdl = 0; pdl < 2; ++pdl)
      printf("blocks %3d threads 256 pdl %d: %.2f us per step\n", blocks, pdl,
             run(blocks, 256, pdl, 20, buf));
  return 0;
}
