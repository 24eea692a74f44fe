// Launch-boundary cost on this GPU: a CUDA graph of N back-to-back small kernels (persistent
// sized grids like the phase kernels), with and without programmatic dependent launch (PDL).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o launch_gap launch_gap.cu && ./launch_gap
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_small(unsigned *p, int pdl) {
  if (pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0) atomicAdd(&p[blockIdx.x & 1023], 1u);
  if (pdl) asm volatile("griddepcontrol.launch_dependents;");
}

int main() {
  unsigned *p;
  cudaMalloc(&p, 4096 * 4);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  const int N = 462;
  for (int grid : {148, 444, 1184}) {
    for (int pdl = 0; pdl < 2; pdl++) {
      cudaGraph_t g;
      cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
      for (int i = 0; i < N; i++) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = grid;
        cfg.blockDim = 256;
        cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = pdl ? 1 : 0;
        cudaLaunchKernelEx(&cfg, k_small, p, pdl);
      }
      cudaStreamEndCapture(s, &g);
      cudaGraphExec_t ge;
      if (cudaGraphInstantiate(&ge, g, 0) != cudaSuccess) { printf("instantiate failed\n"); return 1; }
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaGraphLaunch(ge, s);
      cudaEventRecord(e0, s);
      for (int r = 0; r < 10; r++) cudaGraphLaunch(ge, s);
      cudaEventRecord(e1, s);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      printf("grid %4d pdl %d: %.2f us per kernel (%d kernels)\n", grid, pdl, 1e3f * ms / (10 * N), N);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
