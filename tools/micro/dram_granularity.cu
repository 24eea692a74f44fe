// DRAM bytes per isolated 4-B load: each thread loads one word from its own 1-KB region (no
// two loads share a 128-B line) of a 4 GiB buffer; ncu's dram__bytes_read.sum / loads gives
// the effective DRAM access granularity of scattered reads.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dram_granularity dram_granularity.cu
//   ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum ./dram_granularity
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_touch(const int *__restrict__ buf, size_t n_regions, int stride_words, int *out, int mode) {
  int acc = 0;
  for (size_t r = blockIdx.x * (size_t)blockDim.x + threadIdx.x; r < n_regions; r += (size_t)gridDim.x * blockDim.x) {
    const int *p = buf + r * stride_words;
    int v;
    if (mode == 0) v = __ldcs(p);
    else if (mode == 1) v = __ldg(p);
    else if (mode == 2) v = __ldcg(p);
    else if (mode == 3) asm volatile("ld.global.L2::64B.b32 %0, [%1];" : "=r"(v) : "l"(p));
    else if (mode == 4) asm volatile("ld.global.L2::128B.b32 %0, [%1];" : "=r"(v) : "l"(p));
    else if (mode == 5) asm volatile("ld.global.nc.L2::64B.b32 %0, [%1];" : "=r"(v) : "l"(p));
    else asm volatile("ld.global.cs.L2::64B.b32 %0, [%1];" : "=r"(v) : "l"(p));
    acc += v;
  }
  if (acc == 0x12345678) out[0] = acc;
}

int main() {
  const size_t bytes = 4ull << 30;
  int *buf, *out;
  cudaMalloc(&buf, bytes);
  cudaMalloc(&out, 4);
  cudaMemset(buf, 1, bytes);
  const int stride_words = 256;  // 1 KB apart
  const size_t n = bytes / (stride_words * 4);
  for (int mode = 0; mode < 7; mode++) {
    k_touch<<<148 * 16, 256>>>(buf, n, stride_words, out, mode);
    cudaDeviceSynchronize();
  }
  printf("loads per launch: %zu (%s)\n", n, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
