// Minimal TMA / mbarrier probe: ./tma_probe <variant>  (one variant per process)
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>

__device__ __forceinline__ uint32_t sa(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void k(int variant, const __grid_constant__ CUtensorMap tm, int *out) {
  __shared__ __align__(128) int32_t buf[18 * 68 + 32];
  __shared__ __align__(8) uint64_t mb;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&mb)) : "memory");
    if (variant != 1) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (variant <= 1) {
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(&mb)) : "memory");
    } else {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&mb)), "r"(18 * 68 * 4) : "memory");
      int x = 0, y = 0;
      if (variant == 4) { x = -1; y = -1; }
      if (variant == 5) { x = -1; y = 0; }
      if (variant == 6) { x = 0; y = -1; }
      if (variant == 7) { x = 4; y = 3; }
      if (variant == 8) { x = -16; y = 0; }
      if (variant == 9) { x = -4; y = -1; }
      if (variant >= 5) variant = 2;
      if (variant == 2 || variant == 4)
        asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                     ::"r"(sa(buf)), "l"(reinterpret_cast<uint64_t>(&tm)), "r"(x), "r"(y), "r"(0), "r"(sa(&mb)) : "memory");
      else
        asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                     ::"r"(sa(buf)), "l"(reinterpret_cast<uint64_t>(&tm)), "r"(x), "r"(y), "r"(0), "r"(sa(&mb)) : "memory");
    }
  }
  asm volatile(
      "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(sa(&mb)),
      "r"(0)
      : "memory");
  __syncthreads();
  if (threadIdx.x == 0) { out[0] = buf[0]; out[1] = buf[69]; out[2] = buf[68 * 2 + 3]; }
}

int main(int argc, char **argv) {
  int variant = argc > 1 ? atoi(argv[1]) : 0;
  int nbx = argc > 2 ? atoi(argv[2]) : 8, nby = argc > 3 ? atoi(argv[3]) : 8;
  int32_t *g;
  cudaMalloc(&g, nbx * nby * 4);
  int32_t *h = (int32_t *)malloc(nbx * nby * 4);
  for (int i = 0; i < nbx * nby; i++) h[i] = 1000 + i;
  cudaMemcpy(g, h, nbx * nby * 4, cudaMemcpyHostToDevice);
  int *out;
  cudaMalloc(&out, 16);
  CUtensorMap tm;
  void *fn = nullptr;
  cudaDriverEntryPointQueryResult qr;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  cuuint64_t dims[3] = {(cuuint64_t)nbx, (cuuint64_t)nby, 1};
  cuuint64_t str[2] = {(cuuint64_t)nbx * 4, (cuuint64_t)nbx * nby * 4};
  cuuint32_t box[3] = {68, 18, 1}, es[3] = {1, 1, 1};
  CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_INT32, 3, g, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("variant %d nbx %d nby %d encode=%d fn=%p\n", variant, nbx, nby, (int)r, fn);
  k<<<1, 128>>>(variant, tm, out);
  cudaError_t e = cudaDeviceSynchronize();
  int o[3] = {0, 0, 0};
  cudaMemcpy(o, out, 12, cudaMemcpyDeviceToHost);
  printf("  -> %s  out=%d %d %d\n", cudaGetErrorString(e), o[0], o[1], o[2]);
  return e != cudaSuccess;
}
