// Standalone probe: does a 3-D fp64 TMA box load work with (a) zero and (b) negative
// start coordinates, (c) odd inner box (18 doubles)?  Prints the first values.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdint.h>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void k(const __grid_constant__ CUtensorMap m, int c0, int c1, int c2, double* out, int n) {
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* bar = (uint64_t*)(smem + 65536);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(sa(bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(sa(bar)), "r"(n * 8) : "memory");
    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
      :: "r"(sa(smem)), "l"((uint64_t)&m), "r"(c0), "r"(c1), "r"(c2), "r"(sa(bar)) : "memory");
  }
  uint32_t done = 0;
  do { asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0,1,0,p; }" : "=r"(done) : "r"(sa(bar)) : "memory"); } while (!done);
  for (int i = threadIdx.x; i < n; i += blockDim.x) out[i] = ((double*)smem)[i];
}

int main() {
  const int K = 80, W = 258, H = 281;
  size_t n = (size_t)K * W * H;
  double* h = (double*)malloc(n * 8);
  for (size_t i = 0; i < n; ++i) h[i] = (double)i;
  double *d, *o; cudaMalloc(&d, n * 8); cudaMalloc(&o, 1 << 20);
  cudaMemcpy(d, h, n * 8, cudaMemcpyHostToDevice);
  void* fn; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  CUtensorMap m;
  cuuint64_t dims[3] = {K, W, H}, str[2] = {K * 8, (cuuint64_t)W * K * 8};
  cuuint32_t box[3] = {18, 18, 6}, es[3] = {1, 1, 1};
  CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d\n", (int)r);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 128);
  int nb = 18 * 18 * 6;
  int cs[3][3] = {{0, 0, 0}, {16, 0, 0}, {-1, 0, 0}};
  for (int t = 0; t < 3; ++t) {
    k<<<1, 128, 65536 + 128>>>(m, cs[t][0], cs[t][1], cs[t][2], o, nb);
    cudaError_t e = cudaDeviceSynchronize();
    double hb[4]; cudaMemcpy(hb, o, 32, cudaMemcpyDeviceToHost);
    printf("coords (%d,%d,%d): %s  first %g %g %g\n", cs[t][0], cs[t][1], cs[t][2], cudaGetErrorString(e), hb[0], hb[1], hb[2]);
    if (e) return 1;
  }
  return 0;
}
