// Standalone TMA probe: one CTA loads a 4-D box of fp64 with cp.async.bulk.tensor
// and writes it back, for a few descriptor configurations (debug tool).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void probe(const __grid_constant__ CUtensorMap map, int c0, int c1, int c2, int c3, int bytes, int mode, double* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(sa(&bar)), "r"(1) : "memory");
    if (mode & 1) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    else asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (mode & 2) asm volatile("prefetch.tensormap [%0];" :: "l"(reinterpret_cast<uint64_t>(&map)) : "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(sa(&bar)), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];"
                 :: "r"(sa(sm)), "l"(reinterpret_cast<uint64_t>(&map)), "r"(sa(&bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3) : "memory");
  }
  asm volatile("{\n\t.reg .pred P1;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra W_%=;\n}" :: "r"(sa(&bar)), "r"(0) : "memory");
  const double* s = reinterpret_cast<const double*>(sm);
  for (int i = threadIdx.x; i < bytes / 8; i += blockDim.x) out[i] = s[i];
}

int main(int argc, char** argv) {
  int cs = atoi(argv[1]);
  int S0 = 7, S1 = 6, S2 = 8, P0 = 8;
  long np = (long)P0 * S1 * S2;
  double* g; cudaMalloc(&g, np * 6 * 8);
  double* h = (double*)malloc(np * 6 * 8);
  for (long i = 0; i < np * 6; ++i) h[i] = (double)i;
  cudaMemcpy(g, h, np * 6 * 8, cudaMemcpyHostToDevice);
  double* out; cudaMalloc(&out, 1 << 20);
  cudaDriverEntryPointQueryResult q; void* fn;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto encode = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  alignas(64) CUtensorMap map;
  cuuint64_t dims[4] = {(cuuint64_t)S0, (cuuint64_t)S1, (cuuint64_t)S2, 6};
  cuuint64_t str[3] = {(cuuint64_t)P0 * 8, (cuuint64_t)P0 * S1 * 8, (cuuint64_t)np * 8};
  cuuint32_t box[4] = {34, 10, 1, 3};
  cuuint32_t es[4] = {1, 1, 1, 1};
  if (cs >= 10) { box[0] = 8; }  // box inside the tensor width
  CUresult r = encode(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, g, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  int bytes = box[0] * box[1] * box[2] * box[3] * 8;
  int c0 = 0, c1 = 0, c2 = 0, mode = 0;
  switch (cs % 10) {
    case 0: break;
    case 1: c0 = -1; c1 = -1; break;
    case 2: c2 = -1; break;
    case 3: mode = 1; break;
    case 4: mode = 2; break;
    case 5: c0 = -1; break;
    case 6: c1 = -1; break;
    case 7: c0 = -2; break;
    case 8: c0 = -2; c1 = -1; break;
    case 9: c0 = 2; break;
  }
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
  probe<<<1, 128, 100000>>>(map, c0, c1, c2, 3, bytes, mode, out);
  cudaError_t e = cudaDeviceSynchronize();
  double v[4];
  cudaMemcpy(v, out, 32, cudaMemcpyDeviceToHost);
  printf("case %d encode=%d launch=%s first=%g %g %g\n", cs, (int)r, cudaGetErrorString(e), v[0], v[1], v[2]);
  return 0;
}
