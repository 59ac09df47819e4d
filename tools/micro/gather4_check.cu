// Checks TMA tile::gather4 against a plain tile load of pre-permuted rows
// (same 128B-swizzled shared-memory image?).  Diagnostics only.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdint>
#include <vector>

__device__ __forceinline__ void wait_bar(uint32_t b, uint32_t ph) {
  asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}\n" ::"r"(b), "r"(ph) : "memory");
}
__global__ void k(const __grid_constant__ CUtensorMap g, const __grid_constant__ CUtensorMap t,
                  const int* rows, int nrows, uint8_t* out1, uint8_t* out2) {
  __shared__ __align__(1024) uint8_t s1[16384], s2[16384];
  __shared__ __align__(8) uint64_t bar[2];
  const uint32_t b0 = (uint32_t)__cvta_generic_to_shared(&bar[0]), b1 = (uint32_t)__cvta_generic_to_shared(&bar[1]);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b0));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b1));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b0), "r"(nrows * 128));
    for (int i = 0; i < nrows; i += 4) {
      uint32_t d = (uint32_t)__cvta_generic_to_shared(s1 + i * 128);
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
                   :: "r"(d), "l"(&g), "r"(0), "r"(rows[i]), "r"(rows[i + 1]), "r"(rows[i + 2]), "r"(rows[i + 3]), "r"(b0) : "memory");
    }
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b1), "r"(nrows * 128));
    uint32_t d2 = (uint32_t)__cvta_generic_to_shared(s2);
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                 :: "r"(d2), "l"(&t), "r"(0), "r"(0), "r"(b1) : "memory");
  }
  wait_bar(b0, 0);
  wait_bar(b1, 0);
  for (int i = threadIdx.x; i < nrows * 128; i += blockDim.x) { out1[i] = s1[i]; out2[i] = s2[i]; }
}

int main() {
  const int R = 64, C = 64, NR = 32;  // source rows, bf16 columns (128 B), gathered rows
  std::vector<uint16_t> h(R * C), hp(NR * C);
  std::vector<int> rows(NR);
  for (int i = 0; i < R * C; ++i) h[i] = (uint16_t)(i * 7 + 3);
  for (int i = 0; i < NR; ++i) rows[i] = (i * 37 + 11) % R;
  rows[NR - 1] = R + 5;  // out of range -> zero fill
  for (int i = 0; i < NR; ++i)
    for (int c = 0; c < C; ++c) hp[i * C + c] = rows[i] < R ? h[rows[i] * C + c] : 0;
  void *d, *dp; int* dr; uint8_t *o1, *o2;
  cudaMalloc(&d, h.size() * 2); cudaMalloc(&dp, hp.size() * 2); cudaMalloc(&dr, NR * 4);
  cudaMalloc(&o1, NR * 128); cudaMalloc(&o2, NR * 128);
  cudaMemcpy(d, h.data(), h.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dp, hp.data(), hp.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dr, rows.data(), NR * 4, cudaMemcpyHostToDevice);
  PFN_cuTensorMapEncodeTiled_v12000 enc;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  CUtensorMap g, t;
  cuuint64_t dims[2] = {(cuuint64_t)C, (cuuint64_t)R}, dimsp[2] = {(cuuint64_t)C, (cuuint64_t)NR};
  cuuint64_t st[1] = {(cuuint64_t)C * 2};
  cuuint32_t boxg[2] = {64, 1}, boxt[2] = {64, (cuuint32_t)NR}, es[2] = {1, 1};
  CUresult r1 = enc(&g, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d, dims, st, boxg, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  CUresult r2 = enc(&t, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dp, dimsp, st, boxt, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d %d\n", (int)r1, (int)r2);
  k<<<1, 128>>>(g, t, dr, NR, o1, o2);
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<uint8_t> a(NR * 128), b(NR * 128);
  cudaMemcpy(a.data(), o1, NR * 128, cudaMemcpyDeviceToHost);
  cudaMemcpy(b.data(), o2, NR * 128, cudaMemcpyDeviceToHost);
  int diff = 0;
  for (int i = 0; i < NR * 128; ++i) diff += a[i] != b[i];
  printf("err %s, differing bytes %d of %d\n", cudaGetErrorString(e), diff, NR * 128);
  return 0;
}
