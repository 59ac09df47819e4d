// Microbenchmark: tcgen05.ld (32x32b.x16) throughput per SM with 4..16 warps
// reading a 512-column TMEM allocation.  Diagnostics only (not product code).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(576, 1) tmem_rd(int nw_active, int iters, unsigned long long* out, float* sink) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(&slot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = slot;
  float acc = 0.f;
  unsigned long long t0 = clock64();
  if (warp < nw_active) {
    const int quarter = warp & 3, slice = warp >> 2;
    const uint32_t base = tmem + ((uint32_t)(quarter * 32) << 16);
    for (int it = 0; it < iters; ++it) {
      for (int c = slice * 16; c < 512; c += 16 * ((nw_active + 3) / 4)) {
        uint32_t r[16];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
              "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
            : "r"(base + (uint32_t)c));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int i = 0; i < 16; ++i) acc += __uint_as_float(r[i]);
      }
    }
  }
  __syncthreads();
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = t1 - t0;
  if (acc == 123.f) sink[threadIdx.x] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

int main() {
  unsigned long long* d; float* s;
  cudaMalloc(&d, 8); cudaMalloc(&s, 4096);
  for (int nw : {4, 8, 16}) {
    const int iters = 200;
    tmem_rd<<<148, 576>>>(nw, iters, d, s);
    cudaDeviceSynchronize();
    tmem_rd<<<148, 576>>>(nw, iters, d, s);
    unsigned long long c; cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
    double bytes = 128.0 * 512 * 4 * iters;  // whole 128 x 512 fp32 TMEM per iteration
    printf("warps %2d: %llu clk for %.0f KB -> %.1f B/clk/SM  (err %s)\n", nw, c, bytes / 1024, bytes / c,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
