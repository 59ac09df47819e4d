// Row LayerNorm for hidden layers (cfg3's FastSAC critics, SURVEY.md 8(a)/8(d);
// NOT in the reference, whose MLP is ELU-only, R:tensornet/mlp.py:27-28 -- the
// oracle is oracle/port.py ln_forward / ln_backward, pinned by finite
// differences).  Layer i with LN:  a = W x + b (GEMM, fp32 out),
// n = (a - mean) * rstd * g + beta, h = elu(n).
//   ln_fwd_kernel : warp per row, three passes over the L1-resident row
//                   (mean, centred variance, normalise + ELU + store), row
//                   stats kept for the backward
//   ln_bwd_kernel : dn = dL/dn (the ELU-gradient epilogue's output) ->
//                   da = rstd (dxh - mean(dxh) - xh mean(dxh xh)), dxh = dn g,
//                   written over dn; per-warp smem column accumulators of
//                   dg = sum dn xh, dbeta = sum dn and colsum(da) (the layer's
//                   db), combined per block in fixed warp order -> block
//                   partials for one ReduceJob (deterministic)
#include <cuda_bf16.h>

#include "internal.cuh"

namespace ul {
namespace {

constexpr int kLnWarps = 4;
constexpr float kLnEps = 1e-5f;

template <typename T>
__device__ __forceinline__ float ld1(const T* p);
template <>
__device__ __forceinline__ float ld1<float>(const float* p) {
  return *p;
}
template <>
__device__ __forceinline__ float ld1<__nv_bfloat16>(const __nv_bfloat16* p) {
  return __bfloat162float(*p);
}
template <typename T>
__device__ __forceinline__ void st1(T* p, float v);
template <>
__device__ __forceinline__ void st1<float>(float* p, float v) {
  *p = v;
}
template <>
__device__ __forceinline__ void st1<__nv_bfloat16>(__nv_bfloat16* p, float v) {
  *p = __float2bfloat16_rn(v);
}

template <typename TO>
__global__ void __launch_bounds__(256) ln_fwd_kernel(const float* __restrict__ a, int64_t lda,
                                                     int64_t M, int D, const float* __restrict__ g,
                                                     const float* __restrict__ beta,
                                                     float* __restrict__ stats, TO* __restrict__ h,
                                                     int64_t ldh, int ones_col) {
  pdl_trigger();
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < M; r += nw) {
    const float* ar = a + r * lda;
    float s = 0.f;
    for (int c = lane; c < D; c += 32) s += ar[c];
    const float mean = warp_sum(s) / D;
    float q = 0.f;
    for (int c = lane; c < D; c += 32) {
      const float d = ar[c] - mean;
      q += d * d;
    }
    const float rstd = rsqrtf(warp_sum(q) / D + kLnEps);
    TO* hr = h + r * ldh;
    for (int c = lane; c < D; c += 32) {
      const float n = (ar[c] - mean) * rstd * g[c] + beta[c];
      st1<TO>(hr + c, elu_f(n));
    }
    if (lane == 0) {
      stats[2 * r] = mean;
      stats[2 * r + 1] = rstd;
      if (ones_col >= 0) st1<TO>(hr + ones_col, 1.f);
    }
  }
}

// part: [gridDim.x][3][D] = dg | dbeta | colsum(da)
template <typename TD>
__global__ void __launch_bounds__(kLnWarps * 32) ln_bwd_kernel(
    TD* __restrict__ dn, int64_t ldd, const float* __restrict__ a, int64_t lda,
    const float* __restrict__ stats, const float* __restrict__ g, int64_t M, int D,
    float* __restrict__ part) {
  extern __shared__ float acc[];  // [kLnWarps][3][D]
  pdl_trigger();
  pdl_wait();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  float* my = acc + (int64_t)w * 3 * D;
  for (int c = lane; c < 3 * D; c += 32) my[c] = 0.f;
  __syncwarp();
  const int64_t nw = (int64_t)gridDim.x * kLnWarps;
  for (int64_t r = (int64_t)blockIdx.x * kLnWarps + w; r < M; r += nw) {
    TD* dr = dn + r * ldd;
    const float* ar = a + r * lda;
    const float mean = stats[2 * r], rstd = stats[2 * r + 1];
    float s1 = 0.f, s2 = 0.f;
    for (int c = lane; c < D; c += 32) {
      const float xh = (ar[c] - mean) * rstd;
      const float dx = ld1<TD>(dr + c) * g[c];
      s1 += dx;
      s2 += dx * xh;
    }
    const float m1 = warp_sum(s1) / D, m2 = warp_sum(s2) / D;
    for (int c = lane; c < D; c += 32) {
      const float xh = (ar[c] - mean) * rstd;
      const float dnv = ld1<TD>(dr + c);
      const float da = rstd * (dnv * g[c] - m1 - xh * m2);
      st1<TD>(dr + c, da);
      my[c] += dnv * xh;
      my[D + c] += dnv;
      my[2 * D + c] += da;
    }
  }
  __syncthreads();
  float* pz = part + (int64_t)blockIdx.x * 3 * D;
  for (int c = threadIdx.x; c < 3 * D; c += blockDim.x) {
    float t = 0.f;
    for (int k = 0; k < kLnWarps; ++k) t += acc[(int64_t)k * 3 * D + c];
    pz[c] = t;
  }
}

int ln_blocks(int64_t M) {
  int64_t b = ceil_div(M, kLnWarps * 8);
  return (int)(b > 2 * kNumSMs ? 2 * kNumSMs : (b < 1 ? 1 : b));
}

}  // namespace

int ln_part_floats(int64_t M, int D) { return ln_blocks(M) * 3 * ceil_div(D, 4) * 4; }

int ln_forward(const float* a, int64_t lda, int64_t M, int D, const float* g, const float* beta,
               float* stats, void* h, int64_t ldh, int ones_col, int dtype, cudaStream_t s) {
  if (M == 0) return UL_OK;
  int64_t blocks = ceil_div(M, 8);
  blocks = blocks > 8 * kNumSMs ? 8 * kNumSMs : blocks;
  if (dtype == kBf16)
    return launch_pdl("ln_fwd_kernel", ln_fwd_kernel<__nv_bfloat16>, dim3((unsigned)blocks),
                      dim3(256), 0, s, a, lda, M, D, g, beta, stats,
                      reinterpret_cast<__nv_bfloat16*>(h), ldh, ones_col);
  return launch_pdl("ln_fwd_kernel", ln_fwd_kernel<float>, dim3((unsigned)blocks), dim3(256), 0,
                    s, a, lda, M, D, g, beta, stats, reinterpret_cast<float*>(h), ldh, ones_col);
}

// dn (dtype rows, ld ldd) -> da in place; partials for the ReduceJob in
// *job (segments dg | dbeta | colsum(da), each D long, padded to 4).
int ln_backward(void* dn, int64_t ldd, const float* a, int64_t lda, const float* stats,
                const float* g, int64_t M, int D, float* part, int dtype, float* gg, float* gbeta,
                float* gb, ReduceJob* job, cudaStream_t s) {
  if (M == 0) return UL_OK;
  const int nb = ln_blocks(M);
  const int Dp = (int)(ceil_div(D, 4) * 4);
  const size_t sm = (size_t)kLnWarps * 3 * D * sizeof(float);
  static bool attr[2] = {false, false};
  if (dtype == kBf16) {
    if (!attr[1]) {
      UL_CUDA(cudaFuncSetAttribute(ln_bwd_kernel<__nv_bfloat16>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
      attr[1] = true;
    }
    UL_TRY(launch_pdl("ln_bwd_kernel", ln_bwd_kernel<__nv_bfloat16>, dim3(nb), dim3(kLnWarps * 32),
                      sm, s, reinterpret_cast<__nv_bfloat16*>(dn), ldd, a, lda, stats, g, M, D,
                      part));
  } else {
    if (!attr[0]) {
      UL_CUDA(cudaFuncSetAttribute(ln_bwd_kernel<float>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
      attr[0] = true;
    }
    UL_TRY(launch_pdl("ln_bwd_kernel", ln_bwd_kernel<float>, dim3(nb), dim3(kLnWarps * 32), sm, s,
                      reinterpret_cast<float*>(dn), ldd, a, lda, stats, g, M, D, part));
  }
  // block partials are [3][D] rows; expose them as one segment job of
  // length 3*D (the reduction kernel wants len % 4 == 0: D % 4 == 0 here)
  (void)Dp;
  *job = ReduceJob{};
  job->src = part;
  job->nz = nb;
  job->kind = 1;
  job->len = 3 * (int64_t)D;
  job->n0 = D;
  job->o0 = gg;
  job->n1 = D;
  job->o1 = gbeta;
  job->n2 = gb ? D : 0;
  job->o2 = gb;
  return UL_OK;
}

}  // namespace ul
