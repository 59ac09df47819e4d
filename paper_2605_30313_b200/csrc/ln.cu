// Row LayerNorm for hidden layers (cfg3's FastSAC critics, SURVEY.md 8(a)/8(d);
// NOT in the reference, whose MLP is ELU-only, R:tensornet/mlp.py:27-28 -- the
// oracle is oracle/port.py ln_forward / ln_backward, pinned by finite
// differences).  Layer i with LN:  a = W x + b (GEMM, fp32 out),
// n = (a - mean) * rstd * g + beta, h = elu(n).
//   ln_fwd_reg    : warp per row, the row held in registers (float4 per lane
//                   per 128 columns, D <= 1024): one HBM read of a, one write
//                   of h, row stats (mean, rstd) kept for the backward
//   ln_bwd_reg    : dn = dL/dn (the ELU-gradient epilogue's output) ->
//                   da = rstd (dxh - mean(dxh) - xh mean(dxh xh)), dxh = dn g,
//                   written over dn; one read of a and dn per row.  Column
//                   sums dg = sum dn xh, dbeta = sum dn, colsum(da) (the
//                   layer's db) accumulate in registers over the warp's rows,
//                   are folded across the block's warps in fixed order through
//                   shared memory -> block partials for one ReduceJob
//                   (deterministic).  One 8-warp block per SM.
//   ln_fwd_kernel / ln_bwd_kernel : generic (any D / alignment) versions,
//                   three passes over the row, smem column accumulators
//   Algorithmic bytes per row: fwd 4D (a) + sizeof(TO) D (h) + 8; bwd 4D (a)
//                   + 2 sizeof(TD) D (dn in, da out) + 8.
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


// ---- register-resident row kernels (D <= 128 NV, D % 4 == 0, 16-B rows)
template <typename T>
struct V4;
template <>
struct V4<float> {
  static __device__ __forceinline__ float4 ld(const float* p) {
    return *reinterpret_cast<const float4*>(p);
  }
  static __device__ __forceinline__ void st(float* p, float4 v) {
    *reinterpret_cast<float4*>(p) = v;
  }
};
template <>
struct V4<__nv_bfloat16> {
  static __device__ __forceinline__ float4 ld(const __nv_bfloat16* p) {
    const uint2 u = *reinterpret_cast<const uint2*>(p);
    const float2 lo = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.x));
    const float2 hi = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.y));
    return make_float4(lo.x, lo.y, hi.x, hi.y);
  }
  static __device__ __forceinline__ void st(__nv_bfloat16* p, float4 v) {
    const __nv_bfloat162 lo = __floats2bfloat162_rn(v.x, v.y);
    const __nv_bfloat162 hi = __floats2bfloat162_rn(v.z, v.w);
    uint2 u;
    u.x = *reinterpret_cast<const uint32_t*>(&lo);
    u.y = *reinterpret_cast<const uint32_t*>(&hi);
    *reinterpret_cast<uint2*>(p) = u;
  }
};

constexpr int kRegWarps = 8;

template <int NV, typename TO>
__global__ void __launch_bounds__(kRegWarps * 32) ln_fwd_reg(
    const float* __restrict__ a, int64_t lda, int64_t M, int D, const float* __restrict__ g,
    const float* __restrict__ beta, float* __restrict__ stats, TO* __restrict__ h, int64_t ldh,
    int ones_col) {
  pdl_trigger();
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * kRegWarps;
  float4 gv[NV], bv[NV];
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    const int c = 4 * lane + 128 * j;
    gv[j] = c < D ? V4<float>::ld(g + c) : make_float4(0.f, 0.f, 0.f, 0.f);
    bv[j] = c < D ? V4<float>::ld(beta + c) : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  const float inv_d = 1.f / D;
  for (int64_t r = (int64_t)blockIdx.x * kRegWarps + (threadIdx.x >> 5); r < M; r += nw) {
    const float* ar = a + r * lda;
    float4 x[NV];
    float s = 0.f;
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      const int c = 4 * lane + 128 * j;
      x[j] = c < D ? V4<float>::ld(ar + c) : make_float4(0.f, 0.f, 0.f, 0.f);
      s += (x[j].x + x[j].y) + (x[j].z + x[j].w);
    }
    const float mean = warp_sum(s) * inv_d;
    float q = 0.f;
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      const int c = 4 * lane + 128 * j;
      if (c < D) {
        const float d0 = x[j].x - mean, d1 = x[j].y - mean, d2 = x[j].z - mean,
                    d3 = x[j].w - mean;
        q += (d0 * d0 + d1 * d1) + (d2 * d2 + d3 * d3);
      }
    }
    const float rstd = rsqrtf(warp_sum(q) * inv_d + kLnEps);
    TO* hr = h + r * ldh;
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      const int c = 4 * lane + 128 * j;
      if (c < D) {
        float4 o;
        o.x = elu_f((x[j].x - mean) * rstd * gv[j].x + bv[j].x);
        o.y = elu_f((x[j].y - mean) * rstd * gv[j].y + bv[j].y);
        o.z = elu_f((x[j].z - mean) * rstd * gv[j].z + bv[j].z);
        o.w = elu_f((x[j].w - mean) * rstd * gv[j].w + bv[j].w);
        V4<TO>::st(hr + c, o);
      }
    }
    if (lane == 0) {
      reinterpret_cast<float2*>(stats)[r] = make_float2(mean, rstd);
      if (ones_col >= 0) st1<TO>(hr + ones_col, 1.f);
    }
  }
}

// part: [gridDim.x][3][D] = dg | dbeta | colsum(da); smem [3][D]
template <int NV, typename TD>
__global__ void __launch_bounds__(kRegWarps * 32, 1) ln_bwd_reg(
    TD* __restrict__ dn, int64_t ldd, const float* __restrict__ a, int64_t lda,
    const float* __restrict__ stats, const float* __restrict__ g, int64_t M, int D,
    float* __restrict__ part) {
  extern __shared__ float4 red4[];
  pdl_trigger();
  pdl_wait();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  float4 gv[NV], ag[NV], ab[NV], aa[NV];
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    const int c = 4 * lane + 128 * j;
    gv[j] = c < D ? V4<float>::ld(g + c) : make_float4(0.f, 0.f, 0.f, 0.f);
    ag[j] = ab[j] = aa[j] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  const float inv_d = 1.f / D;
  const int64_t nw = (int64_t)gridDim.x * kRegWarps;
  for (int64_t r = (int64_t)blockIdx.x * kRegWarps + w; r < M; r += nw) {
    TD* dr = dn + r * ldd;
    const float* ar = a + r * lda;
    const float2 st = reinterpret_cast<const float2*>(stats)[r];
    float4 xh[NV], dv[NV];
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      const int c = 4 * lane + 128 * j;
      if (c < D) {
        const float4 x = V4<float>::ld(ar + c);
        dv[j] = V4<TD>::ld(dr + c);
        xh[j] = make_float4((x.x - st.x) * st.y, (x.y - st.x) * st.y, (x.z - st.x) * st.y,
                            (x.w - st.x) * st.y);
        const float e0 = dv[j].x * gv[j].x, e1 = dv[j].y * gv[j].y, e2 = dv[j].z * gv[j].z,
                    e3 = dv[j].w * gv[j].w;
        s1 += (e0 + e1) + (e2 + e3);
        s2 += (e0 * xh[j].x + e1 * xh[j].y) + (e2 * xh[j].z + e3 * xh[j].w);
      } else {
        xh[j] = dv[j] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
    const float m1 = warp_sum(s1) * inv_d, m2 = warp_sum(s2) * inv_d;
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      const int c = 4 * lane + 128 * j;
      if (c < D) {
        float4 da;
        da.x = st.y * (dv[j].x * gv[j].x - m1 - xh[j].x * m2);
        da.y = st.y * (dv[j].y * gv[j].y - m1 - xh[j].y * m2);
        da.z = st.y * (dv[j].z * gv[j].z - m1 - xh[j].z * m2);
        da.w = st.y * (dv[j].w * gv[j].w - m1 - xh[j].w * m2);
        V4<TD>::st(dr + c, da);
        ag[j].x += dv[j].x * xh[j].x;
        ag[j].y += dv[j].y * xh[j].y;
        ag[j].z += dv[j].z * xh[j].z;
        ag[j].w += dv[j].w * xh[j].w;
        ab[j].x += dv[j].x;
        ab[j].y += dv[j].y;
        ab[j].z += dv[j].z;
        ab[j].w += dv[j].w;
        aa[j].x += da.x;
        aa[j].y += da.y;
        aa[j].z += da.z;
        aa[j].w += da.w;
      }
    }
  }
  // fold the warps' column sums in warp order (deterministic)
  const int D4 = D >> 2;
  for (int k = 0; k < kRegWarps; ++k) {
    if (w == k) {
#pragma unroll
      for (int j = 0; j < NV; ++j) {
        const int c4 = lane + 32 * j;
        if (c4 < D4) {
          if (k == 0) {
            red4[c4] = ag[j];
            red4[D4 + c4] = ab[j];
            red4[2 * D4 + c4] = aa[j];
          } else {
            float4 t = red4[c4];
            red4[c4] = make_float4(t.x + ag[j].x, t.y + ag[j].y, t.z + ag[j].z, t.w + ag[j].w);
            t = red4[D4 + c4];
            red4[D4 + c4] =
                make_float4(t.x + ab[j].x, t.y + ab[j].y, t.z + ab[j].z, t.w + ab[j].w);
            t = red4[2 * D4 + c4];
            red4[2 * D4 + c4] =
                make_float4(t.x + aa[j].x, t.y + aa[j].y, t.z + aa[j].z, t.w + aa[j].w);
          }
        }
      }
    }
    __syncthreads();
  }
  float4* pz = reinterpret_cast<float4*>(part + (int64_t)blockIdx.x * 3 * D);
  for (int c = threadIdx.x; c < 3 * D4; c += blockDim.x) pz[c] = red4[c];
}

int ln_blocks(int64_t M) {
  int64_t b = ceil_div(M, kLnWarps * 8);
  return (int)(b > 2 * kNumSMs ? 2 * kNumSMs : (b < 1 ? 1 : b));
}

}  // namespace

int ln_part_floats(int64_t M, int D) { return ln_blocks(M) * 3 * ceil_div(D, 4) * 4; }

namespace {
bool al(const void* p, int bytes) { return ((uintptr_t)p & (bytes - 1)) == 0; }
int reg_nv(int D) {
  if (D > 1024 || D % 4) return 0;
  return D <= 128 ? 1 : D <= 256 ? 2 : D <= 512 ? 4 : 8;
}

template <typename TO>
int fwd_reg(int nv, unsigned blocks, const float* a, int64_t lda, int64_t M, int D, const float* g,
            const float* beta, float* stats, TO* h, int64_t ldh, int ones_col, cudaStream_t s) {
  const dim3 gr(blocks), bl(kRegWarps * 32);
  switch (nv) {
    case 1:
      return launch_pdl("ln_fwd_reg", ln_fwd_reg<1, TO>, gr, bl, 0, s, a, lda, M, D, g, beta,
                        stats, h, ldh, ones_col);
    case 2:
      return launch_pdl("ln_fwd_reg", ln_fwd_reg<2, TO>, gr, bl, 0, s, a, lda, M, D, g, beta,
                        stats, h, ldh, ones_col);
    case 4:
      return launch_pdl("ln_fwd_reg", ln_fwd_reg<4, TO>, gr, bl, 0, s, a, lda, M, D, g, beta,
                        stats, h, ldh, ones_col);
    default:
      return launch_pdl("ln_fwd_reg", ln_fwd_reg<8, TO>, gr, bl, 0, s, a, lda, M, D, g, beta,
                        stats, h, ldh, ones_col);
  }
}

template <typename TD>
int bwd_reg(int nv, unsigned blocks, TD* dn, int64_t ldd, const float* a, int64_t lda,
            const float* stats, const float* g, int64_t M, int D, float* part, cudaStream_t s) {
  const dim3 gr(blocks), bl(kRegWarps * 32);
  const size_t sm = (size_t)3 * D * sizeof(float);
  switch (nv) {
    case 1:
      return launch_pdl("ln_bwd_reg", ln_bwd_reg<1, TD>, gr, bl, sm, s, dn, ldd, a, lda, stats, g,
                        M, D, part);
    case 2:
      return launch_pdl("ln_bwd_reg", ln_bwd_reg<2, TD>, gr, bl, sm, s, dn, ldd, a, lda, stats, g,
                        M, D, part);
    case 4:
      return launch_pdl("ln_bwd_reg", ln_bwd_reg<4, TD>, gr, bl, sm, s, dn, ldd, a, lda, stats, g,
                        M, D, part);
    default:
      return launch_pdl("ln_bwd_reg", ln_bwd_reg<8, TD>, gr, bl, sm, s, dn, ldd, a, lda, stats, g,
                        M, D, part);
  }
}
}  // namespace

int ln_forward(const float* a, int64_t lda, int64_t M, int D, const float* g, const float* beta,
               float* stats, void* h, int64_t ldh, int ones_col, int dtype, cudaStream_t s) {
  if (M == 0) return UL_OK;
  const int nv = reg_nv(D);
  const int hb = dtype == kBf16 ? 8 : 16;
  if (nv && lda % 4 == 0 && ldh % 4 == 0 && al(a, 16) && al(g, 16) && al(beta, 16) &&
      al(stats, 8) && al(h, hb)) {
    int64_t blocks = ceil_div(M, kRegWarps);
    blocks = blocks > 4 * kNumSMs ? 4 * kNumSMs : blocks;
    if (dtype == kBf16)
      return fwd_reg(nv, (unsigned)blocks, a, lda, M, D, g, beta, stats,
                     reinterpret_cast<__nv_bfloat16*>(h), ldh, ones_col, s);
    return fwd_reg(nv, (unsigned)blocks, a, lda, M, D, g, beta, stats, reinterpret_cast<float*>(h),
                   ldh, ones_col, s);
  }
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
  int nb = ln_blocks(M);
  const int Dp = (int)(ceil_div(D, 4) * 4);
  const size_t sm = (size_t)kLnWarps * 3 * D * sizeof(float);
  static bool attr[2] = {false, false};
  const int nv = reg_nv(D);
  const int db = dtype == kBf16 ? 8 : 16;
  if (nv && lda % 4 == 0 && ldd % 4 == 0 && al(a, 16) && al(g, 16) && al(stats, 8) &&
      al(dn, db) && al(part, 16)) {
    int64_t b = ceil_div(M, kRegWarps * 4);
    nb = (int)(b > kNumSMs ? kNumSMs : b);
    if (dtype == kBf16)
      UL_TRY(bwd_reg(nv, nb, reinterpret_cast<__nv_bfloat16*>(dn), ldd, a, lda, stats, g, M, D,
                     part, s));
    else
      UL_TRY(bwd_reg(nv, nb, reinterpret_cast<float*>(dn), ldd, a, lda, stats, g, M, D, part, s));
  } else if (dtype == kBf16) {
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
