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

template <typename TA, typename TO>
__global__ void __launch_bounds__(256) ln_fwd_kernel(const TA* __restrict__ a, int64_t lda,
                                                     int64_t M, int D, const float* __restrict__ g,
                                                     const float* __restrict__ beta,
                                                     float* __restrict__ stats, TO* __restrict__ h,
                                                     int64_t ldh, int ones_col) {
  pdl_trigger();
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < M; r += nw) {
    const TA* ar = a + r * lda;
    float s = 0.f;
    for (int c = lane; c < D; c += 32) s += ld1<TA>(ar + c);
    const float mean = warp_sum(s) / D;
    float q = 0.f;
    for (int c = lane; c < D; c += 32) {
      const float d = ld1<TA>(ar + c) - mean;
      q += d * d;
    }
    const float rstd = rsqrtf(warp_sum(q) / D + kLnEps);
    TO* hr = h + r * ldh;
    for (int c = lane; c < D; c += 32) {
      const float n = (ld1<TA>(ar + c) - mean) * rstd * g[c] + beta[c];
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
template <typename TA, typename TD>
__global__ void __launch_bounds__(kLnWarps * 32) ln_bwd_kernel(
    TD* __restrict__ dn, int64_t ldd, const TA* __restrict__ a, int64_t lda,
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
    const TA* ar = a + r * lda;
    const float mean = stats[2 * r], rstd = stats[2 * r + 1];
    float s1 = 0.f, s2 = 0.f;
    for (int c = lane; c < D; c += 32) {
      const float xh = (ld1<TA>(ar + c) - mean) * rstd;
      const float dx = ld1<TD>(dr + c) * g[c];
      s1 += dx;
      s2 += dx * xh;
    }
    const float m1 = warp_sum(s1) / D, m2 = warp_sum(s2) / D;
    for (int c = lane; c < D; c += 32) {
      const float xh = (ld1<TA>(ar + c) - mean) * rstd;
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

template <int NV, typename TA, typename TO>
__global__ void __launch_bounds__(kRegWarps * 32) ln_fwd_reg(
    const TA* __restrict__ a, int64_t lda, int64_t M, int D, const float* __restrict__ g,
    const float* __restrict__ beta, float* __restrict__ stats, TO* __restrict__ h, int64_t ldh,
    int ones_col) {
  pdl_trigger();
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * kRegWarps;
  // (gain / shift are re-read per row from L1 rather than held in 2 NV
  // float4 registers: the lighter footprint doubles the resident warps)
  const float inv_d = 1.f / D;
  for (int64_t r = (int64_t)blockIdx.x * kRegWarps + (threadIdx.x >> 5); r < M; r += nw) {
    const TA* ar = a + r * lda;
    float4 x[NV];
    float s = 0.f;
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      const int c = 4 * lane + 128 * j;
      x[j] = c < D ? V4<TA>::ld(ar + c) : make_float4(0.f, 0.f, 0.f, 0.f);
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
        const float4 gj = V4<float>::ld(g + c), bj = V4<float>::ld(beta + c);
        float4 o;
        o.x = elu_f((x[j].x - mean) * rstd * gj.x + bj.x);
        o.y = elu_f((x[j].y - mean) * rstd * gj.y + bj.y);
        o.z = elu_f((x[j].z - mean) * rstd * gj.z + bj.z);
        o.w = elu_f((x[j].w - mean) * rstd * gj.w + bj.w);
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
template <int NV, typename TA, typename TD>
__global__ void __launch_bounds__(kRegWarps * 32, 1) ln_bwd_reg(
    TD* __restrict__ dn, int64_t ldd, const TA* __restrict__ a, int64_t lda,
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
    const TA* ar = a + r * lda;
    const float2 st = reinterpret_cast<const float2*>(stats)[r];
    float4 xh[NV], dv[NV];
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      const int c = 4 * lane + 128 * j;
      if (c < D) {
        const float4 x = V4<TA>::ld(ar + c);
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

// ---- two-kernel backward (any D % 4 == 0): rows first, then columns.
// K1 (warp per row, streaming, no row-sized register arrays): the two row
// means of the LN backward, m1 = mean(dn g), m2 = mean(dn g xh) -> rs[M].
// K2 (column-parallel: a thread owns 4 adjacent columns, a block a chunk of
// rows): da = rstd (dn g - m1 - xh m2) written over dn, and the column sums
// dg = sum dn xh, dbeta = sum dn, colsum(da) accumulated in registers over
// the chunk -> block partials [chunk][3][D] (the ReduceJob layout).  Two
// coalesced reads of a and dn, one write of da, full occupancy: the row-
// register kernel held 3 x D column accumulators per warp and ran one
// 8-warp block per SM.
template <typename TA, typename TD>
__global__ void __launch_bounds__(256) ln_bwd_rows(const TD* __restrict__ dn, int64_t ldd,
                                                   const TA* __restrict__ a, int64_t lda,
                                                   const float* __restrict__ stats,
                                                   const float* __restrict__ g, int64_t M, int D,
                                                   float2* __restrict__ rs) {
  pdl_trigger();
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  const float inv_d = 1.f / D;
  for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < M; r += nw) {
    const TD* dr = dn + r * ldd;
    const TA* ar = a + r * lda;
    const float2 st = reinterpret_cast<const float2*>(stats)[r];
    float s1 = 0.f, s2 = 0.f;
    for (int c = 4 * lane; c < D; c += 128) {
      const float4 x = V4<TA>::ld(ar + c), d = V4<TD>::ld(dr + c), gv = V4<float>::ld(g + c);
      const float e0 = d.x * gv.x, e1 = d.y * gv.y, e2 = d.z * gv.z, e3 = d.w * gv.w;
      s1 += (e0 + e1) + (e2 + e3);
      s2 += (e0 * (x.x - st.x) + e1 * (x.y - st.x)) + (e2 * (x.z - st.x) + e3 * (x.w - st.x));
    }
    s1 = warp_sum(s1);
    s2 = warp_sum(s2);
    if (lane == 0) rs[r] = make_float2(s1 * inv_d, s2 * st.y * inv_d);
  }
}

template <typename TA, typename TD>
__global__ void __launch_bounds__(256) ln_bwd_cols(TD* __restrict__ dn, int64_t ldd,
                                                   const TA* __restrict__ a, int64_t lda,
                                                   const float* __restrict__ stats,
                                                   const float2* __restrict__ rs,
                                                   const float* __restrict__ g, int64_t M, int D,
                                                   int64_t rows_per, float* __restrict__ part) {
  pdl_trigger();
  pdl_wait();
  // a thread owns 8 adjacent columns (two 4-wide vectors: 16 B of bf16 per
  // array and row) and keeps U rows of loads in flight -- enough bytes in
  // flight per SM to stream at HBM rate
  constexpr int U = 8;
  const int64_t r0 = (int64_t)blockIdx.x * rows_per;
  const int64_t r1 = r0 + rows_per < M ? r0 + rows_per : M;
  float* pz = part + (int64_t)blockIdx.x * 3 * D;
  for (int c0 = 8 * threadIdx.x; c0 < D; c0 += 8 * blockDim.x) {
    const int nh = c0 + 4 < D ? 2 : 1;  // (D % 4 == 0: the second half may not exist)
    float4 gv[2], ag[2], ab[2], aa[2];
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
      gv[hh] = hh < nh ? V4<float>::ld(g + c0 + 4 * hh) : make_float4(0.f, 0.f, 0.f, 0.f);
      ag[hh] = ab[hh] = aa[hh] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    for (int64_t rb = r0; rb < r1; rb += U) {
      float4 x[U][2], d[U][2];
      float2 st[U], m[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t r = rb + u < r1 ? rb + u : r1 - 1;
        st[u] = reinterpret_cast<const float2*>(stats)[r];
        m[u] = rs[r];
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          const int c = c0 + 4 * (hh < nh ? hh : 0);
          x[u][hh] = V4<TA>::ld(a + r * lda + c);
          d[u][hh] = V4<TD>::ld(dn + r * ldd + c);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (rb + u >= r1) break;
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          if (hh >= nh) break;
          const float4 xv = x[u][hh], dv = d[u][hh], gg = gv[hh];
          const float mu = st[u].x, rstd = st[u].y;
          const float4 xh = make_float4((xv.x - mu) * rstd, (xv.y - mu) * rstd,
                                        (xv.z - mu) * rstd, (xv.w - mu) * rstd);
          const float4 da = make_float4(rstd * (dv.x * gg.x - m[u].x - xh.x * m[u].y),
                                        rstd * (dv.y * gg.y - m[u].x - xh.y * m[u].y),
                                        rstd * (dv.z * gg.z - m[u].x - xh.z * m[u].y),
                                        rstd * (dv.w * gg.w - m[u].x - xh.w * m[u].y));
          V4<TD>::st(dn + (rb + u) * ldd + c0 + 4 * hh, da);
          ag[hh].x += dv.x * xh.x; ag[hh].y += dv.y * xh.y;
          ag[hh].z += dv.z * xh.z; ag[hh].w += dv.w * xh.w;
          ab[hh].x += dv.x; ab[hh].y += dv.y; ab[hh].z += dv.z; ab[hh].w += dv.w;
          aa[hh].x += da.x; aa[hh].y += da.y; aa[hh].z += da.z; aa[hh].w += da.w;
        }
      }
    }
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
      if (hh >= nh) break;
      V4<float>::st(pz + c0 + 4 * hh, ag[hh]);
      V4<float>::st(pz + D + c0 + 4 * hh, ab[hh]);
      V4<float>::st(pz + 2 * D + c0 + 4 * hh, aa[hh]);
    }
  }
}

// ---- two-kernel forward: K1 row statistics (warp per row, streaming, the
// centred variance from a second sweep that hits L1), K2 column-parallel
// normalise + gain / shift + ELU (a thread owns 4 columns, 4 rows in flight).
template <typename TA>
__global__ void __launch_bounds__(256) ln_fwd_rows(const TA* __restrict__ a, int64_t lda,
                                                   int64_t M, int D, float* __restrict__ stats) {
  pdl_trigger();
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  const float inv_d = 1.f / D;
  for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < M; r += nw) {
    const TA* ar = a + r * lda;
    float s = 0.f;
    for (int c = 4 * lane; c < D; c += 128) {
      const float4 x = V4<TA>::ld(ar + c);
      s += (x.x + x.y) + (x.z + x.w);
    }
    const float mean = warp_sum(s) * inv_d;
    float q = 0.f;
    for (int c = 4 * lane; c < D; c += 128) {
      const float4 x = V4<TA>::ld(ar + c);
      const float d0 = x.x - mean, d1 = x.y - mean, d2 = x.z - mean, d3 = x.w - mean;
      q += (d0 * d0 + d1 * d1) + (d2 * d2 + d3 * d3);
    }
    const float rstd = rsqrtf(warp_sum(q) * inv_d + kLnEps);
    if (lane == 0) reinterpret_cast<float2*>(stats)[r] = make_float2(mean, rstd);
  }
}

template <typename TA, typename TO>
__global__ void __launch_bounds__(256) ln_fwd_cols(const TA* __restrict__ a, int64_t lda,
                                                   int64_t M, int D, const float* __restrict__ g,
                                                   const float* __restrict__ beta,
                                                   const float* __restrict__ stats,
                                                   TO* __restrict__ h, int64_t ldh, int ones_col,
                                                   int64_t rows_per) {
  pdl_trigger();
  pdl_wait();
  constexpr int U = 8;  // rows in flight; 8 columns (two 4-wide vectors) per thread
  const int64_t r0 = (int64_t)blockIdx.x * rows_per;
  const int64_t r1 = r0 + rows_per < M ? r0 + rows_per : M;
  for (int c0 = 8 * threadIdx.x; c0 < D; c0 += 8 * blockDim.x) {
    const int nh = c0 + 4 < D ? 2 : 1;
    float4 gv[2], bv[2];
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
      const int c = c0 + 4 * (hh < nh ? hh : 0);
      gv[hh] = V4<float>::ld(g + c);
      bv[hh] = V4<float>::ld(beta + c);
    }
    for (int64_t rb = r0; rb < r1; rb += U) {
      float4 x[U][2];
      float2 st[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t r = rb + u < r1 ? rb + u : r1 - 1;
        st[u] = reinterpret_cast<const float2*>(stats)[r];
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) x[u][hh] = V4<TA>::ld(a + r * lda + c0 + 4 * (hh < nh ? hh : 0));
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (rb + u >= r1) break;
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          if (hh >= nh) break;
          const float mu = st[u].x, rstd = st[u].y;
          float4 o;
          o.x = elu_f((x[u][hh].x - mu) * rstd * gv[hh].x + bv[hh].x);
          o.y = elu_f((x[u][hh].y - mu) * rstd * gv[hh].y + bv[hh].y);
          o.z = elu_f((x[u][hh].z - mu) * rstd * gv[hh].z + bv[hh].z);
          o.w = elu_f((x[u][hh].w - mu) * rstd * gv[hh].w + bv[hh].w);
          V4<TO>::st(h + (rb + u) * ldh + c0 + 4 * hh, o);
        }
      }
    }
  }
  if (ones_col >= 0 && threadIdx.x == 0)
    for (int64_t r = r0; r < r1; ++r) st1<TO>(h + r * ldh + ones_col, 1.f);
}

// ---- one-pass backward (the default when the rows fit shared memory): a
// persistent CTA walks blocks of kFbR rows; each block's dn and a rows land in
// shared memory by cp.async (double-buffered: block i + 1 loads while block i
// computes), warp w takes row w's means m1 = mean(dn g), m2 = mean(dn g x^)
// from shared memory, then a column-parallel pass over the same staged rows
// writes da over dn and accumulates dg = sum dn x^, dbeta = sum dn,
// colsum(da) in registers across all of the CTA's blocks -> one [3][D]
// partial per CTA (the ReduceJob layout).  dn and a cross HBM once.
constexpr int kFbR = 8;   // rows per block (one warp each in the row pass)
constexpr int kFbJ = 2;   // column quads per thread: D <= 256 * 4 * kFbJ

__device__ __forceinline__ void ln_cpa16(void* sdst, const void* gsrc, bool valid) {
  const uint32_t sa = (uint32_t)__cvta_generic_to_shared(sdst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(sa), "l"(gsrc),
               "r"(valid ? 16 : 0)
               : "memory");
}

template <typename TA, typename TD>
__global__ void __launch_bounds__(256) ln_bwd_fused(TD* __restrict__ dn, int64_t ldd,
                                                    const TA* __restrict__ a, int64_t lda,
                                                    const float* __restrict__ stats,
                                                    const float* __restrict__ g, int64_t M, int D,
                                                    float* __restrict__ part) {
  extern __shared__ __align__(16) uint8_t lsm[];
  __shared__ float2 s_m[kFbR], s_st[kFbR];
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  const int ua = D * (int)sizeof(TA) / 16, ud = D * (int)sizeof(TD) / 16;  // 16-B units per row
  TA* sa[2];
  TD* sd[2];
  {
    const size_t blk = (size_t)kFbR * 16 * (ua + ud);
    for (int k = 0; k < 2; ++k) {
      sa[k] = reinterpret_cast<TA*>(lsm + k * blk);
      sd[k] = reinterpret_cast<TD*>(lsm + k * blk + (size_t)kFbR * 16 * ua);
    }
  }
  pdl_trigger();
  pdl_wait();
  const int64_t nblk = (M + kFbR - 1) / kFbR;
  auto load = [&](int64_t rb, int k) {
    const int64_t r0 = rb * kFbR;
    for (int e = tid; e < kFbR * ua; e += blockDim.x) {
      const int rr = e / ua, u = e - rr * ua;
      const int64_t gr = r0 + rr;
      const bool ok = gr < M;
      ln_cpa16(reinterpret_cast<uint8_t*>(sa[k]) + (size_t)e * 16,
               reinterpret_cast<const uint8_t*>(a + (ok ? gr : 0) * lda) + (size_t)u * 16, ok);
    }
    for (int e = tid; e < kFbR * ud; e += blockDim.x) {
      const int rr = e / ud, u = e - rr * ud;
      const int64_t gr = r0 + rr;
      const bool ok = gr < M;
      ln_cpa16(reinterpret_cast<uint8_t*>(sd[k]) + (size_t)e * 16,
               reinterpret_cast<const uint8_t*>(dn + (ok ? gr : 0) * ldd) + (size_t)u * 16, ok);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  const float inv_d = 1.f / D;
  float4 ag[kFbJ], ab[kFbJ], aa[kFbJ], gv[kFbJ];
#pragma unroll
  for (int j = 0; j < kFbJ; ++j) {
    const int c0 = 4 * tid + 1024 * j;
    ag[j] = ab[j] = aa[j] = make_float4(0.f, 0.f, 0.f, 0.f);
    gv[j] = c0 < D ? V4<float>::ld(g + c0) : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  int k = 0;
  if ((int64_t)blockIdx.x < nblk) load(blockIdx.x, 0);
  for (int64_t rb = blockIdx.x; rb < nblk; rb += gridDim.x, k ^= 1) {
    if (rb + gridDim.x < nblk) {
      load(rb + gridDim.x, k ^ 1);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
    // row means (warp w: row w of the block)
    {
      const int64_t gr = rb * kFbR + w;
      if (gr < M) {
        const float2 st = reinterpret_cast<const float2*>(stats)[gr];
        const TA* ar = sa[k] + (size_t)w * D;
        const TD* dr = sd[k] + (size_t)w * D;
        float s1 = 0.f, s2 = 0.f;
        for (int c = 4 * lane; c < D; c += 128) {
          const float4 x = V4<TA>::ld(ar + c), d = V4<TD>::ld(dr + c), gg = V4<float>::ld(g + c);
          const float e0 = d.x * gg.x, e1 = d.y * gg.y, e2 = d.z * gg.z, e3 = d.w * gg.w;
          s1 += (e0 + e1) + (e2 + e3);
          s2 += (e0 * (x.x - st.x) + e1 * (x.y - st.x)) + (e2 * (x.z - st.x) + e3 * (x.w - st.x));
        }
        s1 = warp_sum(s1);
        s2 = warp_sum(s2);
        if (lane == 0) {
          s_m[w] = make_float2(s1 * inv_d, s2 * st.y * inv_d);
          s_st[w] = st;
        }
      }
    }
    __syncthreads();
    // column pass over the staged rows: da over dn, column partials in registers
#pragma unroll
    for (int j = 0; j < kFbJ; ++j) {
      const int c0 = 4 * tid + 1024 * j;
      if (c0 >= D) continue;
      for (int r = 0; r < kFbR; ++r) {
        const int64_t gr = rb * kFbR + r;
        if (gr >= M) break;
        const float4 xv = V4<TA>::ld(sa[k] + (size_t)r * D + c0);
        const float4 dv = V4<TD>::ld(sd[k] + (size_t)r * D + c0);
        const float mu = s_st[r].x, rstd = s_st[r].y;
        const float2 m = s_m[r];
        const float4 gg = gv[j];
        const float4 xh = make_float4((xv.x - mu) * rstd, (xv.y - mu) * rstd,
                                      (xv.z - mu) * rstd, (xv.w - mu) * rstd);
        const float4 da = make_float4(rstd * (dv.x * gg.x - m.x - xh.x * m.y),
                                      rstd * (dv.y * gg.y - m.x - xh.y * m.y),
                                      rstd * (dv.z * gg.z - m.x - xh.z * m.y),
                                      rstd * (dv.w * gg.w - m.x - xh.w * m.y));
        V4<TD>::st(dn + gr * ldd + c0, da);
        ag[j].x += dv.x * xh.x; ag[j].y += dv.y * xh.y; ag[j].z += dv.z * xh.z; ag[j].w += dv.w * xh.w;
        ab[j].x += dv.x; ab[j].y += dv.y; ab[j].z += dv.z; ab[j].w += dv.w;
        aa[j].x += da.x; aa[j].y += da.y; aa[j].z += da.z; aa[j].w += da.w;
      }
    }
    __syncthreads();  // buffer k is re-filled two blocks later
  }
  float* pz = part + (int64_t)blockIdx.x * 3 * D;
#pragma unroll
  for (int j = 0; j < kFbJ; ++j) {
    const int c0 = 4 * tid + 1024 * j;
    if (c0 >= D) continue;
    V4<float>::st(pz + c0, ag[j]);
    V4<float>::st(pz + D + c0, ab[j]);
    V4<float>::st(pz + 2 * D + c0, aa[j]);
  }
}

// row chunks of the column-parallel backward (<= its partial capacity)
int ln_col_chunks(int64_t M) {
  const int64_t b = ceil_div(M, 16);
  return (int)(b > 4 * kNumSMs ? 4 * kNumSMs : (b < 1 ? 1 : b));
}

int ln_blocks(int64_t M) {
  int64_t b = ceil_div(M, kLnWarps * 8);
  return (int)(b > 2 * kNumSMs ? 2 * kNumSMs : (b < 1 ? 1 : b));
}

}  // namespace

// block partials [ln_blocks][3][D] + the two-kernel backward's per-row
// (m1, m2) scratch [M] (8-byte aligned: the partial block is a multiple of 4 floats)
int64_t ln_part_floats(int64_t M, int D) {
  const int64_t nb = ln_blocks(M) > ln_col_chunks(M) ? ln_blocks(M) : ln_col_chunks(M);
  return nb * 3 * ceil_div(D, 4) * 4 + 2 * M;
}

namespace {
bool al(const void* p, int bytes) { return ((uintptr_t)p & (bytes - 1)) == 0; }
int reg_nv(int D) {
  if (D > 1024 || D % 4) return 0;
  return D <= 128 ? 1 : D <= 256 ? 2 : D <= 512 ? 4 : 8;
}

template <typename TA, typename TO>
int fwd_reg(int nv, unsigned blocks, const TA* a, int64_t lda, int64_t M, int D, const float* g,
            const float* beta, float* stats, TO* h, int64_t ldh, int ones_col, cudaStream_t s) {
  const dim3 gr(blocks), bl(kRegWarps * 32);
  switch (nv) {
    case 1:
      return launch_pdl("ln_fwd_reg", ln_fwd_reg<1, TA, TO>, gr, bl, 0, s, a, lda, M, D, g, beta,
                        stats, h, ldh, ones_col);
    case 2:
      return launch_pdl("ln_fwd_reg", ln_fwd_reg<2, TA, TO>, gr, bl, 0, s, a, lda, M, D, g, beta,
                        stats, h, ldh, ones_col);
    case 4:
      return launch_pdl("ln_fwd_reg", ln_fwd_reg<4, TA, TO>, gr, bl, 0, s, a, lda, M, D, g, beta,
                        stats, h, ldh, ones_col);
    default:
      return launch_pdl("ln_fwd_reg", ln_fwd_reg<8, TA, TO>, gr, bl, 0, s, a, lda, M, D, g, beta,
                        stats, h, ldh, ones_col);
  }
}

template <typename TA, typename TD>
int bwd_reg(int nv, unsigned blocks, TD* dn, int64_t ldd, const TA* a, int64_t lda,
            const float* stats, const float* g, int64_t M, int D, float* part, cudaStream_t s) {
  const dim3 gr(blocks), bl(kRegWarps * 32);
  const size_t sm = (size_t)3 * D * sizeof(float);
  switch (nv) {
    case 1:
      return launch_pdl("ln_bwd_reg", ln_bwd_reg<1, TA, TD>, gr, bl, sm, s, dn, ldd, a, lda,
                        stats, g, M, D, part);
    case 2:
      return launch_pdl("ln_bwd_reg", ln_bwd_reg<2, TA, TD>, gr, bl, sm, s, dn, ldd, a, lda,
                        stats, g, M, D, part);
    case 4:
      return launch_pdl("ln_bwd_reg", ln_bwd_reg<4, TA, TD>, gr, bl, sm, s, dn, ldd, a, lda,
                        stats, g, M, D, part);
    default:
      return launch_pdl("ln_bwd_reg", ln_bwd_reg<8, TA, TD>, gr, bl, sm, s, dn, ldd, a, lda,
                        stats, g, M, D, part);
  }
}
}  // namespace

// forward: the row-register kernel measured faster in the SAC update than the
// two-kernel version (cfg3 0.89 vs 0.95 ms / update); UL_LN_FWD_TWO_PASS=1
// selects the latter
static bool ln_fwd_two_pass() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("UL_LN_FWD_TWO_PASS");
    on = e ? atoi(e) != 0 : 0;
  }
  return on == 1;
}

static bool ln_two_pass() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("UL_LN_TWO_PASS");
    on = e ? atoi(e) != 0 : 1;
  }
  return on == 1;
}

// a: the pre-LN rows, fp32 or (a_bf16) bf16; h in dtype
int ln_forward(const void* a, int64_t lda, int64_t M, int D, const float* g, const float* beta,
               float* stats, void* h, int64_t ldh, int ones_col, int dtype, cudaStream_t s,
               bool a_bf16) {
  if (M == 0) return UL_OK;
  using BF = __nv_bfloat16;
  const int nv = reg_nv(D);
  const int hb = dtype == kBf16 ? 8 : 16;
  if (ln_fwd_two_pass() && D % 4 == 0 && lda % 4 == 0 && ldh % 4 == 0 &&
      al(a, a_bf16 ? 8 : 16) && al(g, 16) && al(beta, 16) && al(stats, 8) && al(h, hb)) {
    int64_t b1 = ceil_div(M, 8);
    b1 = b1 > 8 * kNumSMs ? 8 * kNumSMs : b1;
    const int64_t rows_per = 16;
    const int64_t nb = ceil_div(M, rows_per);
    int64_t thr = ceil_div(ceil_div((int64_t)D, 8), 32) * 32;
    thr = thr > 256 ? 256 : thr;
    const dim3 g1((unsigned)b1), g2((unsigned)nb), bl1(256), bl2((unsigned)thr);
#define UL_LNF(TA_, TO_)                                                                     \
  do {                                                                                       \
    UL_TRY(launch_pdl("ln_fwd_rows", ln_fwd_rows<TA_>, g1, bl1, 0, s, (const TA_*)a, lda, M, \
                      D, stats));                                                           \
    return launch_pdl("ln_fwd_cols", ln_fwd_cols<TA_, TO_>, g2, bl2, 0, s, (const TA_*)a,  \
                      lda, M, D, g, beta, (const float*)stats, (TO_*)h, ldh, ones_col,       \
                      rows_per);                                                            \
  } while (0)
    if (a_bf16 && dtype == kBf16) UL_LNF(BF, BF);
    if (a_bf16) UL_LNF(BF, float);
    if (dtype == kBf16) UL_LNF(float, BF);
    UL_LNF(float, float);
#undef UL_LNF
  }
  if (nv && lda % 4 == 0 && ldh % 4 == 0 && al(a, a_bf16 ? 8 : 16) && al(g, 16) &&
      al(beta, 16) && al(stats, 8) && al(h, hb)) {
    int64_t blocks = ceil_div(M, kRegWarps);
    blocks = blocks > 4 * kNumSMs ? 4 * kNumSMs : blocks;
    const unsigned nb = (unsigned)blocks;
    if (a_bf16 && dtype == kBf16)
      return fwd_reg(nv, nb, (const BF*)a, lda, M, D, g, beta, stats, (BF*)h, ldh, ones_col, s);
    if (a_bf16)
      return fwd_reg(nv, nb, (const BF*)a, lda, M, D, g, beta, stats, (float*)h, ldh, ones_col, s);
    if (dtype == kBf16)
      return fwd_reg(nv, nb, (const float*)a, lda, M, D, g, beta, stats, (BF*)h, ldh, ones_col,
                     s);
    return fwd_reg(nv, nb, (const float*)a, lda, M, D, g, beta, stats, (float*)h, ldh, ones_col,
                   s);
  }
  int64_t blocks = ceil_div(M, 8);
  blocks = blocks > 8 * kNumSMs ? 8 * kNumSMs : blocks;
  const dim3 gr((unsigned)blocks), bl(256);
  if (a_bf16 && dtype == kBf16)
    return launch_pdl("ln_fwd_kernel", ln_fwd_kernel<BF, BF>, gr, bl, 0, s, (const BF*)a, lda, M,
                      D, g, beta, stats, (BF*)h, ldh, ones_col);
  if (a_bf16)
    return launch_pdl("ln_fwd_kernel", ln_fwd_kernel<BF, float>, gr, bl, 0, s, (const BF*)a, lda,
                      M, D, g, beta, stats, (float*)h, ldh, ones_col);
  if (dtype == kBf16)
    return launch_pdl("ln_fwd_kernel", ln_fwd_kernel<float, BF>, gr, bl, 0, s, (const float*)a,
                      lda, M, D, g, beta, stats, (BF*)h, ldh, ones_col);
  return launch_pdl("ln_fwd_kernel", ln_fwd_kernel<float, float>, gr, bl, 0, s, (const float*)a,
                    lda, M, D, g, beta, stats, (float*)h, ldh, ones_col);
}

// dn (dtype rows, ld ldd) -> da in place; partials for the ReduceJob in
// *job (segments dg | dbeta | colsum(da), each D long, padded to 4).
int ln_backward(void* dn, int64_t ldd, const void* a, int64_t lda, const float* stats,
                const float* g, int64_t M, int D, float* part, int dtype, float* gg, float* gbeta,
                float* gb, ReduceJob* job, cudaStream_t s, bool a_bf16) {
  if (M == 0) return UL_OK;
  using BF = __nv_bfloat16;
  int nb = ln_blocks(M);
  const int Dp = (int)(ceil_div(D, 4) * 4);
  const size_t sm = (size_t)kLnWarps * 3 * D * sizeof(float);
  static bool attr[4] = {false, false, false, false};
  const int nv = reg_nv(D);
  const int db = dtype == kBf16 ? 8 : 16;
  const bool bd = dtype == kBf16;
  const int64_t nbmax = ln_blocks(M) > ln_col_chunks(M) ? ln_blocks(M) : ln_col_chunks(M);
  float2* rs = reinterpret_cast<float2*>(part + nbmax * 3 * Dp);
  // one-pass kernel: 16-byte staged rows, D <= 2048, both row blocks in
  // shared memory (UL_LN_BWD_FUSED=0 keeps the row + column kernel pair)
  static int fused_env = -1;
  if (fused_env < 0) {
    const char* e = getenv("UL_LN_BWD_FUSED");
    fused_env = e ? atoi(e) != 0 : 1;
  }
  const int eA = a_bf16 ? 2 : 4, eD = bd ? 2 : 4;
  const size_t fsm = (size_t)2 * kFbR * D * (eA + eD);
  if (fused_env && D % 4 == 0 && D <= 1024 * kFbJ && (D * eA) % 16 == 0 && (D * eD) % 16 == 0 &&
      (lda * eA) % 16 == 0 && (ldd * eD) % 16 == 0 && al(a, 16) && al(dn, 16) && al(g, 16) &&
      al(stats, 8) && al(part, 16) && fsm <= 200 * 1024) {
    const int64_t nblk = ceil_div(M, (int64_t)kFbR);
    const int per_sm = fsm <= 72 * 1024 ? 3 : (fsm <= 110 * 1024 ? 2 : 1);
    int64_t grid = (int64_t)per_sm * kNumSMs;
    grid = grid < nblk ? grid : nblk;
    grid = grid < nbmax ? grid : nbmax;  // (the partial buffer's chunk capacity)
    nb = (int)grid;
    static bool fattr[4] = {false, false, false, false};
#define UL_LNF1(TA_, TD_, I_)                                                                     \
  do {                                                                                            \
    if (!fattr[I_]) {                                                                             \
      UL_CUDA(cudaFuncSetAttribute(ln_bwd_fused<TA_, TD_>,                                        \
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));     \
      fattr[I_] = true;                                                                           \
    }                                                                                             \
    UL_TRY(launch_pdl("ln_bwd_fused", ln_bwd_fused<TA_, TD_>, dim3((unsigned)nb), dim3(256), fsm, \
                      s, (TD_*)dn, ldd, (const TA_*)a, lda, stats, g, M, D, part));               \
  } while (0)
    if (a_bf16 && bd) UL_LNF1(BF, BF, 0);
    else if (a_bf16) UL_LNF1(BF, float, 1);
    else if (bd) UL_LNF1(float, BF, 2);
    else UL_LNF1(float, float, 3);
#undef UL_LNF1
  } else if (D % 4 == 0 && lda % 4 == 0 && ldd % 4 == 0 && al(a, a_bf16 ? 8 : 16) &&
      al(g, 16) && al(stats, 8) && al(dn, db) && al(part, 16) && ln_two_pass()) {
    int64_t b1 = ceil_div(M, 8);
    b1 = b1 > 8 * kNumSMs ? 8 * kNumSMs : b1;
    int64_t rows_per = ceil_div(M, (int64_t)ln_col_chunks(M));
    rows_per = rows_per < 16 ? 16 : rows_per;
    nb = (int)ceil_div(M, rows_per);
    int64_t thr = ceil_div(ceil_div((int64_t)D, 8), 32) * 32;
    thr = thr > 256 ? 256 : thr;
    const dim3 g1((unsigned)b1), g2((unsigned)nb), bl1(256), bl2((unsigned)thr);
#define UL_LN2(TA_, TD_)                                                                       \
  do {                                                                                         \
    UL_TRY(launch_pdl("ln_bwd_rows", ln_bwd_rows<TA_, TD_>, g1, bl1, 0, s, (const TD_*)dn, ldd, \
                      (const TA_*)a, lda, stats, g, M, D, rs));                                \
    UL_TRY(launch_pdl("ln_bwd_cols", ln_bwd_cols<TA_, TD_>, g2, bl2, 0, s, (TD_*)dn, ldd,       \
                      (const TA_*)a, lda, stats, (const float2*)rs, g, M, D, rows_per, part)); \
  } while (0)
    if (a_bf16 && bd) UL_LN2(BF, BF);
    else if (a_bf16) UL_LN2(BF, float);
    else if (bd) UL_LN2(float, BF);
    else UL_LN2(float, float);
#undef UL_LN2
  } else if (nv && lda % 4 == 0 && ldd % 4 == 0 && al(a, a_bf16 ? 8 : 16) && al(g, 16) &&
      al(stats, 8) && al(dn, db) && al(part, 16)) {
    int64_t b = ceil_div(M, kRegWarps * 4);
    nb = (int)(b > kNumSMs ? kNumSMs : b);
    if (a_bf16 && bd)
      UL_TRY(bwd_reg(nv, nb, (BF*)dn, ldd, (const BF*)a, lda, stats, g, M, D, part, s));
    else if (a_bf16)
      UL_TRY(bwd_reg(nv, nb, (float*)dn, ldd, (const BF*)a, lda, stats, g, M, D, part, s));
    else if (bd)
      UL_TRY(bwd_reg(nv, nb, (BF*)dn, ldd, (const float*)a, lda, stats, g, M, D, part, s));
    else
      UL_TRY(bwd_reg(nv, nb, (float*)dn, ldd, (const float*)a, lda, stats, g, M, D, part, s));
  } else {
    const int ai = (a_bf16 ? 2 : 0) + (bd ? 1 : 0);
    auto attr_once = [&](const void* fn) -> int {
      if (!attr[ai]) {
        UL_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        attr[ai] = true;
      }
      return UL_OK;
    };
    const dim3 gr(nb), bl(kLnWarps * 32);
    if (a_bf16 && bd) {
      UL_TRY(attr_once((const void*)ln_bwd_kernel<BF, BF>));
      UL_TRY(launch_pdl("ln_bwd_kernel", ln_bwd_kernel<BF, BF>, gr, bl, sm, s, (BF*)dn, ldd,
                        (const BF*)a, lda, stats, g, M, D, part));
    } else if (a_bf16) {
      UL_TRY(attr_once((const void*)ln_bwd_kernel<BF, float>));
      UL_TRY(launch_pdl("ln_bwd_kernel", ln_bwd_kernel<BF, float>, gr, bl, sm, s, (float*)dn, ldd,
                        (const BF*)a, lda, stats, g, M, D, part));
    } else if (bd) {
      UL_TRY(attr_once((const void*)ln_bwd_kernel<float, BF>));
      UL_TRY(launch_pdl("ln_bwd_kernel", ln_bwd_kernel<float, BF>, gr, bl, sm, s, (BF*)dn, ldd,
                        (const float*)a, lda, stats, g, M, D, part));
    } else {
      UL_TRY(attr_once((const void*)ln_bwd_kernel<float, float>));
      UL_TRY(launch_pdl("ln_bwd_kernel", ln_bwd_kernel<float, float>, gr, bl, sm, s, (float*)dn,
                        ldd, (const float*)a, lda, stats, g, M, D, part));
    }
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
