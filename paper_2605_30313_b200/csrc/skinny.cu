// Skinny output layers (N = action dim 12/23/29 or the critic's 1): the last
// MLP layer of every network, R:tensornet/mlp.py:165 (forward) and :192-197
// (backward).  A 128-row UMMA tile wastes > 90 % of its work at N <= 32, so
// these layers get row-tiled SIMT kernels that read h exactly once:
//   skinny_fwd : out[M,N] = h[M,K] W^T + b
//   skinny_bwd : dh[M,K] = (dout W) * elu'(h), block partials of dW = dout^T h,
//                db = colsum(dout) and (optionally) colsum(dh) -- the bias
//                gradient of the layer below, so its dW GEMM needs no extra
//                pass over dh -- then one fixed-order partial reduction.
// A 64-row tile of h (fp32 or bf16 rows) is staged into shared memory with
// 16-byte cp.async copies, all issued before the first wait (one memory round
// trip per tile); W (N x K, the reference's flat layout) sits in shared memory
// for the whole block.  Four threads per row; smem rows are padded by 16 B so
// the per-row 16-byte reads of a warp fall in distinct banks.
#include <cuda_bf16.h>

#include "internal.cuh"

namespace ul {
namespace {

constexpr int kRows = 64, kThr = 256, kMaxN = 32, kMaxW = 8192 /* N*K floats in smem */;
constexpr int kKC = 256;  // K columns per staged chunk

template <typename T>
__device__ __forceinline__ float4 ld4(const T* p);
template <>
__device__ __forceinline__ float4 ld4<float>(const float* p) {
  return *reinterpret_cast<const float4*>(p);
}
template <>
__device__ __forceinline__ float4 ld4<__nv_bfloat16>(const __nv_bfloat16* p) {
  const uint2 u = *reinterpret_cast<const uint2*>(p);
  return make_float4(__uint_as_float(u.x << 16), __uint_as_float(u.x & 0xFFFF0000u),
                     __uint_as_float(u.y << 16), __uint_as_float(u.y & 0xFFFF0000u));
}

template <typename T>
__device__ __forceinline__ void st4(T* p, float4 v);
template <>
__device__ __forceinline__ void st4<float>(float* p, float4 v) {
  *reinterpret_cast<float4*>(p) = v;
}
template <>
__device__ __forceinline__ void st4<__nv_bfloat16>(__nv_bfloat16* p, float4 v) {
  __nv_bfloat162 a = __floats2bfloat162_rn(v.x, v.y), b = __floats2bfloat162_rn(v.z, v.w);
  uint2 u;
  u.x = *reinterpret_cast<uint32_t*>(&a);
  u.y = *reinterpret_cast<uint32_t*>(&b);
  *reinterpret_cast<uint2*>(p) = u;
}

__device__ __forceinline__ void cp_async16(void* sdst, const void* gsrc, bool valid) {
  const uint32_t s = (uint32_t)__cvta_generic_to_shared(sdst);
  const int n = valid ? 16 : 0;  // 0 source bytes -> zero fill
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gsrc), "r"(n)
               : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
}

// smem row pitch (elements) for a chunk of kc columns: 16-byte rows + 16 B pad
template <typename T>
__host__ __device__ constexpr int pitch_of(int kc) {
  return ((kc * (int)sizeof(T) + 15) / 16 * 16 + 16) / (int)sizeof(T);
}

// stage rows [r0, r0+kRows) x columns [k0, k0+kc) of h into sh (pitch P)
template <typename T>
__device__ __forceinline__ void stage_tile(const T* __restrict__ h, int64_t ldh, int64_t M,
                                           int64_t r0, int k0, int kc, T* sh, int P) {
  constexpr int kE = 16 / (int)sizeof(T);  // elements per 16-byte copy
  const int per_row = (kc + kE - 1) / kE;
  for (int e = threadIdx.x; e < kRows * per_row; e += kThr) {
    const int rr = e / per_row, u = e - rr * per_row;
    const int64_t gr = r0 + rr;
    const bool ok = gr < M;
    cp_async16(sh + rr * P + u * kE, h + (ok ? gr : 0) * ldh + k0 + u * kE, ok);
  }
  cp_async_wait_all();
  __syncthreads();
}

// W[:, k0:k0+kc] -> sw (pitch PW, zero beyond kc): all of a thread's loads are
// issued before its smem stores (one memory round trip, not one per element)
__device__ __forceinline__ void stage_w(const float* __restrict__ W, int K, int N, int NP, int k0,
                                        int kc, int KC, float* sw, int PW) {
  const int total = NP * KC;  // rows N..NP-1 are zero padding
  for (int base = threadIdx.x; base < total; base += kThr * 8) {
    float v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = base + u * kThr;
      const int j = e / KC, c = e - j * KC;
      v[u] = (e < total && c < kc && j < N) ? __ldg(W + (int64_t)j * K + k0 + c) : 0.f;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = base + u * kThr;
      const int j = e / KC, c = e - j * KC;
      if (e < total) sw[j * PW + c] = v[u];
    }
  }
}

// out[r, j] = b[j] + sum_k h[r, k] W[j, k].  Thread (row r = t/4, q = t%4)
// covers the 4-column groups c = 4q + 16i for all NP (>= N, padded) outputs;
// the row's four partial sums meet through two lane shuffles.
template <typename TH, int NP>
__global__ void __launch_bounds__(kThr) skinny_fwd_kernel(const TH* __restrict__ h, int64_t ldh,
                                                          int64_t M, int K, int N,
                                                          const float* __restrict__ W,
                                                          const float* __restrict__ b,
                                                          float* __restrict__ out, int64_t ldo) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int KC = K < kKC ? (K + 7) / 8 * 8 : kKC;
  const int P = pitch_of<TH>(KC), PW = pitch_of<float>(KC);
  TH* sh = reinterpret_cast<TH*>(smem);
  float* sw = reinterpret_cast<float*>(smem + (size_t)kRows * P * sizeof(TH));
  const int t = threadIdx.x, r = t >> 2, q = t & 3;
  const int64_t r0 = (int64_t)blockIdx.x * kRows;
  pdl_trigger();
  pdl_wait();
  float acc[NP];
#pragma unroll
  for (int j = 0; j < NP; ++j) acc[j] = 0.f;
  for (int k0 = 0; k0 < K; k0 += KC) {
    const int kc = K - k0 < KC ? K - k0 : KC;
    stage_w(W, K, N, NP, k0, kc, KC, sw, PW);
    stage_tile<TH>(h, ldh, M, r0, k0, kc, sh, P);
    const TH* hr = sh + r * P;
    for (int c = 4 * q; c < kc; c += 16) {
      float4 hv = ld4<TH>(hr + c);
      // cp.async copies whole 16-byte groups: columns >= kc may hold padding
      if (c + 4 > kc) {
        if (c + 1 >= kc) hv.y = 0.f;
        if (c + 2 >= kc) hv.z = 0.f;
        if (c + 3 >= kc) hv.w = 0.f;
      }
#pragma unroll
      for (int j = 0; j < NP; ++j) {
        const float4 w = *reinterpret_cast<const float4*>(sw + j * PW + c);
        acc[j] = fmaf(hv.x, w.x, fmaf(hv.y, w.y, fmaf(hv.z, w.z, fmaf(hv.w, w.w, acc[j]))));
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int j = 0; j < NP; ++j) {
    acc[j] += __shfl_xor_sync(0xffffffffu, acc[j], 1);
    acc[j] += __shfl_xor_sync(0xffffffffu, acc[j], 2);
  }
  const int64_t gr = r0 + r;
  if (gr < M) {
#pragma unroll
    for (int j = 0; j < NP; ++j)
      if ((j & 3) == q && j < N) out[gr * ldo + j] = acc[j] + (b ? __ldg(b + j) : 0.f);
  }
}

// Per block z: part[z] = [dW partial (N x K) | db partial (N) | colsum(dh) (K, if csum)]
template <typename TH, int NP>
__global__ void __launch_bounds__(kThr) skinny_bwd_kernel(
    const TH* __restrict__ h, int64_t ldh, int64_t M, int K, int N, const float* __restrict__ W,
    const float* __restrict__ dout, int64_t ldd, TH* __restrict__ dh, int64_t lddh, int elu_grad,
    float* __restrict__ part, int64_t plen, int want_dw, int csum) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int KC = K < kKC ? (K + 7) / 8 * 8 : kKC;
  const int P = pitch_of<TH>(KC), PW = pitch_of<float>(KC);
  TH* sh = reinterpret_cast<TH*>(smem);
  float* sw = reinterpret_cast<float*>(smem + (size_t)kRows * P * sizeof(TH));
  float* sd = sw + (size_t)NP * PW;        // [kRows][kMaxN + 1] upstream gradient
  float* sdh = sd + kRows * (kMaxN + 1);   // [kRows][PW] dh tile (column sums)
  const int t = threadIdx.x, r = t >> 2, q = t & 3;
  const int64_t r0 = (int64_t)blockIdx.x * kRows;
  float* pz = part + (int64_t)blockIdx.x * plen;
  pdl_trigger();
  pdl_wait();
  for (int base = t; base < kRows * N; base += kThr * 8) {
    float v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = base + u * kThr;
      const int rr = e / N, j = e - rr * N;
      const int64_t gr = r0 + rr;
      v[u] = (e < kRows * N && gr < M) ? __ldg(dout + gr * ldd + j) : 0.f;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = base + u * kThr;
      const int rr = e / N, j = e - rr * N;
      if (e < kRows * N) sd[rr * (kMaxN + 1) + j] = v[u];
    }
  }
  __syncthreads();
  if (want_dw && t < N) {
    float s = 0.f;
    for (int rr = 0; rr < kRows; ++rr) s += sd[rr * (kMaxN + 1) + t];
    pz[(int64_t)N * K + t] = s;
  }
  float g[NP];
#pragma unroll
  for (int j = 0; j < NP; ++j) g[j] = j < N ? sd[r * (kMaxN + 1) + j] : 0.f;
  const int64_t gr = r0 + r;
  for (int k0 = 0; k0 < K; k0 += KC) {
    const int kc = K - k0 < KC ? K - k0 : KC;
    stage_w(W, K, N, NP, k0, kc, KC, sw, PW);
    stage_tile<TH>(h, ldh, M, r0, k0, kc, sh, P);
    // dh for row r, 4-column groups c = 4q, 4q + 16, ...
    if (dh) {
      for (int c = 4 * q; c < kc; c += 16) {
        float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int j = 0; j < NP; ++j) {
          const float4 w = *reinterpret_cast<const float4*>(sw + j * PW + c);
          s.x = fmaf(g[j], w.x, s.x);
          s.y = fmaf(g[j], w.y, s.y);
          s.z = fmaf(g[j], w.z, s.z);
          s.w = fmaf(g[j], w.w, s.w);
        }
        if (elu_grad) {
          const float4 hv = ld4<TH>(sh + r * P + c);
          s.x *= elu_grad_from_act(hv.x);
          s.y *= elu_grad_from_act(hv.y);
          s.z *= elu_grad_from_act(hv.z);
          s.w *= elu_grad_from_act(hv.w);
        }
        if (gr >= M) s = make_float4(0.f, 0.f, 0.f, 0.f);
        if (csum) *reinterpret_cast<float4*>(sdh + r * PW + c) = s;
        if (gr < M) {
          if (c + 4 <= kc) {
            st4<TH>(dh + gr * lddh + k0 + c, s);
          } else {
            const float sv[4] = {s.x, s.y, s.z, s.w};
            for (int i = 0; c + i < kc; ++i) dh[gr * lddh + k0 + c + i] = (TH)sv[i];
          }
        }
      }
    }
    // dW partial: pair (4-column group c4, output j), sum over the tile's rows
    if (want_dw) {
      const int g4 = (kc + 3) / 4;
      for (int pr = t; pr < g4 * N; pr += kThr) {
        const int j = pr / g4, c = 4 * (pr - j * g4);
        float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 8
        for (int rr = 0; rr < kRows; ++rr) {
          const float d = sd[rr * (kMaxN + 1) + j];
          const float4 hv = ld4<TH>(sh + rr * P + c);
          s.x = fmaf(d, hv.x, s.x);
          s.y = fmaf(d, hv.y, s.y);
          s.z = fmaf(d, hv.z, s.z);
          s.w = fmaf(d, hv.w, s.w);
        }
        const float sv[4] = {s.x, s.y, s.z, s.w};
        for (int i = 0; i < 4 && c + i < kc; ++i) pz[(int64_t)j * K + k0 + c + i] = sv[i];
      }
    }
    if (csum) {
      __syncthreads();
      for (int c = t; c < kc; c += kThr) {
        float s = 0.f;
        for (int rr = 0; rr < kRows; ++rr) s += sdh[rr * PW + c];
        pz[(int64_t)N * K + N + k0 + c] = s;
      }
    }
    __syncthreads();
  }
}

// out_d[j] = sum_z part[z * plen + j] for j in segment d (fixed order over z):
// 128 columns per CTA (float4 lanes), 32 warps over z, smem combine.  Three
// destination segments share one launch: [0, n0) -> o0, [n0, n0+n1) -> o1,
// [n0+n1, n0+n1+n2) -> o2 (a null destination skips its segment).
__global__ void __launch_bounds__(1024) reduce_parts_kernel(const float* __restrict__ part,
                                                            int nblk, int64_t plen, int64_t n0,
                                                            float* o0, int64_t n1, float* o1,
                                                            int64_t n2, float* o2) {
  __shared__ float4 sm[32][33];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t total = n0 + n1 + n2;
  pdl_trigger();
  pdl_wait();
  const int64_t j = ((int64_t)blockIdx.x * 32 + lane) * 4;
  float4 a = make_float4(0.f, 0.f, 0.f, 0.f), b = a;
  if (j < total) {
    const bool vec = (plen & 3) == 0 && j + 4 <= total;
    int z = w;
    for (; z < nblk; z += 64) {
      const float* p0 = part + (int64_t)z * plen + j;
      const float* p1 = z + 32 < nblk ? p0 + 32 * plen : nullptr;
      float4 x, y = make_float4(0.f, 0.f, 0.f, 0.f);
      if (vec) {
        x = *reinterpret_cast<const float4*>(p0);
        if (p1) y = *reinterpret_cast<const float4*>(p1);
      } else {
        x = make_float4(p0[0], j + 1 < total ? p0[1] : 0.f, j + 2 < total ? p0[2] : 0.f,
                        j + 3 < total ? p0[3] : 0.f);
        if (p1)
          y = make_float4(p1[0], j + 1 < total ? p1[1] : 0.f, j + 2 < total ? p1[2] : 0.f,
                          j + 3 < total ? p1[3] : 0.f);
      }
      a.x += x.x; a.y += x.y; a.z += x.z; a.w += x.w;
      b.x += y.x; b.y += y.y; b.z += y.z; b.w += y.w;
    }
  }
  sm[w][lane] = make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
  __syncthreads();
  if (w == 0 && j < total) {
    float4 s = sm[0][lane];
    for (int k = 1; k < 32; ++k) {
      const float4 v = sm[k][lane];
      s.x += v.x; s.y += v.y; s.z += v.z; s.w += v.w;
    }
    const float sv[4] = {s.x, s.y, s.z, s.w};
    for (int i = 0; i < 4 && j + i < total; ++i) {
      const int64_t c = j + i;
      if (c < n0) {
        if (o0) o0[c] = sv[i];
      } else if (c < n0 + n1) {
        if (o1) o1[c - n0] = sv[i];
      } else if (o2) {
        o2[c - n0 - n1] = sv[i];
      }
    }
  }
}

template <typename TH>
size_t fwd_smem(int K, int NP) {
  const int KC = K < kKC ? (K + 7) / 8 * 8 : kKC;
  return (size_t)kRows * pitch_of<TH>(KC) * sizeof(TH) + (size_t)NP * pitch_of<float>(KC) * 4;
}
template <typename TH>
size_t bwd_smem(int K, int NP) {
  const int KC = K < kKC ? (K + 7) / 8 * 8 : kKC;
  return fwd_smem<TH>(K, NP) + (size_t)kRows * (kMaxN + 1) * 4 +
         (size_t)kRows * pitch_of<float>(KC) * 4;
}

// padded output count: the kernels are instantiated for these
inline int pad_n(int N) {
  const int sizes[] = {1, 2, 4, 8, 12, 16, 24, 32};
  for (int v : sizes)
    if (N <= v) return v;
  return 0;
}

template <typename TH, int NP>
int fwd_np(const void* h, int64_t ldh, int64_t M, int K, int N, const float* W, const float* b,
           float* out, int64_t ldo, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    UL_CUDA(cudaFuncSetAttribute(skinny_fwd_kernel<TH, NP>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    attr = true;
  }
  return launch_pdl("skinny_fwd_kernel", skinny_fwd_kernel<TH, NP>,
                    dim3((unsigned)ceil_div(M, kRows)), dim3(kThr), fwd_smem<TH>(K, NP), s,
                    reinterpret_cast<const TH*>(h), ldh, M, K, N, W, b, out, ldo);
}

template <typename TH, int NP>
int bwd_np(const void* h, int64_t ldh, int64_t M, int K, int N, const float* W, const float* dout,
           int64_t ldd, void* dh, int64_t lddh, bool elu_grad, float* gw, float* gb, float* gcs,
           float* part, ReduceJob* defer, cudaStream_t s) {
  const int nblk = (int)ceil_div(M, kRows);
  const bool want_dw = gw || gb;
  const bool csum = gcs != nullptr && dh != nullptr;
  // block partial stride, padded to 16 bytes for the float4 reduction
  const int64_t plen = ceil_div((int64_t)N * K + N + (csum ? K : 0), 4) * 4;
  static bool attr = false;
  if (!attr) {
    UL_CUDA(cudaFuncSetAttribute(skinny_bwd_kernel<TH, NP>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    attr = true;
  }
  UL_TRY(launch_pdl("skinny_bwd_kernel", skinny_bwd_kernel<TH, NP>, dim3(nblk), dim3(kThr),
                    bwd_smem<TH>(K, NP), s, reinterpret_cast<const TH*>(h), ldh, M, K, N, W, dout,
                    ldd, reinterpret_cast<TH*>(dh), lddh, elu_grad ? 1 : 0, part, plen,
                    want_dw ? 1 : 0, csum ? 1 : 0));
  if (defer) {
    // the caller folds this reduction into its next reduction launch
    *defer = ReduceJob{};
    defer->src = part;
    defer->nz = nblk;
    defer->kind = 1;
    defer->len = plen;
    defer->n0 = (int64_t)N * K;
    defer->o0 = gw;
    defer->n1 = N;
    defer->o1 = gb;
    defer->n2 = csum ? K : 0;
    defer->o2 = gcs;
    return UL_OK;
  }
  if (want_dw || csum) {
    UL_TRY(launch_pdl("reduce_parts_kernel", reduce_parts_kernel,
                      dim3((unsigned)ceil_div(plen, 128)), dim3(1024), 0, s,
                      (const float*)part, nblk, plen, (int64_t)N * K, gw, (int64_t)N, gb,
                      (int64_t)(csum ? K : 0), gcs));
  }
  return UL_OK;
}

#define UL_SKINNY_NP(FN, ...)                         \
  switch (pad_n(N)) {                                 \
    case 1: return FN<TH, 1>(__VA_ARGS__);            \
    case 2: return FN<TH, 2>(__VA_ARGS__);            \
    case 4: return FN<TH, 4>(__VA_ARGS__);            \
    case 8: return FN<TH, 8>(__VA_ARGS__);            \
    case 12: return FN<TH, 12>(__VA_ARGS__);          \
    case 16: return FN<TH, 16>(__VA_ARGS__);          \
    case 24: return FN<TH, 24>(__VA_ARGS__);          \
    default: return FN<TH, 32>(__VA_ARGS__);          \
  }

template <typename TH>
int fwd_t(const void* h, int64_t ldh, int64_t M, int K, int N, const float* W, const float* b,
          float* out, int64_t ldo, cudaStream_t s) {
  UL_SKINNY_NP(fwd_np, h, ldh, M, K, N, W, b, out, ldo, s)
}

template <typename TH>
int bwd_t(const void* h, int64_t ldh, int64_t M, int K, int N, const float* W, const float* dout,
          int64_t ldd, void* dh, int64_t lddh, bool elu_grad, float* gw, float* gb, float* gcs,
          float* part, ReduceJob* defer, cudaStream_t s) {
  UL_SKINNY_NP(bwd_np, h, ldh, M, K, N, W, dout, ldd, dh, lddh, elu_grad, gw, gb, gcs, part,
               defer, s)
}
#undef UL_SKINNY_NP

}  // namespace

bool skinny_ok(int N, int K) { return N >= 1 && N <= kMaxN && (int64_t)N * K <= kMaxW * 4; }

int64_t skinny_part_floats(int64_t M, int K, int N) {
  return ceil_div(M, kRows) * (ceil_div((int64_t)N * K + N + K, 4) * 4);
}

int skinny_fwd(const void* h, int64_t ldh, int64_t M, int K, int N, const float* W,
               const float* b, float* out, int64_t ldo, int dtype, cudaStream_t s) {
  if (M == 0) return UL_OK;
  if (dtype == kBf16) return fwd_t<__nv_bfloat16>(h, ldh, M, K, N, W, b, out, ldo, s);
  return fwd_t<float>(h, ldh, M, K, N, W, b, out, ldo, s);
}

// gw [N, K], gb [N] and gcs [K] (column sums of dh: the bias gradient of the
// layer below) receive reduced results when non-null; `part` holds
// skinny_part_floats(M, K, N) floats of scratch.
// defer (may be null): instead of launching the partial reduction, describe it
// so the caller can fold it into a later reduction launch.
int skinny_bwd(const void* h, int64_t ldh, int64_t M, int K, int N, const float* W,
               const float* dout, int64_t ldd, void* dh, int64_t lddh, bool elu_grad, float* gw,
               float* gb, float* gcs, float* part, int dtype, ReduceJob* defer, cudaStream_t s) {
  if (M == 0) return UL_OK;
  if (dtype == kBf16)
    return bwd_t<__nv_bfloat16>(h, ldh, M, K, N, W, dout, ldd, dh, lddh, elu_grad, gw, gb, gcs,
                                part, defer, s);
  return bwd_t<float>(h, ldh, M, K, N, W, dout, ldd, dh, lddh, elu_grad, gw, gb, gcs, part,
                      defer, s);
}

}  // namespace ul
