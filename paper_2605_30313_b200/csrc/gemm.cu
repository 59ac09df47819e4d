// K7/K8: fp32 SIMT GEMM with fused MLP epilogues + the MLP forward/backward drivers.
//
// This is the exact-fp32 (parity) GEMM path: 128x128x8 CTA tiles, 256 threads,
// 8x8 register micro-tiles, register-prefetched double-buffered shared memory.
// Three operand layouts cover the MLP (R:tensornet/mlp.py:153-198):
//   forward  Z = H W^T + b      A K-major [M,K], B K-major (W is [out,in])
//   dX       dH = dZ W          A K-major,        B N-major
//   dW       dW = dZ^T H        A M-major,        B N-major  (reduction over the
//                                batch: split-K into a workspace + fixed-order
//                                reduction, db fused as the row-sum of dZ^T)
// Epilogues fuse bias, ELU (R:tensornet/mlp.py:134-138) and the ELU gradient
// from the cached activation (:141-143), so no separate elementwise pass runs.
#include "internal.cuh"

namespace ul {
namespace {

constexpr int BM = 128, BN = 128, BK = 8, kThreads = 256;
constexpr int SPAD = 4;  // smem row pad: kills the 2-way transposed-store conflict

struct KArgs {
  int64_t M, N, K;
  const float* A;
  int64_t lda;
  const float* B;
  int64_t ldb;
  float* C;
  int64_t ldc;
  const float* bias;
  const float* aux;
  int64_t ldaux;
  int64_t k_per_split;
  float* rowsum;
  int ones_col;
};

template <bool KMAJOR>
__device__ __forceinline__ void load_tile(const float* __restrict__ P, int64_t ld, int64_t rows,
                                          int64_t K, int64_t r0, int64_t k0, int64_t k_end,
                                          int tid, float (&reg)[4]) {
  if (KMAJOR) {  // element (r, k) = P[r*ld + k]; thread -> (r = tid/2, k = (tid%2)*4 + j)
    const int64_t r = r0 + (tid >> 1);
    const int64_t kb = k0 + (tid & 1) * 4;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t k = kb + j;
      reg[j] = (r < rows && k < k_end) ? __ldg(P + r * ld + k) : 0.f;
    }
  } else {  // element (r, k) = P[k*ld + r]; thread -> (k = tid/32, r = (tid%32)*4 + j)
    const int64_t k = k0 + (tid >> 5);
    const int64_t rb = r0 + (tid & 31) * 4;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t r = rb + j;
      reg[j] = (r < rows && k < k_end) ? __ldg(P + k * ld + r) : 0.f;
    }
  }
}

template <bool KMAJOR>
__device__ __forceinline__ void store_tile(float (*S)[BM + SPAD], int tid, const float (&reg)[4]) {
  if (KMAJOR) {
    const int r = tid >> 1, kb = (tid & 1) * 4;
#pragma unroll
    for (int j = 0; j < 4; ++j) S[kb + j][r] = reg[j];
  } else {
    const int k = tid >> 5, rb = (tid & 31) * 4;
    *reinterpret_cast<float4*>(&S[k][rb]) = make_float4(reg[0], reg[1], reg[2], reg[3]);
  }
}

template <bool A_K, bool B_K, int EPI, bool SPLIT, bool ROWSUM>
__global__ void __launch_bounds__(kThreads) sgemm_kernel(KArgs p) {
  __shared__ __align__(16) float As[2][BK][BM + SPAD];
  __shared__ __align__(16) float Bs[2][BK][BN + SPAD];
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  const int64_t m0 = (int64_t)blockIdx.x * BM, n0 = (int64_t)blockIdx.y * BN;
  const int64_t kb = (int64_t)blockIdx.z * p.k_per_split;
  const int64_t ke = kb + p.k_per_split < p.K ? kb + p.k_per_split : p.K;
  const bool do_rowsum = ROWSUM && blockIdx.y == 0;

  float acc[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;
  float rs[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) rs[i] = 0.f;

  float ra[4], rb[4];
  load_tile<A_K>(p.A, p.lda, p.M, p.K, m0, kb, ke, tid, ra);
  load_tile<B_K>(p.B, p.ldb, p.N, p.K, n0, kb, ke, tid, rb);
  store_tile<A_K>(As[0], tid, ra);
  store_tile<B_K>(Bs[0], tid, rb);
  __syncthreads();

  int buf = 0;
  for (int64_t k0 = kb; k0 < ke; k0 += BK) {
    const bool has_next = k0 + BK < ke;
    if (has_next) {
      load_tile<A_K>(p.A, p.lda, p.M, p.K, m0, k0 + BK, ke, tid, ra);
      load_tile<B_K>(p.B, p.ldb, p.N, p.K, n0, k0 + BK, ke, tid, rb);
    }
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float a[8], b[8];
      const float4 a0 = *reinterpret_cast<const float4*>(&As[buf][kk][ty * 4]);
      const float4 a1 = *reinterpret_cast<const float4*>(&As[buf][kk][64 + ty * 4]);
      const float4 b0 = *reinterpret_cast<const float4*>(&Bs[buf][kk][tx * 4]);
      const float4 b1 = *reinterpret_cast<const float4*>(&Bs[buf][kk][64 + tx * 4]);
      a[0] = a0.x; a[1] = a0.y; a[2] = a0.z; a[3] = a0.w;
      a[4] = a1.x; a[5] = a1.y; a[6] = a1.z; a[7] = a1.w;
      b[0] = b0.x; b[1] = b0.y; b[2] = b0.z; b[3] = b0.w;
      b[4] = b1.x; b[5] = b1.y; b[6] = b1.z; b[7] = b1.w;
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
      if (do_rowsum) {
#pragma unroll
        for (int i = 0; i < 8; ++i) rs[i] += a[i];
      }
    }
    if (has_next) {
      store_tile<A_K>(As[buf ^ 1], tid, ra);
      store_tile<B_K>(Bs[buf ^ 1], tid, rb);
    }
    __syncthreads();
    buf ^= 1;
  }

  float* C = p.C;
  if (SPLIT) C += (int64_t)blockIdx.z * p.M * p.N;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int64_t m = m0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + (i - 4));
    if (m >= p.M) continue;
    if (do_rowsum && tx == 0) p.rowsum[(int64_t)blockIdx.z * p.M + m] = rs[i];
    if (!SPLIT && p.ones_col >= 0 && blockIdx.y == 0 && tx == 0) C[m * p.ldc + p.ones_col] = 1.f;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int64_t n = n0 + (j < 4 ? tx * 4 + j : 64 + tx * 4 + (j - 4));
      if (n >= p.N) continue;
      float v = acc[i][j];
      if (EPI == kEpiBias || EPI == kEpiBiasElu) v += p.bias[n];
      if (EPI == kEpiBiasElu) v = elu_f(v);
      if (EPI == kEpiEluGrad) v *= elu_grad_from_act(p.aux[m * p.ldaux + n]);
      C[m * p.ldc + n] = v;
    }
  }
}

// out[j] = sum_z ws[z*len + j]: 32 outputs per CTA (coalesced lanes), splits
// spread over 8 warps with 4 loads in flight each, fixed-order combine.
__global__ void __launch_bounds__(256) reduce_splits_kernel(const float* __restrict__ ws,
                                                            int splits, int64_t len,
                                                            float* __restrict__ out,
                                                            int64_t ld_rows, int64_t row_len) {
  __shared__ float sm[8][33];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t j = (int64_t)blockIdx.x * 32 + lane;
  pdl_trigger();
  pdl_wait();
  float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
  if (j < len) {
    int z = w;
    for (; z + 24 < splits; z += 32) {
      s0 += ws[(int64_t)z * len + j];
      s1 += ws[(int64_t)(z + 8) * len + j];
      s2 += ws[(int64_t)(z + 16) * len + j];
      s3 += ws[(int64_t)(z + 24) * len + j];
    }
    for (; z < splits; z += 8) s0 += ws[(int64_t)z * len + j];
  }
  sm[w][lane] = (s0 + s1) + (s2 + s3);
  __syncthreads();
  if (w == 0 && j < len) {
    float t = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) t += sm[k][lane];
    // out may be strided by rows (ld_rows) when row_len < ld_rows
    const int64_t r = j / row_len, c = j - r * row_len;
    out[r * ld_rows + c] = t;
  }
}

template <bool A_K, bool B_K, int EPI, bool SPLIT, bool ROWSUM>
void launch_t(const GemmDesc& d, const KArgs& a, dim3 grid, cudaStream_t s) {
  sgemm_kernel<A_K, B_K, EPI, SPLIT, ROWSUM><<<grid, kThreads, 0, s>>>(a);
}

}  // namespace

static int64_t k_per_split(int64_t K, int splits) {
  splits = splits < 1 ? 1 : splits;
  return ceil_div(ceil_div(K > 0 ? K : 1, splits), BK) * BK;
}

int gemm_num_splits(int64_t K, int splits) {
  return (int)ceil_div(K > 0 ? K : 1, k_per_split(K, splits));
}

int gemm_f32(const GemmDesc& d, cudaStream_t s) {
  if (d.M == 0 || d.N == 0) return UL_OK;
  KArgs a{d.M, d.N, d.K, d.A, d.lda, d.B, d.ldb, d.C, d.ldc, d.bias, d.aux, d.ldaux, 0, d.rowsum,
          d.ones_col};
  a.k_per_split = k_per_split(d.K, d.splits);
  const int zs = gemm_num_splits(d.K, d.splits);
  dim3 grid((unsigned)ceil_div(d.M, BM), (unsigned)ceil_div(d.N, BN), (unsigned)zs);
  const bool split = zs > 1 || d.rowsum != nullptr;
  if (split && d.epi != kEpiStore) {
    set_error("gemm: split-K needs the store epilogue");
    return UL_ERR_VALUE;
  }
  // dispatch: (a_k, b_k, epi, split, rowsum) combinations the MLP uses
  if (d.a_kmajor && d.b_kmajor) {  // forward
    switch (d.epi) {
      case kEpiStore: launch_t<true, true, kEpiStore, false, false>(d, a, grid, s); break;
      case kEpiBias: launch_t<true, true, kEpiBias, false, false>(d, a, grid, s); break;
      case kEpiBiasElu: launch_t<true, true, kEpiBiasElu, false, false>(d, a, grid, s); break;
      default: set_error("gemm: epilogue %d unsupported for NT", d.epi); return UL_ERR_VALUE;
    }
  } else if (d.a_kmajor && !d.b_kmajor) {  // dX
    switch (d.epi) {
      case kEpiStore: launch_t<true, false, kEpiStore, false, false>(d, a, grid, s); break;
      case kEpiEluGrad: launch_t<true, false, kEpiEluGrad, false, false>(d, a, grid, s); break;
      default: set_error("gemm: epilogue %d unsupported for NN", d.epi); return UL_ERR_VALUE;
    }
  } else if (!d.a_kmajor && !d.b_kmajor) {  // dW (split-K, optional row sums)
    if (d.epi != kEpiStore) {
      set_error("gemm: TN layout supports the store epilogue only");
      return UL_ERR_VALUE;
    }
    if (d.rowsum) launch_t<false, false, kEpiStore, true, true>(d, a, grid, s);
    else if (zs > 1) launch_t<false, false, kEpiStore, true, false>(d, a, grid, s);
    else launch_t<false, false, kEpiStore, false, false>(d, a, grid, s);
  } else {
    set_error("gemm: layout (A M-major, B K-major) unsupported");
    return UL_ERR_VALUE;
  }
  return check_launch("sgemm_kernel");
}

int reduce_splits(const float* ws, int splits, int64_t len, float* out, int64_t ld_rows,
                  int64_t row_len, cudaStream_t s) {
  if (len == 0) return UL_OK;
  const unsigned blocks = (unsigned)ceil_div(len, 32);
  return launch_pdl("reduce_splits_kernel", reduce_splits_kernel, dim3(blocks), dim3(256), 0, s,
                    ws, splits, len, out, ld_rows, row_len);
}

}  // namespace ul

extern "C" int ul_gemm_f32(int layout, int epi, int64_t M, int64_t N, int64_t K, const float* A,
                           int64_t lda, const float* B, int64_t ldb, float* C, int64_t ldc,
                           const float* bias, const float* aux, int64_t ldaux, void* stream) {
  ul::GemmDesc g{};
  g.M = M; g.N = N; g.K = K; g.A = A; g.lda = lda; g.B = B; g.ldb = ldb; g.C = C; g.ldc = ldc;
  g.bias = bias; g.aux = aux; g.ldaux = ldaux;
  g.a_kmajor = layout & 1; g.b_kmajor = (layout >> 1) & 1; g.epi = epi; g.splits = 1;
  return ul::gemm_f32(g, ul::as_stream(stream));
}
