// Skinny output layers (N = action dim 12/23/29 or the critic's 1): the last
// MLP layer of every network, R:tensornet/mlp.py:165 (forward) and :192-197
// (backward).  A 128x128 GEMM tile wastes > 90 % of its work at N <= 32, so
// these layers get row-blocked kernels instead:
//   skinny_fwd : out[M,N] = h[M,K] W^T + b      (one pass over h)
//   skinny_bwd : dh[M,K] = (dout W) * elu'(h)  AND  dW/db block partials,
//                reading h and dout exactly once (the dW and dX GEMMs of the
//                last layer fused), then a fixed-order partial reduction.
// Rows are staged through shared memory in 64-column chunks with coalesced
// loads; W (N x K, the reference's flat layout) is read through L1/L2.
#include "internal.cuh"

namespace ul {
namespace {

constexpr int kRows = 64, kCols = 64, kThr = 256, kMaxN = 32;

__global__ void __launch_bounds__(kThr) skinny_fwd_kernel(const float* __restrict__ h, int64_t ldh,
                                                          int64_t M, int K, int N,
                                                          const float* __restrict__ W,
                                                          const float* __restrict__ b,
                                                          float* __restrict__ out, int64_t ldo) {
  __shared__ float sh[kRows][kCols + 1];
  __shared__ float sw[kMaxN][kCols + 1];
  const int t = threadIdx.x;
  const int64_t r0 = (int64_t)blockIdx.x * kRows;
  const int r = t >> 2, q = t & 3;  // row, output lane (outputs q, q+4, ...)
  float acc[kMaxN / 4];
#pragma unroll
  for (int u = 0; u < kMaxN / 4; ++u) acc[u] = 0.f;
  for (int k0 = 0; k0 < K; k0 += kCols) {
    for (int e = t; e < kRows * kCols; e += kThr) {
      const int rr = e / kCols, cc = e % kCols;
      const int64_t gr = r0 + rr;
      sh[rr][cc] = (gr < M && k0 + cc < K) ? h[gr * ldh + k0 + cc] : 0.f;
    }
    for (int e = t; e < N * kCols; e += kThr) {
      const int j = e / kCols, cc = e % kCols;
      sw[j][cc] = k0 + cc < K ? W[(int64_t)j * K + k0 + cc] : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < kMaxN / 4; ++u) {
      const int j = q + 4 * u;
      if (j < N) {
        float s = acc[u];
#pragma unroll 8
        for (int c = 0; c < kCols; ++c) s = fmaf(sh[r][c], sw[j][c], s);
        acc[u] = s;
      }
    }
    __syncthreads();
  }
  const int64_t gr = r0 + r;
  if (gr < M) {
#pragma unroll
    for (int u = 0; u < kMaxN / 4; ++u) {
      const int j = q + 4 * u;
      if (j < N) out[gr * ldo + j] = acc[u] + b[j];
    }
  }
}

// part_w: [gridDim.x, N, K], part_b: [gridDim.x, N]
__global__ void __launch_bounds__(kThr) skinny_bwd_kernel(
    const float* __restrict__ h, int64_t ldh, int64_t M, int K, int N,
    const float* __restrict__ W, const float* __restrict__ dout, int64_t ldd,
    float* __restrict__ dh, int64_t lddh, int elu_grad, float* __restrict__ part_w,
    float* __restrict__ part_b) {
  __shared__ float sh[kRows][kCols + 1];
  __shared__ float sd[kRows][kMaxN + 1];
  const int t = threadIdx.x;
  const int64_t r0 = (int64_t)blockIdx.x * kRows;
  for (int e = t; e < kRows * N; e += kThr) {
    const int rr = e / N, j = e % N;
    const int64_t gr = r0 + rr;
    sd[rr][j] = gr < M ? dout[gr * ldd + j] : 0.f;
  }
  __syncthreads();
  if (part_b && t < N) {
    float s = 0.f;
    for (int rr = 0; rr < kRows; ++rr) s += sd[rr][t];
    part_b[(int64_t)blockIdx.x * N + t] = s;
  }
  const int c = t & (kCols - 1), rq = t >> 6;  // column, row quarter (4 groups of 16 rows)
  for (int k0 = 0; k0 < K; k0 += kCols) {
    for (int e = t; e < kRows * kCols; e += kThr) {
      const int rr = e / kCols, cc = e % kCols;
      const int64_t gr = r0 + rr;
      sh[rr][cc] = (gr < M && k0 + cc < K) ? h[gr * ldh + k0 + cc] : 0.f;
    }
    __syncthreads();
    const int k = k0 + c;
    if (k < K) {
      // W column k for all N outputs
      float wk[kMaxN];
#pragma unroll
      for (int j = 0; j < kMaxN; ++j) wk[j] = j < N ? __ldg(W + (int64_t)j * K + k) : 0.f;
      if (dh) {
        for (int rr = rq * 16; rr < rq * 16 + 16; ++rr) {
          const int64_t gr = r0 + rr;
          if (gr >= M) break;
          float s = 0.f;
#pragma unroll
          for (int j = 0; j < kMaxN; ++j)
            if (j < N) s = fmaf(sd[rr][j], wk[j], s);
          if (elu_grad) s *= elu_grad_from_act(sh[rr][c]);
          dh[gr * lddh + k] = s;
        }
      }
      if (part_w) {
        // dW[j, k] partial over this block's rows; outputs j = rq, rq+4, ...
        for (int j = rq; j < N; j += 4) {
          float s = 0.f;
#pragma unroll 8
          for (int rr = 0; rr < kRows; ++rr) s = fmaf(sd[rr][j], sh[rr][c], s);
          part_w[((int64_t)blockIdx.x * N + j) * K + k] = s;
        }
      }
    }
    __syncthreads();
  }
}

// out[j] = sum_z part[z*len + j]: 32 outputs per CTA (coalesced lanes), the
// partial index split across 8 warps, fixed-order smem combine (deterministic)
__global__ void __launch_bounds__(256) reduce_parts_kernel(const float* __restrict__ part,
                                                           int nblk, int64_t len,
                                                           float* __restrict__ out) {
  __shared__ float sm[8][33];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t j = (int64_t)blockIdx.x * 32 + lane;
  float s = 0.f;
  if (j < len) {
    float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
    int z = w;
    for (; z + 24 < nblk; z += 32) {
      s0 += part[(int64_t)z * len + j];
      s1 += part[(int64_t)(z + 8) * len + j];
      s2 += part[(int64_t)(z + 16) * len + j];
      s3 += part[(int64_t)(z + 24) * len + j];
    }
    for (; z < nblk; z += 8) s0 += part[(int64_t)z * len + j];
    s = (s0 + s1) + (s2 + s3);
  }
  sm[w][lane] = s;
  __syncthreads();
  if (w == 0 && j < len) {
    float t = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) t += sm[k][lane];
    out[j] = t;
  }
}

}  // namespace

bool skinny_ok(int N) { return N >= 1 && N <= kMaxN; }

int64_t skinny_part_floats(int64_t M, int K, int N) {
  return ceil_div(M, kRows) * (int64_t)N * (K + 1);
}

int skinny_fwd(const float* h, int64_t ldh, int64_t M, int K, int N, const float* W,
               const float* b, float* out, int64_t ldo, cudaStream_t s) {
  if (M == 0) return UL_OK;
  skinny_fwd_kernel<<<(unsigned)ceil_div(M, kRows), kThr, 0, s>>>(h, ldh, M, K, N, W, b, out, ldo);
  return check_launch("skinny_fwd_kernel");
}

// gw [N, K] and gb [N] receive the reduced gradients when non-null; `part`
// holds skinny_part_floats(M, K, N) floats of scratch.
int skinny_bwd(const float* h, int64_t ldh, int64_t M, int K, int N, const float* W,
               const float* dout, int64_t ldd, float* dh, int64_t lddh, bool elu_grad,
               float* gw, float* gb, float* part, cudaStream_t s) {
  if (M == 0) return UL_OK;
  const int nblk = (int)ceil_div(M, kRows);
  float* pw = gw ? part : nullptr;
  float* pb = gb ? part + (int64_t)nblk * N * K : nullptr;
  skinny_bwd_kernel<<<nblk, kThr, 0, s>>>(h, ldh, M, K, N, W, dout, ldd, dh, lddh, elu_grad ? 1 : 0,
                                          pw, pb);
  UL_TRY(check_launch("skinny_bwd_kernel"));
  if (gw) {
    reduce_parts_kernel<<<(unsigned)ceil_div((int64_t)N * K, 32), 256, 0, s>>>(pw, nblk,
                                                                               (int64_t)N * K, gw);
    UL_TRY(check_launch("reduce_parts_kernel"));
  }
  if (gb) {
    reduce_parts_kernel<<<(unsigned)ceil_div(N, 32), 256, 0, s>>>(pb, nblk, N, gb);
    UL_TRY(check_launch("reduce_parts_kernel"));
  }
  return UL_OK;
}

}  // namespace ul
