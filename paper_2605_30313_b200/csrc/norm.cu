// K3 running observation normaliser: batch moments + parallel-Welford (Chan)
// merge into float64 running statistics, then normalise + clip.
//
// Replaces R:tensornet/normalizer.py:27-45 (update), :47-49 (apply) and
// :61-66 (norm_update_apply).  Device state layout (float64):
//     state[0] = count, state[1 .. D] = mean, state[1+D .. 2D] = var.
// Moments: each CTA owns a 32-column strip x a row chunk; threads walk rows
// (coalesced 128 B per warp-row) accumulating shifted sums
// S1 = sum(x - c), S2 = sum((x - c)^2) in f64 with c = x[0, d] (no
// cancellation for |mean| >> std).  Partials land in a workspace; the last CTA
// (ticket) reduces them in fixed order and applies the Chan merge -- one
// launch, deterministic.  Bytes: 4 B/element read (+4 B write when applying).
#include "internal.cuh"

namespace ul {
namespace {

constexpr int kColTile = 32, kRowWarps = 8, kMaxChunks = 64;
// vectorised variant (D % 4 == 0, 16-byte rows): lane = 4-column group, 32
// warps per CTA walk the rows with 8 float4 loads in flight each, one CTA
// per SM; partials [CTA][D][2] merged by the last CTA (columns x CTA phases)
constexpr int kV4Warps = 32, kV4Inflight = 8, kV4Cols = 4 * 32, kV4MaxChunks = kNumSMs;

__global__ void __launch_bounds__(256) moments_kernel(const float* __restrict__ x, int64_t B,
                                                      int64_t D, int64_t ldx, int64_t rows_per,
                                                      double* __restrict__ state, double* work,
                                                      unsigned int* ticket, int frozen) {
  __shared__ double s1[kRowWarps][kColTile], s2[kRowWarps][kColTile];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t d = (int64_t)blockIdx.x * kColTile + lane;
  const int64_t r0 = (int64_t)blockIdx.y * rows_per;
  const int64_t r1 = r0 + rows_per < B ? r0 + rows_per : B;
  double a1 = 0.0, a2 = 0.0;
  if (d < D) {
    const double c = (double)x[d];
    // 4 rows in flight per warp (independent loads), then fold
    double b1 = 0.0, b2 = 0.0, e1 = 0.0, e2 = 0.0, f1 = 0.0, f2 = 0.0;
    int64_t r = r0 + w;
    for (; r + 3 * kRowWarps < r1; r += 4 * kRowWarps) {
      const double v0 = (double)__ldg(x + r * ldx + d) - c;
      const double v1 = (double)__ldg(x + (r + kRowWarps) * ldx + d) - c;
      const double v2 = (double)__ldg(x + (r + 2 * kRowWarps) * ldx + d) - c;
      const double v3 = (double)__ldg(x + (r + 3 * kRowWarps) * ldx + d) - c;
      a1 += v0;
      a2 += v0 * v0;
      b1 += v1;
      b2 += v1 * v1;
      e1 += v2;
      e2 += v2 * v2;
      f1 += v3;
      f2 += v3 * v3;
    }
    for (; r < r1; r += kRowWarps) {
      const double v = (double)x[r * ldx + d] - c;
      a1 += v;
      a2 += v * v;
    }
    a1 = (a1 + b1) + (e1 + f1);
    a2 = (a2 + b2) + (e2 + f2);
  }
  s1[w][lane] = a1;
  s2[w][lane] = a2;
  __syncthreads();
  if (w == 0 && d < D) {
    double t1 = 0.0, t2 = 0.0;
    for (int j = 0; j < kRowWarps; ++j) {
      t1 += s1[j][lane];
      t2 += s2[j][lane];
    }
    work[((int64_t)blockIdx.y * D + d) * 2 + 0] = t1;
    work[((int64_t)blockIdx.y * D + d) * 2 + 1] = t2;
  }
  const unsigned int nblk = gridDim.x * gridDim.y;
  if (!last_block_ticket(ticket, nblk)) return;
  if (frozen) return;
  // last CTA: fixed-order reduction + Chan merge for every column
  const double n = (double)B;
  const double cnt = state[0];
  const double tot = cnt + n;
  for (int64_t j = threadIdx.x; j < D; j += blockDim.x) {
    double t1 = 0.0, t2 = 0.0;
    for (int c = 0; c < (int)gridDim.y; ++c) {
      t1 += work[((int64_t)c * D + j) * 2 + 0];
      t2 += work[((int64_t)c * D + j) * 2 + 1];
    }
    const double shift = (double)x[j];
    const double m1 = t1 / n;
    const double bmean = shift + m1;
    double bvar = t2 / n - m1 * m1;
    bvar = bvar < 0.0 ? 0.0 : bvar;
    const double mean = state[1 + j], var = state[1 + D + j];
    const double delta = bmean - mean;
    state[1 + j] = mean + delta * (n / tot);
    state[1 + D + j] = (var * cnt + bvar * n + delta * delta * (cnt * n / tot)) / tot;
  }
  __syncthreads();
  if (threadIdx.x == 0) state[0] = tot;
}

__device__ __forceinline__ void chan_merge(double* state, int64_t D, int64_t j, double t1, double t2,
                                           double shift, double n) {
  const double cnt = state[0];
  const double tot = cnt + n;
  const double m1 = t1 / n;
  const double bmean = shift + m1;
  double bvar = t2 / n - m1 * m1;
  bvar = bvar < 0.0 ? 0.0 : bvar;
  const double mean = state[1 + j], var = state[1 + D + j];
  const double delta = bmean - mean;
  state[1 + j] = mean + delta * (n / tot);
  state[1 + D + j] = (var * cnt + bvar * n + delta * delta * (cnt * n / tot)) / tot;
}

__global__ void __launch_bounds__(kV4Warps * 32) moments_v4_kernel(
    const float* __restrict__ x, int64_t B, int64_t D, int64_t ldx, int64_t rows_per,
    double* __restrict__ state, double* work, unsigned int* ticket) {
  // per warp pair-reduction scratch: [16 warps][32 lanes][4 cols][2 sums]
  __shared__ double red[kV4Warps / 2][32][8];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t c0 = ((int64_t)blockIdx.x * 32 + lane) * 4;  // first of this lane's 4 columns
  const bool on = c0 < D;
  const int64_t r0 = (int64_t)blockIdx.y * rows_per;
  const int64_t r1 = r0 + rows_per < B ? r0 + rows_per : B;
  double a[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};  // S1[0..3], S2[0..3]
  if (on) {
    const float4 cf = __ldg(reinterpret_cast<const float4*>(x + c0));
    const double sh[4] = {(double)cf.x, (double)cf.y, (double)cf.z, (double)cf.w};
    for (int64_t r = r0 + w; r < r1; r += (int64_t)kV4Warps * kV4Inflight) {
      float4 v[kV4Inflight];
#pragma unroll
      for (int k = 0; k < kV4Inflight; ++k) {
        const int64_t rr = r + (int64_t)k * kV4Warps;
        v[k] = rr < r1 ? __ldg(reinterpret_cast<const float4*>(x + rr * ldx + c0))
                       : make_float4(cf.x, cf.y, cf.z, cf.w);  // (shift: contributes 0)
      }
#pragma unroll
      for (int k = 0; k < kV4Inflight; ++k) {
        const double e[4] = {(double)v[k].x - sh[0], (double)v[k].y - sh[1],
                             (double)v[k].z - sh[2], (double)v[k].w - sh[3]};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          a[q] += e[q];
          a[4 + q] = fma(e[q], e[q], a[4 + q]);
        }
      }
    }
  }
  // fixed-order pairwise reduction over the 32 warps
  for (int half = kV4Warps / 2; half >= 1; half >>= 1) {
    if (w >= half && w < 2 * half)
#pragma unroll
      for (int q = 0; q < 8; ++q) red[w - half][lane][q] = a[q];
    __syncthreads();
    if (w < half)
#pragma unroll
      for (int q = 0; q < 8; ++q) a[q] += red[w][lane][q];
    __syncthreads();
  }
  if (w == 0 && on) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if (c0 + q < D) {
        work[((int64_t)blockIdx.y * D + c0 + q) * 2 + 0] = a[q];
        work[((int64_t)blockIdx.y * D + c0 + q) * 2 + 1] = a[4 + q];
      }
    }
  }
  const unsigned int nblk = gridDim.x * gridDim.y;
  if (!last_block_ticket(ticket, nblk)) return;
  // last CTA: column j, chunk phase p (P phases in parallel), fixed order
  const int nchunk = (int)gridDim.y;
  const int P = (int)(blockDim.x / D) < 1 ? 1 : (int)(blockDim.x / D);
  double* sred = &red[0][0][0];  // reused: [P][D][2] doubles (<= 32 KB)
  const int Pm = (int)((sizeof(red) / sizeof(double)) / (2 * D)) < P
                     ? (int)((sizeof(red) / sizeof(double)) / (2 * D)) : P;
  for (int64_t j0 = 0; j0 < D; j0 += blockDim.x) {
    const int64_t j = j0 + (threadIdx.x % (Pm > 1 ? D : blockDim.x));
    const int p = Pm > 1 ? (int)(threadIdx.x / D) : 0;
    double t1 = 0.0, t2 = 0.0;
    if (p < Pm && j < D) {
      for (int c = p; c < nchunk; c += Pm) {
        t1 += work[((int64_t)c * D + j) * 2 + 0];
        t2 += work[((int64_t)c * D + j) * 2 + 1];
      }
      if (Pm > 1) {
        sred[((int64_t)p * D + j) * 2 + 0] = t1;
        sred[((int64_t)p * D + j) * 2 + 1] = t2;
      }
    }
    __syncthreads();
    if (p == 0 && j < D) {
      if (Pm > 1) {
        t1 = 0.0;
        t2 = 0.0;
        for (int q = 0; q < Pm; ++q) {
          t1 += sred[((int64_t)q * D + j) * 2 + 0];
          t2 += sred[((int64_t)q * D + j) * 2 + 1];
        }
      }
      chan_merge(state, D, j, t1, t2, (double)x[j], (double)B);
    }
    __syncthreads();
    if (Pm > 1) break;  // (Pm > 1 means D <= blockDim.x: every column done)
  }
  __syncthreads();
  if (threadIdx.x == 0) state[0] += (double)B;
}

__global__ void apply_kernel(const float* __restrict__ x, int64_t B, int64_t D, int64_t ldx,
                             const double* __restrict__ state, float* __restrict__ out,
                             int64_t ldo) {
  const int64_t total = B * D;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += stride) {
    const int64_t r = i / D, d = i - r * D;
    const double z = ((double)x[r * ldx + d] - state[1 + d]) / sqrt(state[1 + D + d] + 1e-8);
    out[r * ldo + d] = (float)fmin(fmax(z, -10.0), 10.0);
  }
}

}  // namespace
}  // namespace ul

// workspace: ul_norm_work_bytes(D) bytes of device memory (partials + ticket).
extern "C" int64_t ul_norm_work_bytes(int64_t D) {
  const int64_t chunks = ul::kMaxChunks > ul::kV4MaxChunks ? ul::kMaxChunks : ul::kV4MaxChunks;
  return (int64_t)sizeof(double) * 2 * chunks * D + 64;
}

extern "C" int ul_norm_update(const float* x, int64_t B, int64_t D, int64_t ldx, double* state,
                              void* work, int frozen, void* stream) {
  UL_CHECK_ARG(B >= 0 && D >= 1 && ldx >= D, "normalizer: bad shape");
  if (B == 0 || frozen) return UL_OK;
  double* partial = reinterpret_cast<double*>(work);
  unsigned int* ticket =
      reinterpret_cast<unsigned int*>(reinterpret_cast<char*>(work) + ul_norm_work_bytes(D) - 64);
  if (D % 4 == 0 && ldx % 4 == 0 && ((uintptr_t)x & 15) == 0) {
    // vectorised: one 1024-thread CTA per SM (per column tile of 128)
    const int64_t col_tiles = ul::ceil_div(D, ul::kV4Cols);
    int64_t chunks = ul::ceil_div(ul::kNumSMs, col_tiles);
    const int64_t cap = ul::ceil_div(B, 256);
    chunks = chunks < cap ? chunks : cap;
    chunks = chunks < 1 ? 1 : chunks;
    const int64_t rows_per = ul::ceil_div(B, chunks);
    chunks = ul::ceil_div(B, rows_per);
    ul::moments_v4_kernel<<<dim3((unsigned)col_tiles, (unsigned)chunks), ul::kV4Warps * 32, 0,
                            ul::as_stream(stream)>>>(x, B, D, ldx, rows_per, state, partial,
                                                     ticket);
    return ul::check_launch("moments_v4_kernel");
  }
  const int64_t col_tiles = ul::ceil_div(D, ul::kColTile);
  int64_t chunks = ul::ceil_div(2 * ul::kNumSMs, col_tiles);
  const int64_t cap = ul::ceil_div(B, 64);
  chunks = chunks < cap ? chunks : cap;
  chunks = chunks < 1 ? 1 : (chunks > ul::kMaxChunks ? ul::kMaxChunks : chunks);
  const int64_t rows_per = ul::ceil_div(B, chunks);
  chunks = ul::ceil_div(B, rows_per);
  ul::moments_kernel<<<dim3((unsigned)col_tiles, (unsigned)chunks), 256, 0,
                       ul::as_stream(stream)>>>(x, B, D, ldx, rows_per, state, partial, ticket,
                                                frozen);
  return ul::check_launch("moments_kernel");
}

extern "C" int ul_norm_apply(const float* x, int64_t B, int64_t D, int64_t ldx,
                             const double* state, float* out, int64_t ldo, void* stream) {
  UL_CHECK_ARG(B >= 0 && D >= 1 && ldx >= D && ldo >= D, "normalizer: bad shape");
  if (B == 0) return UL_OK;
  int64_t blocks = ul::ceil_div(B * D, 256);
  blocks = blocks > 8 * ul::kNumSMs ? 8 * ul::kNumSMs : blocks;
  ul::apply_kernel<<<(unsigned)blocks, 256, 0, ul::as_stream(stream)>>>(x, B, D, ldx, state, out,
                                                                       ldo);
  return ul::check_launch("norm_apply_kernel");
}
