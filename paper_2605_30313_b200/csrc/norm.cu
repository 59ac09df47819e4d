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
  return (int64_t)sizeof(double) * 2 * ul::kMaxChunks * D + 64;
}

extern "C" int ul_norm_update(const float* x, int64_t B, int64_t D, int64_t ldx, double* state,
                              void* work, int frozen, void* stream) {
  UL_CHECK_ARG(B >= 0 && D >= 1 && ldx >= D, "normalizer: bad shape");
  if (B == 0 || frozen) return UL_OK;
  const int64_t col_tiles = ul::ceil_div(D, ul::kColTile);
  int64_t chunks = ul::ceil_div(2 * ul::kNumSMs, col_tiles);
  const int64_t cap = ul::ceil_div(B, 64);
  chunks = chunks < cap ? chunks : cap;
  chunks = chunks < 1 ? 1 : (chunks > ul::kMaxChunks ? ul::kMaxChunks : chunks);
  const int64_t rows_per = ul::ceil_div(B, chunks);
  chunks = ul::ceil_div(B, rows_per);
  double* partial = reinterpret_cast<double*>(work);
  unsigned int* ticket =
      reinterpret_cast<unsigned int*>(reinterpret_cast<char*>(work) + ul_norm_work_bytes(D) - 64);
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
