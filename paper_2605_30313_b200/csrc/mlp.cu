// MLP forward / backward drivers over the two GEMM back ends (R:tensornet/mlp.py:153-198).
//
// Activation layout: hidden layer i output h_i is [M, ld_i] with
// ld_i = round_up(d_i + 1, 4): 16-byte rows (TMA-legal) plus one spare column
// that the tensor-core forward epilogue fills with 1.0.  That "ones column"
// turns every dW GEMM into [dW | db] = dZ^T [H | 1]: the bias gradient falls
// out of the same tcgen05 GEMM instead of a separate column-sum pass.
// Weights for the tensor-core path are staged per step into 16-byte-aligned
// padded rows (ul_stage_weights) since the reference flat layout
// (R:tensornet/mlp.py:53-57) puts W0 rows at 940-byte pitch.
// Back ends: 0 = fp32 SIMT (exact-fp32 parity path), 1 = tcgen05 kind::tf32.
// Per GEMM the tensor-core path is used when the shape fills a 128-row UMMA
// tile (the 12-/1-wide heads stay on the SIMT kernel).
#include <cuda_bf16.h>

#include "internal.cuh"
#include "opt_tail.cuh"

namespace ul {

int gemm_tc(const GemmDesc& d, int ones_col, cudaStream_t s);
int gemm_tc_group(const GemmDesc& d0, const GemmDesc& d1, cudaStream_t s);
int gemm_tc_group_n(const GemmDesc* d, int n, cudaStream_t s);
bool tc_eligible(const GemmDesc& d);
int tc_num_splits(int64_t K, int splits, int dtype);
bool tc_dw_pairs();
bool skinny_ok(int N, int K);
int64_t skinny_part_floats(int64_t M, int K, int N);
int skinny_fwd(const void* h, int64_t ldh, int64_t M, int K, int N, const float* W,
               const float* b, float* out, int64_t ldo, int dtype, cudaStream_t s);
int skinny_bwd(const void* h, int64_t ldh, int64_t M, int K, int N, const float* W,
               const float* dout, int64_t ldd, void* dh, int64_t lddh, bool elu_grad, float* gw,
               float* gb, float* gcs, float* part, int dtype, ReduceJob* defer, cudaStream_t s);

namespace {

int64_t rup(int64_t x, int64_t m) { return ceil_div(x, m) * m; }

// ws: splits x [out, ldp] fp32 partials (ldp % 4 == 0); column `in` is the
// bias gradient, columns > in are TMA-row padding.  A warp owns 128 columns
// (float4 lanes) and the splits z = w, w + 8, ... with every load issued
// before the adds; the 8 warps combine in fixed order (deterministic).
struct ReduceTable {
  ReduceJob r[kMaxReduceJobs];  // blockIdx.y selects the job
};

template <int W>  // warps per block: 8 for split-K depths (<= 64), 32 for deep partial sets
__global__ void __launch_bounds__(W * 32) reduce_dw_kernel(ReduceTable tab) {
  __shared__ float4 sm[W][32];
  const ReduceJob& q = tab.r[blockIdx.y];
  const float* __restrict__ ws = q.src;
  const int splits = q.nz;
  const int64_t in = q.in, ldp = q.ldp;
  float* __restrict__ gw = q.gw;
  float* __restrict__ gb = q.gb;
  const int64_t len = q.len;
  pdl_trigger();
  pdl_wait();
  if ((int64_t)blockIdx.x * 128 >= len) return;  // block-uniform
  // W warps over the partials (z = w, w + W, ...), 8 loads in flight each:
  // one round trip for a 35-split dW (W = 8) or a 384-deep head set (W = 32)
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t j = ((int64_t)blockIdx.x * 32 + lane) * 4;
  float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
  if (j < len) {
    for (int z0 = w; z0 < splits; z0 += 8 * W) {
      float4 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int z = z0 + W * u;
        v[u] = z < splits ? __ldg(reinterpret_cast<const float4*>(ws + (int64_t)z * len + j))
                          : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        s.x += v[u].x;
        s.y += v[u].y;
        s.z += v[u].z;
        s.w += v[u].w;
      }
    }
  }
  sm[w][lane] = s;
  __syncthreads();
  if (w == 0 && j < len) {
    float4 t = sm[0][lane];
    for (int k = 1; k < W; ++k) {
      const float4 q4 = sm[k][lane];
      t.x += q4.x;
      t.y += q4.y;
      t.z += q4.z;
      t.w += q4.w;
    }
    const float tv[4] = {t.x, t.y, t.z, t.w};
    if (q.kind == 0) {
      const int64_t r = j / ldp, c0 = j - r * ldp;  // 4 | ldp: one row per float4
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int64_t c = c0 + e;
        if (c < in) gw[r * in + c] = tv[e];
        else if (c == in && gb) gb[r] = tv[e];
      }
    } else {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int64_t c = j + e;
        if (c < q.n0) {
          if (q.o0) q.o0[c] = tv[e];
        } else if (c < q.n0 + q.n1) {
          if (q.o1) q.o1[c - q.n0] = tv[e];
        } else if (c < q.n0 + q.n1 + q.n2) {
          if (q.o2) q.o2[c - q.n0 - q.n1] = tv[e];
        }
      }
    }
  }
}

constexpr int kShallowZ = 64;
struct ReduceAll {
  ReduceJob r[kMaxReduceJobs];
  int end[kMaxReduceJobs];
  int n;
  SqFold fold;
};

// (fold) value v stored at address a: sum of squares / finiteness per segment
struct FoldAcc {
  double s0 = 0.0, s1 = 0.0;
  int bad = 0;
  __device__ __forceinline__ void add(const SqFold& f, const float* a, float v) {
    const int64_t o = (int64_t)((uintptr_t)a - (uintptr_t)f.base) / (int64_t)sizeof(float);
    if (o >= 0 && o < f.n0) {
      s0 += (double)v * (double)v;
      bad |= isfinite(v) ? 0 : 1;
    } else if (o >= f.n0 && o < f.n0 + f.n1) {
      s1 += (double)v * (double)v;
      bad |= isfinite(v) ? 0 : 2;
    }
  }
};

template <bool FOLD>
__device__ __forceinline__ void reduce_store(const ReduceJob& q, int64_t j, float4 t, const SqFold& f,
                                             FoldAcc& fa) {
  const float tv[4] = {t.x, t.y, t.z, t.w};
  if (q.kind == 0) {
    const int64_t r = j / q.ldp, c0 = j - r * q.ldp;  // 4 | ldp: one row per float4
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int64_t c = c0 + e;
      float* dst = nullptr;
      if (c < q.in) dst = q.gw + r * q.in + c;
      else if (c == q.in && q.gb) dst = q.gb + r;
      if (dst) {
        *dst = tv[e];
        if (FOLD) fa.add(f, dst, tv[e]);
      }
    }
  } else {
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int64_t c = j + e;
      float* dst = nullptr;
      if (c < q.n0) {
        if (q.o0) dst = q.o0 + c;
      } else if (c < q.n0 + q.n1) {
        if (q.o1) dst = q.o1 + (c - q.n0);
      } else if (c < q.n0 + q.n1 + q.n2) {
        if (q.o2) dst = q.o2 + (c - q.n0 - q.n1);
      }
      if (dst) {
        *dst = tv[e];
        if (FOLD) fa.add(f, dst, tv[e]);
      }
    }
  }
}

// Every partial reduction of a pass in ONE launch.  Blocks [end[i-1], end[i])
// belong to job i.  Shallow jobs (split-K dW, nz <= kShallowZ): one thread per
// float4 column, all of its nz loads in flight, summed in z order.  Deep jobs
// (per-block / per-CTA partial sets): 8 float4 columns per block, 32 z-phases
// combined in fixed order.  Deterministic.  FOLD: the K13 prepare pass rides
// along (SqFold) -- per-block sum g^2 / non-finite partials of the stored
// gradients, the last block runs the prepare tail, so the Adam apply kernel
// follows this launch directly.
template <bool FOLD>
__global__ void __launch_bounds__(256) reduce_all_kernel(const __grid_constant__ ReduceAll tab) {
  __shared__ float4 sm[8][32];
  int ji = 0;
  while (ji < tab.n - 1 && (int)blockIdx.x >= tab.end[ji]) ++ji;
  const ReduceJob& q = tab.r[ji];
  const int blk = (int)blockIdx.x - (ji ? tab.end[ji - 1] : 0);
  FoldAcc fa;
  pdl_trigger();
  pdl_wait();
  const float* __restrict__ ws = q.src;
  const int nz = q.nz;
  if (nz <= kShallowZ) {
    const int64_t j = ((int64_t)blk * 256 + threadIdx.x) * 4;
    if (j < q.len) {
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int z0 = 0; z0 < nz; z0 += 8) {
        float4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u)
          v[u] = z0 + u < nz ? __ldg(reinterpret_cast<const float4*>(ws + (int64_t)(z0 + u) * q.len + j))
                             : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          acc.x += v[u].x;
          acc.y += v[u].y;
          acc.z += v[u].z;
          acc.w += v[u].w;
        }
      }
      reduce_store<FOLD>(q, j, acc, tab.fold, fa);
    }
  } else {
    // deep sets: 8 float4 columns per CTA, 32 z-phases (the CTA's 256 threads)
    // each summing z = phase, phase + 32, ... with 8 loads in flight, then a
    // fixed-order combine of the phases
    const int c8 = threadIdx.x & 7, ph = threadIdx.x >> 3;
    const int64_t j = ((int64_t)blk * 8 + c8) * 4;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    if (j < q.len) {
      for (int z0 = ph; z0 < nz; z0 += 32 * 8) {
        float4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int z = z0 + 32 * u;
          v[u] = z < nz ? __ldg(reinterpret_cast<const float4*>(ws + (int64_t)z * q.len + j))
                        : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          acc.x += v[u].x;
          acc.y += v[u].y;
          acc.z += v[u].z;
          acc.w += v[u].w;
        }
      }
    }
    float4* sp = &sm[0][0];  // [32 phases][8 columns]
    sp[ph * 8 + c8] = acc;
    __syncthreads();
    if (ph == 0 && j < q.len) {
      float4 t = sp[c8];
      for (int k = 1; k < 32; ++k) {
        const float4 q4 = sp[k * 8 + c8];
        t.x += q4.x;
        t.y += q4.y;
        t.z += q4.z;
        t.w += q4.w;
      }
      reduce_store<FOLD>(q, j, t, tab.fold, fa);
    }
  }
  if constexpr (FOLD) {
    __shared__ double scratch[32];
    const SqFold& F = tab.fold;
    const double t0 = block_sum(fa.s0, scratch);
    const double t1 = block_sum(fa.s1, scratch + 16);
    const int any0 = __syncthreads_or(fa.bad & 1), any1 = __syncthreads_or(fa.bad & 2);
    if (threadIdx.x == 0) {
      F.part[2 * blockIdx.x] = t0;
      F.part[2 * blockIdx.x + 1] = t1;
      F.bad[2 * blockIdx.x] = any0 ? 1 : 0;
      F.bad[2 * blockIdx.x + 1] = any1 ? 1 : 0;
    }
    if (!last_block_ticket(F.ticket, gridDim.x)) return;
    prepare_tail(2, F.part, F.bad, 2, F.ctl, F.lf, 1, (int)gridDim.x, scratch);
  }
}

__device__ __forceinline__ float to_f(float v) { return v; }
__device__ __forceinline__ float to_f(__nv_bfloat16 v) { return __bfloat162float(v); }

// db partials: column sums of dh [M, N] over row chunks; a thread owns 8
// consecutive columns (one 16 B bf16 / 2 x 16 B fp32 load per row), 8 warps
// stride the rows with 4 rows in flight; part[chunk][N].  Needs ld % 8 == 0
// and a 16 B-aligned base (the hidden-gradient buffers).
template <typename T>
__device__ __forceinline__ void load8(const T* p, float (&f)[8]);
template <>
__device__ __forceinline__ void load8<float>(const float* p, float (&f)[8]) {
  const float4 a = __ldg(reinterpret_cast<const float4*>(p));
  const float4 b = __ldg(reinterpret_cast<const float4*>(p) + 1);
  f[0] = a.x; f[1] = a.y; f[2] = a.z; f[3] = a.w; f[4] = b.x; f[5] = b.y; f[6] = b.z; f[7] = b.w;
}
template <>
__device__ __forceinline__ void load8<__nv_bfloat16>(const __nv_bfloat16* p, float (&f)[8]) {
  const uint4 u = __ldg(reinterpret_cast<const uint4*>(p));
  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    f[2 * i] = __uint_as_float(w[i] << 16);
    f[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
  }
}

template <typename T>
__global__ void __launch_bounds__(256) colsum_kernel(const T* __restrict__ x, int64_t ld,
                                                     int64_t M, int64_t N, int64_t rows_per,
                                                     float* __restrict__ part) {
  __shared__ float sm[8][32 * 8 + 1];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t c = ((int64_t)blockIdx.x * 32 + lane) * 8;  // first of 8 columns
  const int64_t r0 = (int64_t)blockIdx.y * rows_per;
  const int64_t r1 = r0 + rows_per < M ? r0 + rows_per : M;
  pdl_trigger();
  pdl_wait();
  float s[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  if (c < N && c + 8 > ld) {
    // row tail narrower than 8 columns of pitch: scalar loads
    for (int64_t r = r0 + w; r < r1; r += 8)
      for (int i = 0; i < 8 && c + i < N; ++i) s[i] += to_f(x[r * ld + c + i]);
  } else if (c < N) {
    int64_t r = r0 + w;
    for (; r + 24 < r1; r += 32) {
      float f[4][8];
#pragma unroll
      for (int k = 0; k < 4; ++k) load8<T>(x + (r + 8 * k) * ld + c, f[k]);
#pragma unroll
      for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int i = 0; i < 8; ++i) s[i] += f[k][i];
    }
    for (; r < r1; r += 8) {
      float f[8];
      load8<T>(x + r * ld + c, f);
#pragma unroll
      for (int i = 0; i < 8; ++i) s[i] += f[i];
    }
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) sm[w][lane * 8 + i] = s[i];
  __syncthreads();
  for (int q = threadIdx.x; q < 256; q += blockDim.x) {
    const int64_t cc = (int64_t)blockIdx.x * 256 + q;
    if (cc >= N) continue;
    float t = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) t += sm[k][q];
    part[(int64_t)blockIdx.y * N + cc] = t;
  }
}

// fp32 rows -> bf16 rows (the upstream gradient of a wide output layer on the
// bf16 path)
// out[j][c] = W[c][col0 + j]: the input-gradient column slice, transposed
__global__ void slice_t_kernel(const float* __restrict__ W, int ldw, int col0, int nc, int K,
                               float* __restrict__ out) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)nc * K) return;
  const int c = (int)(e % K), j = (int)(e / K);
  out[e] = W[(int64_t)c * ldw + col0 + j];
}

__global__ void f32_to_bf16_kernel(const float* __restrict__ x, int64_t ldx, int64_t M,
                                   int64_t N, __nv_bfloat16* __restrict__ y, int64_t ldy) {
  const int64_t total = M * N;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += stride) {
    const int64_t r = i / N, c = i - r * N;
    y[r * ldy + c] = __float2bfloat16_rn(x[r * ldx + c]);
  }
}

struct StageTable {
  int n;
  int64_t src_off[UL_MAX_LAYERS], dst_off[UL_MAX_LAYERS];
  int rows[UL_MAX_LAYERS], cols[UL_MAX_LAYERS], ld[UL_MAX_LAYERS];
  int64_t total;  // padded elements
};

template <typename T>
__global__ void stage_weights_kernel(const float* __restrict__ params, StageTable t,
                                     T* __restrict__ wp) {
  pdl_trigger();
  pdl_wait();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < t.total; j += stride) {
    int l = 0;
    while (l + 1 < t.n && j >= t.dst_off[l + 1]) ++l;
    const int64_t k = j - t.dst_off[l];
    const int64_t r = k / t.ld[l], c = k - r * t.ld[l];
    wp[j] = (T)(c < t.cols[l] ? params[t.src_off[l] + r * t.cols[l] + c] : 0.f);
  }
}

}  // namespace

int64_t act_ld(int d, int dtype) { return rup((int64_t)d + 1, dtype == kBf16 ? 8 : 4); }

int make_view(const ul_net_desc* d, NetView* v) {
  UL_CHECK_ARG(d != nullptr, "net: null descriptor");
  UL_CHECK_ARG(d->n_layers >= 1 && d->n_layers <= UL_MAX_LAYERS,
               "net: n_layers %d outside [1,%d]", d->n_layers, UL_MAX_LAYERS);
  v->n_layers = d->n_layers;
  v->ln = d->layer_norm ? 1 : 0;
  int64_t off = 0, woff = 0;
  for (int i = 0; i <= d->n_layers; ++i) {
    UL_CHECK_ARG(d->dims[i] > 0, "all layer dims must be positive");
    v->dims[i] = d->dims[i];
  }
  for (int i = 0; i < d->n_layers; ++i) {
    v->w_off[i] = off;
    off += (int64_t)v->dims[i + 1] * v->dims[i];
    v->b_off[i] = off;
    off += v->dims[i + 1];
    v->g_off[i] = v->beta_off[i] = -1;
    if (v->ln && i < d->n_layers - 1) {  // hidden layer: LayerNorm gain / shift
      UL_CHECK_ARG(v->dims[i + 1] % 4 == 0, "layer_norm: hidden widths must be multiples of 4");
      v->g_off[i] = off;
      off += v->dims[i + 1];
      v->beta_off[i] = off;
      off += v->dims[i + 1];
    }
    v->wp_off[i] = woff;
    woff += (int64_t)v->dims[i + 1] * rup(v->dims[i], 4);
  }
  int64_t boff = 0;
  for (int i = 0; i < d->n_layers; ++i) {
    v->wb_off[i] = boff;
    boff += (int64_t)v->dims[i + 1] * rup(v->dims[i], 8);
  }
  v->logstd_off = off;
  v->total = off + v->dims[d->n_layers];
  v->wp_total = woff;
  return UL_OK;
}

int64_t act_floats(const NetView& v, int64_t M) {
  int64_t s = 0;
  for (int i = 1; i < v.n_layers; ++i) s += act_ld(v.dims[i]) * M;
  if (v.ln)  // pre-LayerNorm rows + row stats per hidden layer
    for (int i = 1; i < v.n_layers; ++i) s += (rup(v.dims[i], 4) + 2) * M;
  return s;
}

// pre-LN rows in bf16 on the bf16 back end (UL_LN_A_BF16=0: fp32 rows)
// the whole LayerNorm forward in the tcgen05 epilogue (kEpiLnFull); read on
// every call (a plan captures its choice), UL_LN_FUSED=0 keeps the separate
// row / column kernels
bool ln_fused_enabled() {
  const char* e = getenv("UL_LN_FUSED");
  return e ? atoi(e) != 0 : true;
}

bool ln_a_bf16(int dtype) {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("UL_LN_A_BF16");
    on = e ? atoi(e) != 0 : 1;
  }
  return dtype == kBf16 && on == 1;
}

void ln_bufs(const NetView& v, const float* acts, int64_t M, int i, float** a, int64_t* lda,
             float** stats) {
  int64_t off = 0;
  for (int j = 1; j < v.n_layers; ++j) off += act_ld(v.dims[j]) * M;
  for (int j = 1; j <= i; ++j) off += (rup(v.dims[j], 4) + 2) * M;
  *lda = rup(v.dims[i + 1], 4);
  *a = const_cast<float*>(acts) + off;
  *stats = *a + *lda * M;
}

static int64_t max_hidden_ld(const NetView& v) {
  int64_t h = 4;
  for (int i = 1; i <= v.n_layers; ++i) h = act_ld(v.dims[i]) > h ? act_ld(v.dims[i]) : h;
  return h;
}

// dW split count: about one persistent wave of tiles, >= 512 batch rows per split
static int dw_splits(int64_t out, int64_t in, int64_t M, bool tc) {
  const int64_t tiles = tc ? ceil_div(out, 128) * ceil_div(in + 1, 256)
                           : ceil_div(out, 128) * ceil_div(in, 128);
  int64_t sp = ceil_div(tc ? kNumSMs : 2 * kNumSMs, tiles);
  const int64_t cap = ceil_div(M, 512);
  sp = sp < cap ? sp : cap;
  sp = sp < 1 ? 1 : sp;
  return (int)(sp > 64 ? 64 : sp);
}

// backward workspace: [hidden-gradient buffers][split-K dW + column-sum
// partials, one region per layer][skinny head partials][dX column-sum
// partials, one region per layer][LayerNorm partials][dX column slice].
// Layer-by-layer backward reuses region 0 and two gradient buffers (the
// head's partials outlive the next layer's dW GEMM: their reduction is folded
// into that layer's reduction); the deferred-dW backward keeps every layer's
// dZ and partials alive until one batched dW launch + one reduction at the end.
static int64_t dw_layer_floats(const NetView& v, int64_t M, int i) {
  const int64_t out = v.dims[i + 1], in = v.dims[i];
  const int sp = dw_splits(out, in, M, false) > dw_splits(out, in, M, true)
                     ? dw_splits(out, in, M, false) : dw_splits(out, in, M, true);
  return rup((int64_t)sp * (out * rup(in + 1, 4) + out) + 256 * out, 64);
}

static int64_t dw_ws_floats(const NetView& v, int64_t M) {
  int64_t ws = 0;
  for (int i = 0; i < v.n_layers; ++i) ws += dw_layer_floats(v, M, i);
  return ws;
}

static int64_t dw_layer_off(const NetView& v, int64_t M, int i) {
  int64_t o = 0;
  for (int j = 0; j < i; ++j) o += dw_layer_floats(v, M, j);
  return o;
}

static int n_dh_bufs(const NetView& v) { return v.n_layers > 2 ? v.n_layers : 2; }
constexpr int64_t kCsRegion = (int64_t)kNumSMs * kCsumMaxN;  // one dX GEMM's column-sum partials

static int64_t sk_ws_floats(const NetView& v, int64_t M) {
  const int last = v.n_layers - 1;
  int64_t sk = skinny_part_floats(M, v.dims[last], v.dims[last + 1]);
  // (the region also holds the dX epilogue's per-CTA column-sum partials)
  sk = sk > (int64_t)kNumSMs * kCsumMaxN ? sk : (int64_t)kNumSMs * kCsumMaxN;
  return rup(sk, 64);
}

// LayerNorm block partials: one region per LN layer (with the deferred dW
// pass every layer's partials live until the single reduction at the end)
static int64_t ln_layer_off(const NetView& v, int64_t M, int i) {
  int64_t o = 0;
  if (v.ln)
    for (int j = 0; j < i && j < v.n_layers - 1; ++j) o += rup(ln_part_floats(M, v.dims[j + 1]), 64);
  return o;
}

// largest 3xTF32 split scratch one GEMM of a pass over M rows needs: the
// forward (A [M, 3Kp], B [N, 3Kp]), the input gradient (A [M, 3 out_p],
// B [3 out_p, ld_in]) and the weight gradient (A [3 Mp, ld_out],
// B [3 Mp, ld_in + ones]) of every layer
size_t x3_bound(const NetView& v, int64_t M) {
  size_t mx = 0;
  // (each split-K chunk is padded to a multiple of 32: at most 64 chunks)
  const int64_t Mk = rup(M, 32) + 32 * 64;
  for (int i = 0; i < v.n_layers; ++i) {
    const int64_t in = v.dims[i], out = v.dims[i + 1];
    const int64_t ip = rup(in + 1, 32), op = rup(out + 1, 32);
    const int64_t ldi = rup(in + 1, 4), ldo = rup(out + 1, 4);
    const size_t fwd = (size_t)(rup(M * 3 * ip, 64) + out * 3 * ip);
    const size_t dx = (size_t)(rup(M * 3 * op, 64) + 3 * op * ldi);
    const size_t dw = (size_t)(rup(3 * Mk * ldo, 64) + 3 * Mk * ldi);
    const size_t m = fwd > dx ? fwd : dx;
    mx = m > mx ? m : mx;
    mx = dw > mx ? dw : mx;
  }
  return mx;
}

int64_t bwd_work_floats(const NetView& v, int64_t M) {
  const int64_t sk = sk_ws_floats(v, M);
  const int64_t lnp = ln_layer_off(v, M, v.n_layers - 1);
  // + the transposed W column slice of the skinny input-gradient path
  return n_dh_bufs(v) * M * max_hidden_ld(v) + dw_ws_floats(v, M) + sk +
         kCsRegion * v.n_layers + rup(lnp, 64) + rup((int64_t)kSkinnyDxMax * v.dims[1], 64);
}

float* bwd_head_dz(const NetView& v, float* work, int64_t M) {
  (void)v;
  (void)M;
  return work;
}

float* bwd_head_part(const NetView& v, float* work, int64_t M) {
  return work + n_dh_bufs(v) * M * max_hidden_ld(v) + dw_ws_floats(v, M);
}

// hidden layer i's activation rows (byte offsets: bf16 rows are half as wide)
const float* act_ptr(const NetView& v, const float* acts, int64_t M, int i, int dtype) {
  const int64_t eb = dtype == kBf16 ? 2 : 4;
  int64_t off = 0;
  for (int j = 1; j <= i; ++j) off += act_ld(v.dims[j], dtype) * M * eb;
  return reinterpret_cast<const float*>(reinterpret_cast<const char*>(acts) + off);
}

int stage_weights_dt(const NetView& v, const float* params, void* wp, int dtype, cudaStream_t s) {
  StageTable t{};
  t.n = v.n_layers;
  const int a = dtype == kBf16 ? 8 : 4;
  for (int i = 0; i < v.n_layers; ++i) {
    t.src_off[i] = v.w_off[i];
    t.dst_off[i] = dtype == kBf16 ? v.wb_off[i] : v.wp_off[i];
    t.rows[i] = v.dims[i + 1];
    t.cols[i] = v.dims[i];
    t.ld[i] = (int)rup(v.dims[i], a);
  }
  const int last = v.n_layers - 1;
  t.total = t.dst_off[last] + (int64_t)t.rows[last] * t.ld[last];
  int64_t blocks = ceil_div(t.total, 256);
  blocks = blocks > 4 * kNumSMs ? 4 * kNumSMs : blocks;
  if (dtype == kBf16)
    return launch_pdl("stage_weights_kernel", stage_weights_kernel<__nv_bfloat16>,
                      dim3((unsigned)blocks), dim3(256), 0, s, params, t,
                      reinterpret_cast<__nv_bfloat16*>(wp));
  return launch_pdl("stage_weights_kernel", stage_weights_kernel<float>, dim3((unsigned)blocks),
                    dim3(256), 0, s, params, t, reinterpret_cast<float*>(wp));
}

// Several networks' staged operand rows in ONE launch (the SAC plan restages
// actor, q1, q2 and both targets every update): warp per staged row, lanes
// across the row (coalesced), zero padding to the 16-byte pitch.
constexpr int kMultiStage = 5 * UL_MAX_LAYERS;
struct MultiStage {
  const float* src[kMultiStage];
  void* dst[kMultiStage];
  int cols[kMultiStage], ld[kMultiStage];
  int64_t row0[kMultiStage + 1];  // prefix sums of rows
  int n;
};

template <typename T>
__global__ void stage_multi_kernel(const __grid_constant__ MultiStage t) {
  pdl_trigger();
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < t.row0[t.n];
       r += nw) {
    int e = 0;
    while (e + 1 < t.n && r >= t.row0[e + 1]) ++e;
    const int64_t rr = r - t.row0[e];
    const float* s = t.src[e] + rr * t.cols[e];
    T* d = reinterpret_cast<T*>(t.dst[e]) + rr * t.ld[e];
    for (int c = lane; c < t.ld[e]; c += 32) d[c] = (T)(c < t.cols[e] ? s[c] : 0.f);
  }
}

int stage_weights_multi(int n, const NetView* const* v, const float* const* params,
                        void* const* wp, int dtype, cudaStream_t s) {
  MultiStage t{};
  const int a = dtype == kBf16 ? 8 : 4;
  const int eb = dtype == kBf16 ? 2 : 4;
  int e = 0;
  t.row0[0] = 0;
  for (int k = 0; k < n; ++k)
    for (int i = 0; i < v[k]->n_layers; ++i) {
      UL_CHECK_ARG(e < kMultiStage, "stage_weights_multi: too many layers");
      t.src[e] = params[k] + v[k]->w_off[i];
      t.dst[e] = reinterpret_cast<char*>(wp[k]) +
                 (dtype == kBf16 ? v[k]->wb_off[i] : v[k]->wp_off[i]) * eb;
      t.cols[e] = v[k]->dims[i];
      t.ld[e] = (int)rup(v[k]->dims[i], a);
      t.row0[e + 1] = t.row0[e] + v[k]->dims[i + 1];
      ++e;
    }
  t.n = e;
  int64_t blocks = ceil_div(t.row0[e], 8);
  blocks = blocks > 8 * kNumSMs ? 8 * kNumSMs : (blocks < 1 ? 1 : blocks);
  if (dtype == kBf16)
    return launch_pdl("stage_multi_kernel", stage_multi_kernel<__nv_bfloat16>,
                      dim3((unsigned)blocks), dim3(256), 0, s, t);
  return launch_pdl("stage_multi_kernel", stage_multi_kernel<float>, dim3((unsigned)blocks),
                    dim3(256), 0, s, t);
}

int stage_weights(const NetView& v, const float* params, float* wp, cudaStream_t s) {
  return stage_weights_dt(v, params, wp, kF32, s);
}

// staged W_i for a dtype and its row pitch (elements)
static const float* staged_w(const NetView& v, const float* wp, int i, int dtype, int64_t* ld) {
  if (dtype == kBf16) {
    *ld = rup(v.dims[i], 8);
    return reinterpret_cast<const float*>(reinterpret_cast<const __nv_bfloat16*>(wp) +
                                          v.wb_off[i]);
  }
  *ld = rup(v.dims[i], 4);
  return wp + v.wp_off[i];
}

static int run_gemm(GemmDesc g, bool use_tc, int ones_col, cudaStream_t s) {
  g.ones_col = ones_col;
  if (use_tc && tc_eligible(g)) return gemm_tc(g, ones_col, s);
  UL_CHECK_ARG(g.dtype == kF32, "bf16 MLP: GEMM %lldx%lldx%lld not tensor-core eligible "
               "(alignment)", (long long)g.M, (long long)g.N, (long long)g.K);
  return gemm_f32(g, s);
}

static bool al16(const void* p, int64_t ld, int eb) {
  return ((uintptr_t)p & 15) == 0 && (ld * eb) % 16 == 0;
}

// ---------------------------------------------------------------- drivers
// One or two networks advance layer by layer in lockstep: their tensor-core
// GEMMs of a layer share one grouped launch (gemm_tc_group), the per-network
// small kernels (skinny heads, split-K reductions, column sums) of network 1
// run on the side lane.
namespace {

struct Lanes {
  cudaStream_t s, side;
  cudaEvent_t fork, join;
  cudaStream_t of(int k) const { return k == 1 && side ? side : s; }
  int open() const {
    if (!side) return UL_OK;
    UL_CUDA(cudaEventRecord(fork, s));
    UL_CUDA(cudaStreamWaitEvent(side, fork, 0));
    return UL_OK;
  }
  int close() const {
    if (!side) return UL_OK;
    UL_CUDA(cudaEventRecord(join, side));
    UL_CUDA(cudaStreamWaitEvent(s, join, 0));
    return UL_OK;
  }
};

// one launch for up to kMaxReduceJobs fixed-order partial reductions
// fold (may be null): run the K13 prepare pass inside the reduction when
// every job fits one launch and the block partials fit the fold's arrays;
// *folded (may be null) tells the caller whether it did
int launch_reduce(const ReduceJob* jobs, int nj, cudaStream_t s, const SqFold* fold = nullptr,
                  bool* folded = nullptr) {
  static int one = -1;
  if (one < 0) {
    const char* e = getenv("UL_REDUCE_ONE");
    one = e ? atoi(e) != 0 : 1;
  }
  if (folded) *folded = false;
  if (one) {
    // every job in one launch (reduce_all_kernel), kMaxReduceJobs per launch
    int live = 0;
    for (int q = 0; q < nj; ++q) live += (jobs[q].len > 0 && jobs[q].nz > 0) ? 1 : 0;
    for (int q = 0; q < nj;) {
      ReduceAll tab{};
      int blocks = 0;
      for (; q < nj && tab.n < kMaxReduceJobs; ++q) {
        if (jobs[q].len <= 0 || jobs[q].nz <= 0) continue;
        tab.r[tab.n] = jobs[q];
        const int64_t cols = ceil_div(jobs[q].len, 4);
        blocks += (int)ceil_div(cols, jobs[q].nz <= kShallowZ ? 256 : 8);
        tab.end[tab.n++] = blocks;
      }
      if (tab.n == 0) continue;
      if (fold && fold->on && live <= kMaxReduceJobs && blocks <= fold->cap) {
        tab.fold = *fold;
        UL_TRY(launch_pdl("reduce_all_kernel", reduce_all_kernel<true>, dim3((unsigned)blocks),
                          dim3(256), 0, s, tab));
        if (folded) *folded = true;
      } else {
        UL_TRY(launch_pdl("reduce_all_kernel", reduce_all_kernel<false>, dim3((unsigned)blocks),
                          dim3(256), 0, s, tab));
      }
    }
    return UL_OK;
  }
  // shallow (split-K) and deep (per-block / per-CTA partial) jobs take the
  // 8- and 32-warp variants; at most kMaxReduceJobs per launch
  for (int deep = 0; deep < 2; ++deep) {
    int q = 0;
    while (q < nj) {
      ReduceTable tab{};
      int64_t bx = 1;
      int cnt = 0;
      for (; q < nj && cnt < kMaxReduceJobs; ++q) {
        if ((jobs[q].nz > 64) != (deep == 1)) continue;
        tab.r[cnt++] = jobs[q];
        const int64_t b = ceil_div(jobs[q].len, 128);
        bx = b > bx ? b : bx;
      }
      if (cnt == 0) continue;
      if (deep)
        UL_TRY(launch_pdl("reduce_dw_kernel", reduce_dw_kernel<32>,
                          dim3((unsigned)bx, (unsigned)cnt), dim3(1024), 0, s, tab));
      else
        UL_TRY(launch_pdl("reduce_dw_kernel", reduce_dw_kernel<8>,
                          dim3((unsigned)bx, (unsigned)cnt), dim3(256), 0, s, tab));
    }
  }
  return UL_OK;
}

// run 1 to kMaxNets independent GEMMs (n: how many slots); when every
// present one runs on the tensor cores they share one grouped launch
int run_gemms(GemmDesc* g, const bool* has, const bool* use_tc, const int* ones, cudaStream_t s,
              int n = 2) {
  bool tc_ok[kMaxNets];
  int n_has = 0, n_tc = 0;
  for (int k = 0; k < n; ++k) {
    g[k].ones_col = ones[k];
    tc_ok[k] = has[k] && use_tc[k] && tc_eligible(g[k]);
    n_has += has[k];
    n_tc += tc_ok[k];
  }
  if (n == 2 && tc_ok[0] && tc_ok[1]) return gemm_tc_group(g[0], g[1], s);
  if (n > 2 && n_tc == n_has && n_tc > 1) {
    GemmDesc q[kMaxNets];
    int m = 0;
    for (int k = 0; k < n; ++k)
      if (has[k]) q[m++] = g[k];
    return gemm_tc_group_n(q, m, s);
  }
  for (int k = 0; k < n; ++k)
    if (has[k]) UL_TRY(run_gemm(g[k], use_tc[k], ones[k], s));
  return UL_OK;
}

bool ones_free_of(int64_t n_in, bool ones) {
  auto bn_of = [](int64_t n) { return n > 128 ? 256 : 128; };
  return ones && bn_of(n_in + 1) == bn_of(n_in) &&
         ceil_div(n_in + 1, bn_of(n_in + 1)) == ceil_div(n_in, bn_of(n_in));
}

}  // namespace

bool head_needs_colsum(const MlpNet& N) {
  const NetView& v = *N.v;
  const int nl = v.n_layers;
  if (nl < 2 || !N.want_dw || !N.wp || v.ln) return false;
  const int64_t in_below = v.dims[nl - 2];
  const bool below_ones = nl - 2 == 0 ? N.x_has_ones && N.ldx >= in_below + 1 : true;
  return !ones_free_of(in_below, below_ones);
}

// Chained hidden layers (gemm_tc_chain; opt-in UL_CHAIN_FWD=1): bf16, no
// LayerNorm, 1-2 networks of equal hidden widths, shallow K.  Bit-identical
// to one launch per layer; measured 4.40 vs 4.31 ms per cfg2 update (the
// three launches serialised under ncu: 66.0 vs 65.9 us) -- the in-kernel
// handoff between a chain's layers (stores landed -> next layer's loads)
// costs what the launch boundaries did, and the chain gives up the
// B-resident first / last layers
constexpr int kMaxChainLayers = 4;
static bool chain_fwd_ok(const MlpNet* nets, int n, int dt, int64_t M) {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("UL_CHAIN_FWD");
    on = e ? atoi(e) != 0 : 0;
  }
  if (!on || dt != kBf16 || n < 1 || n > 2 || M <= 0 || M >= (int64_t(1) << 31)) return false;
  const NetView& v0 = *nets[0].v;
  const int L = v0.n_layers - 1;
  if (L < 2 || L > kMaxChainLayers) return false;
  for (int k = 0; k < n; ++k) {
    const NetView& v = *nets[k].v;
    if (v.ln || !nets[k].wp || v.n_layers != v0.n_layers) return false;
    if (((uintptr_t)nets[k].x & 15) || (nets[k].ldx * 2) % 16) return false;
    for (int i = 1; i <= L; ++i)
      if (v.dims[i] != v0.dims[i]) return false;  // (equal widths per layer)
    // (deep-K layers -- the FlashSAC 1024-wide critics -- run better as CTA-pair launches)
    for (int i = 0; i < L; ++i)
      if (v.dims[i] > 512) return false;
  }
  return true;
}

int mlp_forward_n(const MlpNet* nets, int n, int backend, int64_t M, cudaStream_t s,
                  cudaStream_t side, cudaEvent_t fork, cudaEvent_t join) {
  UL_CHECK_ARG(n >= 1 && n <= kMaxNets, "mlp_forward_n: 1..kMaxNets networks");
  for (int k = 1; k < n; ++k)
    if (nets[k].v->n_layers != nets[0].v->n_layers) {  // (lockstep needs equal depths)
      for (int j = 0; j < n; ++j)
        UL_TRY(mlp_forward_n(nets + j, 1, backend, M, s, nullptr, nullptr, nullptr));
      return UL_OK;
    }
  const Lanes L{s, n == 2 ? side : nullptr, fork, join};
  const int dt = backend_dtype(backend);
  const int eb = dt == kBf16 ? 2 : 4;
  const bool tc = backend >= 1;
  const float* h[kMaxNets];
  int64_t ldh[kMaxNets];
  for (int k = 0; k < n; ++k) {
    UL_CHECK_ARG(dt == kF32 || nets[k].wp, "bf16 MLP needs staged weights");
    h[k] = nets[k].x;
    ldh[k] = nets[k].ldx;
  }
  const int nl = nets[0].v->n_layers;
  bool ln_pending[kMaxNets] = {};
  int i0 = 0;
  if (tc && fused_fwd_ok(nets, n, dt)) {  // every hidden layer in one launch
    UL_TRY(fused_forward(nets, n, M, s));
    for (int k = 0; k < n; ++k) {
      h[k] = act_ptr(*nets[k].v, nets[k].acts, M, nl - 2, dt);
      ldh[k] = act_ld(nets[k].v->dims[nl - 1], dt);
    }
    i0 = nl - 1;
  } else if (tc && chain_fwd_ok(nets, n, dt, M)) {
    // every hidden layer of both networks as one chained tcgen05 launch (row
    // chains per CTA, gemm_tc_chain); the output layers follow as usual
    const int L = nl - 1;
    GemmDesc g[2 * kMaxChainLayers] = {};
    for (int k = 0; k < n; ++k) {
      const MlpNet& N = nets[k];
      const NetView& v = *N.v;
      for (int i = 0; i < L; ++i) {
        GemmDesc& G = g[k * L + i];
        G.M = M; G.N = v.dims[i + 1]; G.K = v.dims[i];
        G.A = i == 0 ? N.x : act_ptr(v, N.acts, M, i - 1, dt);
        G.lda = i == 0 ? N.ldx : act_ld(v.dims[i], dt);
        G.B = staged_w(v, N.wp, i, dt, &G.ldb);
        G.bias = N.params + v.b_off[i];
        G.C = const_cast<float*>(act_ptr(v, N.acts, M, i, dt));
        G.ldc = act_ld(v.dims[i + 1], dt);
        G.a_kmajor = true; G.b_kmajor = true;
        G.epi = kEpiBiasElu; G.splits = 1; G.dtype = dt;
        G.ones_col = (int)v.dims[i + 1];
      }
      h[k] = act_ptr(v, N.acts, M, L - 1, dt);
      ldh[k] = act_ld(v.dims[L], dt);
    }
    UL_TRY(gemm_tc_chain(g, n, L, s));
    i0 = L;
  }
  for (int i = i0; i < nl; ++i) {
    const bool last = i == nl - 1;
    GemmDesc g[kMaxNets] = {};
    bool has[kMaxNets] = {}, use[kMaxNets] = {}, skinny[kMaxNets] = {};
    bool ln_full[kMaxNets] = {};
    int ones[kMaxNets] = {-1, -1, -1, -1};
    bool any_skinny = false;
    for (int k = 0; k < n; ++k) {
      const MlpNet& N = nets[k];
      const NetView& v = *N.v;
      if (last && N.head_external) continue;  // the fused output stage computes it
      float* dst = last ? N.out : const_cast<float*>(act_ptr(v, N.acts, M, i, dt));
      const int64_t lddst = last ? N.ld_out : act_ld(v.dims[i + 1], dt);
      if (last && skinny_ok(v.dims[i + 1], v.dims[i]) && al16(h[k], ldh[k], eb)) {
        skinny[k] = any_skinny = true;  // 12-/1-wide head, launched below
        continue;
      }
      GemmDesc& G = g[k];
      G.M = M; G.N = v.dims[i + 1]; G.K = v.dims[i];
      G.A = h[k]; G.lda = ldh[k];
      G.bias = N.params + v.b_off[i];
      G.a_kmajor = true; G.b_kmajor = true;
      G.epi = last ? kEpiBias : kEpiBiasElu;
      G.splits = 1;
      G.C = dst; G.ldc = lddst;
      G.dtype = dt;
      G.x3 = backend == kBackendTf32x3;
      if (v.ln && !last) {  // a = W x + b -> LayerNorm + ELU kernel below
        float* la;
        float* lst;
        int64_t lla;
        ln_bufs(v, N.acts, M, i, &la, &lla, &lst);
        // bf16 back end: the epilogue writes the pre-LN rows as bf16 (half
        // the bytes the LN kernels stream in the forward and the backward)
        const bool abf = ln_a_bf16(dt);
        G.epi = abf ? kEpiBiasLn : kEpiBias;
        G.C = la;
        G.ldc = abf ? rup(v.dims[i + 1], 8) : lla;
        ln_pending[k] = true;
        if (abf && tc && N.wp && ln_fused_enabled() && v.dims[i + 1] <= kLnFullMaxN) {
          // the whole LayerNorm in the GEMM epilogue (row statistics across
          // a cluster of N-tile CTAs): a, h and the row stats in one launch
          GemmDesc T = G;
          T.B = staged_w(v, N.wp, i, dt, &T.ldb);
          T.epi = kEpiLnFull;
          T.ln_h = dst;
          T.ldh = lddst;
          T.ln_g = N.params + v.g_off[i];
          T.ln_beta = N.params + v.beta_off[i];
          T.ln_stats = lst;
          T.ln_h_ones = (int)v.dims[i + 1];
          if (tc_eligible(T) && ((uintptr_t)lst & 7) == 0 && ((uintptr_t)dst & 15) == 0 &&
              (lddst * 2) % 16 == 0) {
            G.epi = kEpiLnFull;
            G.ln_h = T.ln_h;
            G.ldh = T.ldh;
            G.ln_g = T.ln_g;
            G.ln_beta = T.ln_beta;
            G.ln_stats = T.ln_stats;
            G.ln_h_ones = T.ln_h_ones;
            ln_pending[k] = false;
            ln_full[k] = true;
          }
        }
      }
      // tf32 keeps a wide output layer on the SIMT kernel; bf16 runs it on
      // the tensor cores with an fp32 bias epilogue
      use[k] = tc && N.wp && (!last || dt == kBf16);
      if (use[k]) {
        G.B = staged_w(v, N.wp, i, dt, &G.ldb);
      } else {
        G.B = N.params + v.w_off[i];
        G.ldb = v.dims[i];
      }
      has[k] = true;
      ones[k] = (last || ln_pending[k] || ln_full[k]) ? -1 : v.dims[i + 1];
      h[k] = dst;
      ldh[k] = lddst;
    }
    UL_TRY(run_gemms(g, has, use, ones, s, n > 2 ? n : 2));
    for (int k = 0; k < n; ++k) {
      if (!ln_pending[k]) continue;
      ln_pending[k] = false;
      const MlpNet& N = nets[k];
      const NetView& v = *N.v;
      float* la;
      float* lst;
      int64_t lla;
      ln_bufs(v, N.acts, M, i, &la, &lla, &lst);
      const bool abf = ln_a_bf16(dt);
      UL_TRY(ln_forward(la, abf ? rup(v.dims[i + 1], 8) : lla, M, v.dims[i + 1],
                        N.params + v.g_off[i], N.params + v.beta_off[i], lst,
                        const_cast<float*>(h[k]), ldh[k], v.dims[i + 1], dt, s, abf));
    }
    if (any_skinny) {
      UL_TRY(L.open());
      for (int k = 0; k < n; ++k) {
        if (!skinny[k]) continue;
        const MlpNet& N = nets[k];
        const NetView& v = *N.v;
        UL_TRY(skinny_fwd(h[k], ldh[k], M, v.dims[i], v.dims[i + 1], N.params + v.w_off[i],
                          N.params + v.b_off[i], N.out, N.ld_out, dt, L.of(k)));
      }
      UL_TRY(L.close());
    }
  }
  return UL_OK;
}

// Deferred dW: collected descs + their reductions, launched as one batched
// tensor-core launch and one reduction pass (run_deferred_dw).
bool deferred_dw_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("UL_DEFER_DW");
    on = e ? atoi(e) != 0 : 1;
  }
  return on == 1;
}

void DeferredDw::add(const GemmDesc& g, const ReduceJob& j) {
  if (ndw >= kMax || nj >= 3 * kMax) return;  // (callers stay far below: 2 nets x UL_MAX_LAYERS)
  dw[ndw] = g;
  jobs[nj] = j;
  dw_job[ndw++] = nj++;
}

int run_deferred_dw(DeferredDw& D, cudaStream_t s) {
  UL_TRY(run_deferred_dw_gemms(D, s));
  return run_deferred_dw_reduce(D, s);
}

int run_deferred_dw_gemms(DeferredDw& D, cudaStream_t s) {
  if (D.ndw) {
    // one split count for the batch: about one persistent wave of tile-splits
    // over 85 % of the SMs (CTA pairs: two CTAs per 256-row tile, a lone
    // 128-row tile included).  Measured per update, 85 vs 100 %: cfg2 4.261
    // vs 4.290 ms, APPO cfg5 15.9 vs 16.1 ms, SAC cfg3 / cfg4 unchanged
    // (fewer split partials to reduce; 2-3 waves were slower)
    const int64_t pm = tc_dw_pairs() ? 2 : 1;
    int64_t tiles = 0;
    for (int i = 0; i < D.ndw; ++i)
      tiles += ceil_div(ceil_div(D.dw[i].M, 128), pm) * pm *
               ceil_div(D.dw[i].N, D.dw[i].N > 128 ? 256 : 128);
    static int fill = -1;  // (UL_DW_FILL: percent of the SMs the tile-splits target)
    if (fill < 0) {
      const char* e = getenv("UL_DW_FILL");
      fill = e ? atoi(e) : 85;
      fill = fill < 10 ? 10 : fill;
    }
    int64_t sp = fill * kNumSMs / (100 * (tiles > 0 ? tiles : 1));
    const int64_t cap = ceil_div(D.dw[0].K, 512);
    sp = sp < cap ? sp : cap;
    sp = sp < 1 ? 1 : sp;
    for (int i = 0; i < D.ndw; ++i) {
      // never more splits than the layer's workspace region was sized for
      const int want = (int)(sp < D.max_splits[i] ? sp : D.max_splits[i]);
      D.dw[i].splits = tc_num_splits(D.dw[i].K, want, D.dw[i].dtype);
      D.jobs[D.dw_job[i]].nz = D.dw[i].splits;
    }
    if (!(ablate_mask() & 32)) UL_TRY(gemm_tc_batch(D.dw, D.ndw, s));
  }
  D.ndw = 0;
  return UL_OK;
}

int run_deferred_dw_reduce(DeferredDw& D, cudaStream_t s) {
  D.folded = false;
  if (D.nj && !(ablate_mask() & 64)) UL_TRY(launch_reduce(D.jobs, D.nj, s, D.fold, &D.folded));
  D.ndw = D.nj = 0;
  return UL_OK;
}

// LayerNorm networks join the deferred dW pass (UL_LN_DEFER=0: per-layer dW)
static bool ln_defer_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("UL_LN_DEFER");
    on = e ? atoi(e) != 0 : 1;
  }
  return on == 1;
}

int mlp_backward_n(const MlpNet* nets, int n, int backend, int64_t M, cudaStream_t s,
                   cudaStream_t side, cudaEvent_t fork, cudaEvent_t join, DeferredDw* dd) {
  if (n == 2 && nets[0].v->n_layers != nets[1].v->n_layers) {
    UL_TRY(mlp_backward_n(nets, 1, backend, M, s, nullptr, nullptr, nullptr, dd));
    return mlp_backward_n(nets + 1, 1, backend, M, s, nullptr, nullptr, nullptr, dd);
  }
  const Lanes L{s, n == 2 ? side : nullptr, fork, join};
  const int dt = backend_dtype(backend);
  const int eb = dt == kBf16 ? 2 : 4;
  const bool tc = backend >= 1;
  // Deferred dW (bf16 tensor-core back end, LayerNorm included): the dX chain runs
  // first and keeps every layer's dZ; all dW GEMMs of the pass (of both
  // networks when the caller shares its collector) then run as one batched
  // launch with few K splits, and every partial reduction as one pass.
  bool defer = deferred_dw_enabled() && tc && dt == kBf16;
  for (int k = 0; k < n; ++k)
    defer = defer && nets[k].want_dw && nets[k].wp && (!nets[k].v->ln || ln_defer_enabled());
  DeferredDw local_dd;
  DeferredDw* D = defer ? (dd ? dd : &local_dd) : nullptr;
  struct St {
    float* dh_base;  // n_bufs hidden-gradient buffers, dh_stride floats apart
    int64_t dh_stride;
    int nbuf;
    float* ws;
    const float* dh;  // fp32 until the first hidden layer, then dt
    int64_t lddh;
    bool dh_f32;
    int ping;
    int db_done;  // layer whose db the layer above already produced (skinny column sums)
    float* sk_part;
    float* cs_part;
    float* ln_part;
    float* dxw;
    float* next() {
      float* b = dh_base + (int64_t)ping * dh_stride;
      ping = (ping + 1) % nbuf;
      return b;
    }
  } st[2];
  ReduceJob pend[16];  // deferred reductions (skinny heads, column sums, LayerNorm) for the next reduce launch
  int npend = 0;
  const int nl = nets[0].v->n_layers;
  UL_TRY(L.open());
  for (int k = 0; k < n; ++k) {
    const MlpNet& N = nets[k];
    const NetView& v = *N.v;
    UL_CHECK_ARG(dt == kF32 || N.wp, "bf16 MLP needs staged weights");
    UL_CHECK_ARG(dt == kF32 || N.dx == nullptr || N.dx_ncols <= kSkinnyDxMax,
                 "bf16 MLP backward: input gradients (dx) wider than %d columns need the fp32 "
                 "/ tf32 back end", kSkinnyDxMax);
    const int64_t H = max_hidden_ld(v);
    St& S = st[k];
    S.dh_base = N.work;
    S.dh_stride = M * H;
    S.nbuf = defer ? n_dh_bufs(v) : 2;
    S.ws = N.work + n_dh_bufs(v) * M * H;
    S.sk_part = S.ws + dw_ws_floats(v, M);
    S.cs_part = S.sk_part + sk_ws_floats(v, M);
    S.ln_part = S.cs_part + kCsRegion * v.n_layers;
    S.dxw = S.ln_part + rup(ln_layer_off(v, M, v.n_layers - 1), 64);
    S.dh = N.dout;
    S.lddh = N.ld_dout;
    S.dh_f32 = true;
    S.ping = 0;
    S.db_done = -1;
    if (N.head_external) {
      // dZ of the layer below the output layer, in gradient buffer 0
      UL_CHECK_ARG(nl >= 2 && N.dout == N.work, "external head: dZ must sit in work buffer 0");
      S.dh_f32 = dt == kF32;
      S.ping = 1;
      if (N.head_db_below) S.db_done = nl - 2;
    }
    if (N.want_dw && N.zero_logstd && N.grads)
      UL_CUDA(cudaMemsetAsync(N.grads + v.logstd_off, 0, sizeof(float) * v.dims[nl], L.of(k)));
  }
  for (int i = nl - 1; i >= 0; --i) {
    // ---- fused last-layer backward (skinny heads): dW, db, dh_prev and, when
    // the layer below cannot get its db from the ones column, colsum(dh_prev)
    bool skinny_done[2] = {false, false};
    for (int k = 0; k < n; ++k) {
      const MlpNet& N = nets[k];
      const NetView& v = *N.v;
      const int64_t out = v.dims[i + 1], in = v.dims[i];
      const float* inp = i == 0 ? N.x : act_ptr(v, N.acts, M, i - 1, dt);
      const int64_t ldin = i == 0 ? N.ldx : act_ld(v.dims[i], dt);
      if (i == nl - 1 && N.head_external) {  // done by the fused output stage
        skinny_done[k] = true;
        continue;
      }
      if (!(i == nl - 1 && skinny_ok((int)out, (int)in) && i > 0 && al16(inp, ldin, eb)))
        continue;
      St& S = st[k];
      float* nxt = S.next();
      const int64_t in_below = v.dims[i - 1];
      const bool below_ones = i - 1 == 0 ? N.x_has_ones && N.ldx >= in_below + 1 : true;
      // (a LayerNorm layer's db is colsum of its da, which ln_backward makes)
      const bool need_cs =
          N.want_dw && tc && N.wp && !v.ln && !ones_free_of(in_below, below_ones);
      // its partial reduction waits for the next layer's reduce launch
      ReduceJob* dj = (N.want_dw || need_cs) ? &pend[npend] : nullptr;
      UL_TRY(skinny_bwd(inp, ldin, M, (int)in, (int)out, N.params + v.w_off[i], S.dh, S.lddh,
                        nxt, act_ld((int)in, dt), true, N.want_dw ? N.grads + v.w_off[i] : nullptr,
                        N.want_dw ? N.grads + v.b_off[i] : nullptr,
                        need_cs ? N.grads + v.b_off[i - 1] : nullptr, S.sk_part, dt, dj, L.of(k)));
      if (dj) ++npend;
      if (need_cs) S.db_done = i - 1;
      S.dh = nxt;
      S.lddh = act_ld((int)in, dt);
      S.dh_f32 = dt == kF32;
      skinny_done[k] = true;
    }
    if (skinny_done[0] || skinny_done[1]) {
      bool any_rest = false;
      for (int k = 0; k < n; ++k) any_rest |= !skinny_done[k];
      if (!any_rest) continue;
    }
    // ---- upstream gradient of a wide output layer on the bf16 path -> bf16 rows
    for (int k = 0; k < n; ++k) {
      St& S = st[k];
      if (skinny_done[k] || !(S.dh_f32 && dt == kBf16)) continue;
      const int64_t out = nets[k].v->dims[i + 1];
      float* cv = S.next();
      const int64_t ldcv = act_ld((int)out, dt);
      int64_t blocks = ceil_div(M * out, 256);
      blocks = blocks > 8 * kNumSMs ? 8 * kNumSMs : blocks;
      f32_to_bf16_kernel<<<(unsigned)blocks, 256, 0, L.of(k)>>>(
          S.dh, S.lddh, M, out, reinterpret_cast<__nv_bfloat16*>(cv), ldcv);
      UL_TRY(check_launch("f32_to_bf16_kernel"));
      S.dh = cv;
      S.lddh = ldcv;
      S.dh_f32 = false;
    }
    // ---- LayerNorm of hidden layer i: dn (grad at the LN output, from the
    // ELU-gradient epilogue above) -> da in place, + dg / dbeta / db partials
    for (int k = 0; k < n; ++k) {
      const MlpNet& N = nets[k];
      const NetView& v = *N.v;
      if (!v.ln || i >= nl - 1 || skinny_done[k]) continue;
      St& S = st[k];
      const bool has_ones = i == 0 ? (N.x_has_ones && N.ldx >= v.dims[i] + 1) : true;
      const bool db_here = N.want_dw && tc && N.wp && !ones_free_of(v.dims[i], has_ones);
      float* la;
      float* lst;
      int64_t lla;
      ln_bufs(v, N.acts, M, i, &la, &lla, &lst);
      ReduceJob job;
      const bool abf = ln_a_bf16(dt);
      UL_TRY(ln_backward(const_cast<float*>(S.dh), S.lddh, la,
                         abf ? rup(v.dims[i + 1], 8) : lla, lst, N.params + v.g_off[i], M,
                         v.dims[i + 1], S.ln_part + ln_layer_off(v, M, i), dt,
                         N.want_dw ? N.grads + v.g_off[i] : nullptr,
                         N.want_dw ? N.grads + v.beta_off[i] : nullptr,
                         db_here ? N.grads + v.b_off[i] : nullptr, &job, L.of(k), abf));
      if (N.want_dw) pend[npend++] = job;
      if (db_here) S.db_done = i;
    }
    UL_TRY(L.close());
    // ---- dW (+db via the ones column) for both networks: one grouped launch
    // (deferred: collected for the batched launch at the end)
    GemmDesc gw[2] = {};
    bool has_w[2] = {false, false}, tc_w[2] = {false, false}, free_w[2] = {false, false};
    for (int k = 0; k < n; ++k) {
      const MlpNet& N = nets[k];
      const NetView& v = *N.v;
      if (skinny_done[k] || !N.want_dw) continue;
      const int64_t out = v.dims[i + 1], in = v.dims[i];
      const float* inp = i == 0 ? N.x : act_ptr(v, N.acts, M, i - 1, dt);
      const int64_t ldin = i == 0 ? N.ldx : act_ld(v.dims[i], dt);
      const bool has_ones = i == 0 ? (N.x_has_ones && N.ldx >= in + 1) : true;
      GemmDesc& G = gw[k];
      G.M = out; G.K = M;
      G.A = st[k].dh; G.lda = st[k].lddh; G.B = inp; G.ldb = ldin;
      G.a_kmajor = false; G.b_kmajor = false; G.epi = kEpiStore;
      G.C = defer ? st[k].ws + dw_layer_off(v, M, i) : st[k].ws;
      G.dtype = dt;
      G.x3 = backend == kBackendTf32x3;
      free_w[k] = ones_free_of(in, has_ones);
      G.N = free_w[k] ? in + 1 : in;
      G.splits = dw_splits(out, in, M, true);
      G.ldc = rup(G.N, 4);  // 16 B fp32 partial rows (TMA store)
      tc_w[k] = tc && N.wp && (out >= 64 || dt == kBf16) && tc_eligible(G);
      if (tc_w[k]) G.splits = tc_num_splits(M, G.splits, dt);
      has_w[k] = true;
    }
    UL_CHECK_ARG(!defer || ((!has_w[0] || tc_w[0]) && (!has_w[1] || tc_w[1])),
                 "deferred dW: GEMM not tensor-core eligible");
    ReduceJob wj[2];
    for (int k = 0; k < n; ++k) {
      if (!tc_w[k]) continue;
      const NetView& v = *nets[k].v;
      const int64_t out = v.dims[i + 1], in = v.dims[i];
      ReduceJob& J = wj[k];
      J = ReduceJob{};
      J.src = gw[k].C;
      J.nz = gw[k].splits;
      J.kind = 0;
      J.len = out * gw[k].ldc;
      J.ldp = gw[k].ldc;
      J.in = in;
      J.gw = nets[k].grads + v.w_off[i];
      J.gb = free_w[k] ? nets[k].grads + v.b_off[i] : nullptr;
    }
    if (defer) {
      for (int k = 0; k < n; ++k) {
        if (!tc_w[k]) continue;
        const NetView& v = *nets[k].v;
        D->max_splits[D->ndw] = gw[k].splits;
        D->add(gw[k], wj[k]);
        (void)v;
      }
    } else {
      if (tc_w[0] && tc_w[1]) UL_TRY(gemm_tc_group(gw[0], gw[1], s));
      else
        for (int k = 0; k < n; ++k)
          if (tc_w[k]) UL_TRY(gemm_tc(gw[k], -1, s));
      if (tc_w[0] || tc_w[1]) {
        ReduceJob jobs[2 + 16];
        int nj = 0;
        for (int k = 0; k < n; ++k)
          if (tc_w[k]) jobs[nj++] = wj[k];
        for (int q = 0; q < npend; ++q) jobs[nj++] = pend[q];
        npend = 0;
        UL_TRY(launch_reduce(jobs, nj, s));
      }
    }
    UL_TRY(L.open());
    for (int k = 0; k < n; ++k) {
      if (!has_w[k]) continue;
      const MlpNet& N = nets[k];
      const NetView& v = *N.v;
      const int64_t out = v.dims[i + 1], in = v.dims[i];
      St& S = st[k];
      cudaStream_t sk = L.of(k);
      if (tc_w[k]) {
        if (!free_w[k] && S.db_done != i) {
          // 128-row chunks (8 warps x 4 rows in flight x 4), at most 256 of them
          const int64_t chunks = ceil_div(M, 128) < 256 ? ceil_div(M, 128) : 256;
          const int64_t rows_per = ceil_div(M, chunks);
          float* part = gw[k].C + (int64_t)gw[k].splits * out * gw[k].ldc;
          const dim3 grid((unsigned)ceil_div(out, 256), (unsigned)chunks);
          if (dt == kBf16)
            UL_TRY(launch_pdl("colsum_kernel", colsum_kernel<__nv_bfloat16>, grid, dim3(256), 0,
                              sk, reinterpret_cast<const __nv_bfloat16*>(S.dh), S.lddh, M,
                              (int64_t)out, rows_per, part));
          else
            UL_TRY(launch_pdl("colsum_kernel", colsum_kernel<float>, grid, dim3(256), 0, sk,
                              (const float*)S.dh, S.lddh, M, (int64_t)out, rows_per, part));
          UL_TRY(reduce_splits(part, (int)chunks, out, N.grads + v.b_off[i], out, out, sk));
        }
      } else {
        UL_CHECK_ARG(dt == kF32, "bf16 MLP: dW GEMM not tensor-core eligible");
        GemmDesc G = gw[k];
        const int sp = gemm_num_splits(M, dw_splits(out, in, M, false));
        G.N = in;
        G.splits = sp;
        G.ldc = in;
        G.rowsum = S.ws + (int64_t)sp * out * in;
        UL_TRY(gemm_f32(G, sk));
        UL_TRY(reduce_splits(S.ws, sp, out * in, N.grads + v.w_off[i], in, in, sk));
        UL_TRY(reduce_splits(G.rowsum, sp, out, N.grads + v.b_off[i], out, out, sk));
      }
    }
    if (i == 0) {
      for (int k = 0; k < n; ++k) {
        const MlpNet& N = nets[k];
        if (N.dx == nullptr) continue;
        const NetView& v = *N.v;
        const int dxdt = st[k].dh_f32 ? kF32 : dt;
        const int dxeb = dxdt == kBf16 ? 2 : 4;
        if (N.dx_ncols <= kSkinnyDxMax && skinny_ok(N.dx_ncols, v.dims[1]) &&
            al16(st[k].dh, st[k].lddh, dxeb)) {
          // few input columns (SAC's dQ/da): dX = dh W[:, cols] as a skinny
          // product over the once-transposed column slice, one read of dh
          const int64_t tot = (int64_t)N.dx_ncols * v.dims[1];
          slice_t_kernel<<<(unsigned)ceil_div(tot, 256), 256, 0, L.of(k)>>>(
              N.params + v.w_off[0], v.dims[0], N.dx_col0, N.dx_ncols, v.dims[1], st[k].dxw);
          UL_TRY(check_launch("slice_t_kernel"));
          UL_TRY(skinny_fwd(st[k].dh, st[k].lddh, M, v.dims[1], N.dx_ncols, st[k].dxw, nullptr,
                            N.dx, N.lddx, dxdt, L.of(k)));
          continue;
        }
        UL_CHECK_ARG(dxdt == kF32, "bf16 MLP backward: dx GEMM needs fp32 rows");
        GemmDesc G{};
        G.M = M; G.N = N.dx_ncols; G.K = v.dims[1];
        G.A = st[k].dh; G.lda = st[k].lddh; G.B = N.params + v.w_off[0] + N.dx_col0;
        G.ldb = v.dims[0];
        G.C = N.dx; G.ldc = N.lddx;
        G.a_kmajor = true; G.b_kmajor = false; G.epi = kEpiStore; G.splits = 1;
        UL_TRY(gemm_f32(G, L.of(k)));
      }
      UL_TRY(L.close());
      break;
    }
    UL_TRY(L.close());
    if (npend && !defer) {  // no dW reduction at this layer to ride on
      UL_TRY(launch_reduce(pend, npend, s));
      npend = 0;
    }
    // ---- dh_prev = (dh W) * elu'(h_{i-1}) for both networks: one grouped launch
    GemmDesc gx[2] = {};
    bool has_x[2] = {false, false}, tc_x[2] = {false, false};
    const int no_ones[2] = {-1, -1};
    int cs_nz[2] = {0, 0};
    bool cs_on[2] = {false, false};
    for (int k = 0; k < n; ++k) {
      const MlpNet& N = nets[k];
      const NetView& v = *N.v;
      if (skinny_done[k]) continue;
      const int64_t out = v.dims[i + 1], in = v.dims[i];
      St& S = st[k];
      float* nxt = S.next();
      GemmDesc& G = gx[k];
      G.M = M; G.N = in; G.K = out;
      G.A = S.dh; G.lda = S.lddh;
      G.C = nxt; G.ldc = act_ld((int)in, dt);
      G.aux = act_ptr(v, N.acts, M, i - 1, dt); G.ldaux = act_ld((int)in, dt);
      G.a_kmajor = true; G.b_kmajor = false; G.epi = kEpiEluGrad; G.splits = 1;
      G.dtype = dt;
      G.x3 = backend == kBackendTf32x3;
      tc_x[k] = tc && N.wp && (out >= 32 || dt == kBf16);
      if (tc_x[k]) {
        G.B = staged_w(v, N.wp, i, dt, &G.ldb);
      } else {
        G.B = N.params + v.w_off[i];
        G.ldb = in;
      }
      // the layer below needs colsum(dh_prev) for its db: let this GEMM's
      // epilogue produce per-CTA partials (reduced with the next reduction)
      const int64_t in_below = v.dims[i - 1];
      const bool below_ones = i - 1 == 0 ? N.x_has_ones && N.ldx >= in_below + 1 : true;
      if (N.want_dw && tc_x[k] && in <= kCsumMaxN && S.db_done != i - 1 && !v.ln &&
          !ones_free_of(in_below, below_ones)) {
        // (deferred: every layer's partials live until the final reduction)
        G.csum_part = defer ? S.cs_part + kCsRegion * i : S.sk_part;
        G.csum_nz = &cs_nz[k];
        cs_on[k] = true;
      }
      has_x[k] = true;
      S.dh = nxt;
      S.lddh = act_ld((int)in, dt);
    }
    if (!(ablate_mask() & 16)) UL_TRY(run_gemms(gx, has_x, tc_x, no_ones, s));
    for (int k = 0; k < n; ++k) {
      if (!cs_on[k]) continue;
      if (cs_nz[k] == 0) continue;  // GEMM fell back to SIMT: colsum kernel later
      const NetView& v = *nets[k].v;
      const int64_t in = v.dims[i];
      ReduceJob& J = pend[npend++];
      J = ReduceJob{};
      J.src = gx[k].csum_part;
      J.nz = cs_nz[k];
      J.kind = 1;
      J.len = ceil_div(in, 4) * 4;
      J.n0 = in;
      J.o0 = nets[k].grads + v.b_off[i - 1];
      st[k].db_done = i - 1;
    }
    UL_TRY(L.open());
  }
  if (defer) {
    for (int q = 0; q < npend; ++q) D->jobs[D->nj++] = pend[q];
    npend = 0;
    if (D == &local_dd) UL_TRY(run_deferred_dw(local_dd, s));
  }
  if (npend) UL_TRY(launch_reduce(pend, npend, s));
  return UL_OK;
}


int mlp_forward(const NetView& v, const float* params, const float* wp, int backend,
                const float* x, int64_t ldx, int64_t M, float* acts, float* out, int64_t ld_out,
                cudaStream_t s) {
  MlpNet N{};
  N.v = &v; N.params = params; N.wp = backend >= 1 ? wp : nullptr;
  N.x = x; N.ldx = ldx; N.acts = acts; N.out = out; N.ld_out = ld_out;
  return mlp_forward_n(&N, 1, backend, M, s, nullptr, nullptr, nullptr);
}

int mlp_backward(const NetView& v, const float* params, const float* wp, int backend,
                 const float* x, int64_t ldx, bool x_has_ones, int64_t M, const float* acts,
                 const float* dout, int64_t ld_dout, float* grads, float* dx, int64_t lddx,
                 int dx_col0, int dx_ncols, bool want_dw, bool zero_logstd, float* work,
                 cudaStream_t s) {
  MlpNet N{};
  N.v = &v; N.params = params; N.wp = backend >= 1 ? wp : nullptr;
  N.x = x; N.ldx = ldx; N.x_has_ones = x_has_ones;
  N.acts = const_cast<float*>(acts);
  N.dout = dout; N.ld_dout = ld_dout; N.grads = grads;
  N.dx = dx; N.lddx = lddx; N.dx_col0 = dx_col0; N.dx_ncols = dx_ncols;
  N.want_dw = want_dw; N.zero_logstd = zero_logstd; N.work = work;
  return mlp_backward_n(&N, 1, backend, M, s, nullptr, nullptr, nullptr);
}

}  // namespace ul

// -------------------------------------------------------------- C ABI
extern "C" int64_t ul_net_param_count(const ul_net_desc* net) {
  ul::NetView v;
  if (ul::make_view(net, &v) != UL_OK) return -1;
  return v.total;
}

extern "C" int64_t ul_mlp_act_floats(const ul_net_desc* net, int64_t M) {
  ul::NetView v;
  if (ul::make_view(net, &v) != UL_OK) return -1;
  return ul::act_floats(v, M);
}

extern "C" int64_t ul_mlp_bwd_work_floats(const ul_net_desc* net, int64_t M) {
  ul::NetView v;
  if (ul::make_view(net, &v) != UL_OK) return -1;
  return ul::bwd_work_floats(v, M);
}

extern "C" int64_t ul_mlp_wstage_floats(const ul_net_desc* net) {
  ul::NetView v;
  if (ul::make_view(net, &v) != UL_OK) return -1;
  return v.wp_total;
}

extern "C" int ul_stage_weights(const ul_net_desc* net, const float* params, float* wstage,
                                void* stream) {
  ul::NetView v;
  UL_TRY(ul::make_view(net, &v));
  return ul::stage_weights(v, params, wstage, ul::as_stream(stream));
}

extern "C" int64_t ul_mlp_act_ld(int d, int backend) {
  return ul::act_ld(d, ul::backend_dtype(backend));
}

extern "C" int ul_stage_weights_ex(const ul_net_desc* net, const float* params, void* wstage,
                                   int backend, void* stream) {
  ul::NetView v;
  UL_TRY(ul::make_view(net, &v));
  return ul::stage_weights_dt(v, params, wstage, ul::backend_dtype(backend),
                              ul::as_stream(stream));
}

extern "C" int ul_mlp_forward(const ul_net_desc* net, const float* params, const float* wstage,
                              int backend, const float* x, int64_t ldx, int64_t M, float* acts,
                              float* out, int64_t ld_out, void* stream) {
  ul::NetView v;
  UL_TRY(ul::make_view(net, &v));
  UL_CHECK_ARG(M >= 0, "forward: negative batch");
  UL_CHECK_ARG(ldx >= v.dims[0], "forward: ldx %lld < input_dim %d", (long long)ldx, v.dims[0]);
  UL_CHECK_ARG(backend >= 0 && backend <= 3,
               "forward: backend must be 0 (fp32), 1 (tf32), 2 (bf16) or 3 (3xTF32)");
  return ul::mlp_forward(v, params, wstage, backend, x, ldx, M, acts, out, ld_out,
                         ul::as_stream(stream));
}

// Two independent networks over the same M rows in lockstep (APPO's target
// recompute: actor on obs, critic on critic_obs): one grouped tensor-core
// launch per layer; each network's result is the same as ul_mlp_forward's.
extern "C" int ul_mlp_forward2(const ul_net_desc* net_a, const float* params_a, const float* wstage_a,
                               const float* x_a, int64_t ldx_a, float* acts_a, float* out_a,
                               int64_t ld_out_a, const ul_net_desc* net_b, const float* params_b,
                               const float* wstage_b, const float* x_b, int64_t ldx_b,
                               float* acts_b, float* out_b, int64_t ld_out_b, int backend,
                               int64_t M, void* stream) {
  ul::NetView va, vb;
  UL_TRY(ul::make_view(net_a, &va));
  UL_TRY(ul::make_view(net_b, &vb));
  UL_CHECK_ARG(M >= 0, "forward2: negative batch");
  UL_CHECK_ARG(ldx_a >= va.dims[0] && ldx_b >= vb.dims[0], "forward2: ldx below input_dim");
  UL_CHECK_ARG(backend >= 0 && backend <= 3,
               "forward2: backend must be 0 (fp32), 1 (tf32), 2 (bf16) or 3 (3xTF32)");
  ul::MlpNet n[2] = {};
  const ul::NetView* v[2] = {&va, &vb};
  const float* pr[2] = {params_a, params_b};
  const float* ws[2] = {wstage_a, wstage_b};
  const float* x[2] = {x_a, x_b};
  const int64_t ldx[2] = {ldx_a, ldx_b};
  float* acts[2] = {acts_a, acts_b};
  float* out[2] = {out_a, out_b};
  const int64_t ldo[2] = {ld_out_a, ld_out_b};
  for (int k = 0; k < 2; ++k) {
    n[k].v = v[k];
    n[k].params = pr[k];
    n[k].wp = backend >= 1 ? ws[k] : nullptr;
    n[k].x = x[k];
    n[k].ldx = ldx[k];
    n[k].acts = acts[k];
    n[k].out = out[k];
    n[k].ld_out = ldo[k];
  }
  return ul::mlp_forward_n(n, 2, backend, M, ul::as_stream(stream), nullptr, nullptr, nullptr);
}

extern "C" int ul_mlp_backward(const ul_net_desc* net, const float* params, const float* wstage,
                               int backend, const float* x, int64_t ldx, int x_has_ones, int64_t M,
                               const float* acts, const float* dout, int64_t ld_dout,
                               float* grads, float* dx, int64_t lddx, float* work, void* stream) {
  ul::NetView v;
  UL_TRY(ul::make_view(net, &v));
  UL_CHECK_ARG(M >= 0, "backward: negative batch");
  UL_CHECK_ARG(backend >= 0 && backend <= 3,
               "backward: backend must be 0 (fp32), 1 (tf32), 2 (bf16) or 3 (3xTF32)");
  return ul::mlp_backward(v, params, wstage, backend, x, ldx, x_has_ones != 0, M, acts, dout,
                          ld_dout, grads, dx, lddx, 0, v.dims[0], true, true, work,
                          ul::as_stream(stream));
}
