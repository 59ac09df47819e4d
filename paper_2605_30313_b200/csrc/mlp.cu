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
#include "internal.cuh"

namespace ul {

int gemm_tc(const GemmDesc& d, int ones_col, cudaStream_t s);
bool tc_eligible(const GemmDesc& d);
int tc_num_splits(int64_t K, int splits);
bool skinny_ok(int N);
int64_t skinny_part_floats(int64_t M, int K, int N);
int skinny_fwd(const float* h, int64_t ldh, int64_t M, int K, int N, const float* W,
               const float* b, float* out, int64_t ldo, cudaStream_t s);
int skinny_bwd(const float* h, int64_t ldh, int64_t M, int K, int N, const float* W,
               const float* dout, int64_t ldd, float* dh, int64_t lddh, bool elu_grad,
               float* gw, float* gb, float* part, cudaStream_t s);

namespace {

int64_t rup(int64_t x, int64_t m) { return ceil_div(x, m) * m; }

__global__ void __launch_bounds__(256) reduce_dw_kernel(const float* __restrict__ ws, int splits,
                                                        int64_t out, int64_t in, int64_t ldp,
                                                        float* __restrict__ gw,
                                                        float* __restrict__ gb) {
  // ws: splits x [out, ldp]; column `in` is the bias gradient, columns > in
  // are TMA-row padding.  32 outputs per CTA, splits spread over 8 warps,
  // fixed-order combine (deterministic).
  __shared__ float sm[8][33];
  const int64_t len = out * ldp;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t j = (int64_t)blockIdx.x * 32 + lane;
  float s = 0.f;
  if (j < len) {
    // four independent accumulators keep 4 loads in flight per warp
    float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
    int z = w;
    for (; z + 24 < splits; z += 32) {
      s0 += ws[(int64_t)z * len + j];
      s1 += ws[(int64_t)(z + 8) * len + j];
      s2 += ws[(int64_t)(z + 16) * len + j];
      s3 += ws[(int64_t)(z + 24) * len + j];
    }
    for (; z < splits; z += 8) s0 += ws[(int64_t)z * len + j];
    s = (s0 + s1) + (s2 + s3);
  }
  sm[w][lane] = s;
  __syncthreads();
  if (w == 0 && j < len) {
    float t = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) t += sm[k][lane];
    const int64_t r = j / ldp, c = j - r * ldp;
    if (c < in) gw[r * in + c] = t;
    else if (c == in && gb) gb[r] = t;
  }
}

// db partials: column sums of dh [M, N] over row chunks; lanes = columns
// (coalesced 128 B rows), 8 warps stride the rows; part[chunk][N]
__global__ void __launch_bounds__(256) colsum_kernel(const float* __restrict__ x, int64_t ld,
                                                     int64_t M, int64_t N, int64_t rows_per,
                                                     float* __restrict__ part) {
  __shared__ float sm[8][33];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t c = (int64_t)blockIdx.x * 32 + lane;
  const int64_t r0 = (int64_t)blockIdx.y * rows_per;
  const int64_t r1 = r0 + rows_per < M ? r0 + rows_per : M;
  float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
  if (c < N) {
    int64_t r = r0 + w;
    for (; r + 24 < r1; r += 32) {
      s0 += x[r * ld + c];
      s1 += x[(r + 8) * ld + c];
      s2 += x[(r + 16) * ld + c];
      s3 += x[(r + 24) * ld + c];
    }
    for (; r < r1; r += 8) s0 += x[r * ld + c];
  }
  sm[w][lane] = (s0 + s1) + (s2 + s3);
  __syncthreads();
  if (w == 0 && c < N) {
    float t = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) t += sm[k][lane];
    part[(int64_t)blockIdx.y * N + c] = t;
  }
}

struct StageTable {
  int n;
  int64_t src_off[UL_MAX_LAYERS], dst_off[UL_MAX_LAYERS];
  int rows[UL_MAX_LAYERS], cols[UL_MAX_LAYERS], ld[UL_MAX_LAYERS];
  int64_t total;  // padded elements
};

__global__ void stage_weights_kernel(const float* __restrict__ params, StageTable t,
                                     float* __restrict__ wp) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < t.total; j += stride) {
    int l = 0;
    while (l + 1 < t.n && j >= t.dst_off[l + 1]) ++l;
    const int64_t k = j - t.dst_off[l];
    const int64_t r = k / t.ld[l], c = k - r * t.ld[l];
    wp[j] = c < t.cols[l] ? params[t.src_off[l] + r * t.cols[l] + c] : 0.f;
  }
}

}  // namespace

int64_t act_ld(int d) { return rup((int64_t)d + 1, 4); }

int make_view(const ul_net_desc* d, NetView* v) {
  UL_CHECK_ARG(d != nullptr, "net: null descriptor");
  UL_CHECK_ARG(d->n_layers >= 1 && d->n_layers <= UL_MAX_LAYERS,
               "net: n_layers %d outside [1,%d]", d->n_layers, UL_MAX_LAYERS);
  v->n_layers = d->n_layers;
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
    v->wp_off[i] = woff;
    woff += (int64_t)v->dims[i + 1] * rup(v->dims[i], 4);
  }
  v->logstd_off = off;
  v->total = off + v->dims[d->n_layers];
  v->wp_total = woff;
  return UL_OK;
}

int64_t act_floats(const NetView& v, int64_t M) {
  int64_t s = 0;
  for (int i = 1; i < v.n_layers; ++i) s += act_ld(v.dims[i]) * M;
  return s;
}

static int64_t max_hidden_ld(const NetView& v) {
  int64_t h = 4;
  for (int i = 1; i <= v.n_layers; ++i) h = act_ld(v.dims[i]) > h ? act_ld(v.dims[i]) : h;
  return h;
}

// dW split count: enough CTAs for ~2 waves, >= 512 batch rows per split
static int dw_splits(int64_t out, int64_t in, int64_t M, bool tc) {
  const int64_t tiles = tc ? ceil_div(out, 128) * ceil_div(in + 1, 256)
                           : ceil_div(out, 128) * ceil_div(in, 128);
  int64_t sp = ceil_div(tc ? kNumSMs : 2 * kNumSMs, tiles);
  const int64_t cap = ceil_div(M, 512);
  sp = sp < cap ? sp : cap;
  sp = sp < 1 ? 1 : sp;
  return (int)(sp > 64 ? 64 : sp);
}

int64_t bwd_work_floats(const NetView& v, int64_t M) {
  int64_t ws = 0;
  for (int i = 0; i < v.n_layers; ++i) {
    const int64_t out = v.dims[i + 1], in = v.dims[i];
    const int sp = dw_splits(out, in, M, false) > dw_splits(out, in, M, true)
                       ? dw_splits(out, in, M, false) : dw_splits(out, in, M, true);
    int64_t need = (int64_t)sp * (out * rup(in + 1, 4) + out) + 256 * out;
    if (skinny_ok((int)out)) {
      const int64_t sk = skinny_part_floats(M, (int)in, (int)out);
      need = sk > need ? sk : need;
    }
    ws = need > ws ? need : ws;
  }
  return 2 * M * max_hidden_ld(v) + ws;
}

const float* act_ptr(const NetView& v, const float* acts, int64_t M, int i) {
  int64_t off = 0;
  for (int j = 1; j <= i; ++j) off += act_ld(v.dims[j]) * M;
  return acts + off;
}

int stage_weights(const NetView& v, const float* params, float* wp, cudaStream_t s) {
  StageTable t{};
  t.n = v.n_layers;
  for (int i = 0; i < v.n_layers; ++i) {
    t.src_off[i] = v.w_off[i];
    t.dst_off[i] = v.wp_off[i];
    t.rows[i] = v.dims[i + 1];
    t.cols[i] = v.dims[i];
    t.ld[i] = (int)rup(v.dims[i], 4);
  }
  t.total = v.wp_total;
  int64_t blocks = ceil_div(t.total, 256);
  blocks = blocks > 4 * kNumSMs ? 4 * kNumSMs : blocks;
  stage_weights_kernel<<<(unsigned)blocks, 256, 0, s>>>(params, t, wp);
  return check_launch("stage_weights_kernel");
}

static int run_gemm(GemmDesc g, bool use_tc, int ones_col, cudaStream_t s) {
  g.ones_col = ones_col;
  if (use_tc && tc_eligible(g)) return gemm_tc(g, ones_col, s);
  return gemm_f32(g, s);
}

int mlp_forward(const NetView& v, const float* params, const float* wp, int backend,
                const float* x, int64_t ldx, int64_t M, float* acts, float* out, int64_t ld_out,
                cudaStream_t s) {
  const float* h = x;
  int64_t ldh = ldx;
  const bool tc = backend == 1 && wp != nullptr;
  for (int i = 0; i < v.n_layers; ++i) {
    const bool last = i == v.n_layers - 1;
    float* dst = last ? out : const_cast<float*>(act_ptr(v, acts, M, i));
    const int64_t lddst = last ? ld_out : act_ld(v.dims[i + 1]);
    GemmDesc g{};
    g.M = M; g.N = v.dims[i + 1]; g.K = v.dims[i];
    g.A = h; g.lda = ldh;
    g.bias = params + v.b_off[i];
    g.a_kmajor = true; g.b_kmajor = true;
    g.epi = last ? kEpiBias : kEpiBiasElu;
    g.splits = 1;
    g.C = dst; g.ldc = lddst;
    if (last && skinny_ok(v.dims[i + 1])) {  // 12-/1-wide head layer
      UL_TRY(skinny_fwd(h, ldh, M, v.dims[i], v.dims[i + 1], params + v.w_off[i],
                        params + v.b_off[i], dst, lddst, s));
      break;
    }
    const bool tc_here = tc && !last;
    if (tc_here) {
      g.B = wp + v.wp_off[i];
      g.ldb = rup(v.dims[i], 4);
    } else {
      g.B = params + v.w_off[i];
      g.ldb = v.dims[i];
    }
    UL_TRY(run_gemm(g, tc_here, last ? -1 : v.dims[i + 1], s));
    h = dst;
    ldh = lddst;
  }
  return UL_OK;
}

int mlp_backward(const NetView& v, const float* params, const float* wp, int backend,
                 const float* x, int64_t ldx, bool x_has_ones, int64_t M, const float* acts,
                 const float* dout, int64_t ld_dout, float* grads, float* dx, int64_t lddx,
                 int dx_col0, int dx_ncols, bool want_dw, bool zero_logstd, float* work,
                 cudaStream_t s) {
  const int64_t H = max_hidden_ld(v);
  float* dh_buf[2] = {work, work + M * H};
  float* ws = work + 2 * M * H;
  const float* dh = dout;
  int64_t lddh = ld_dout;
  int ping = 0;
  const bool tc = backend == 1 && wp != nullptr;
  if (want_dw && zero_logstd && grads)
    UL_CUDA(cudaMemsetAsync(grads + v.logstd_off, 0, sizeof(float) * v.dims[v.n_layers], s));
  for (int i = v.n_layers - 1; i >= 0; --i) {
    const int64_t out = v.dims[i + 1], in = v.dims[i];
    const float* inp = i == 0 ? x : act_ptr(v, acts, M, i - 1);
    const int64_t ldin = i == 0 ? ldx : act_ld(v.dims[i]);
    const bool has_ones = i == 0 ? (x_has_ones && ldx >= in + 1) : true;
    if (i == v.n_layers - 1 && skinny_ok((int)out) && i > 0) {
      // fused last-layer backward: dW, db and dh_prev in one pass over h
      float* nxt = dh_buf[ping];
      ping ^= 1;
      UL_TRY(skinny_bwd(inp, ldin, M, (int)in, (int)out, params + v.w_off[i], dh, lddh, nxt,
                        act_ld((int)in), true, want_dw ? grads + v.w_off[i] : nullptr,
                        want_dw ? grads + v.b_off[i] : nullptr, ws, s));
      dh = nxt;
      lddh = act_ld((int)in);
      continue;
    }
    if (want_dw) {
      GemmDesc g{};
      g.M = out; g.K = M;
      g.A = dh; g.lda = lddh; g.B = inp; g.ldb = ldin;
      g.a_kmajor = false; g.b_kmajor = false; g.epi = kEpiStore;
      g.C = ws;
      // [dW | db] through the ones column when that column rides in a tile the
      // GEMM computes anyway; otherwise dW alone + a column-sum pass for db
      auto bn_of = [](int64_t n) { return n > 128 ? 256 : 128; };
      const bool ones_free = has_ones && bn_of(in + 1) == bn_of(in) &&
                             ceil_div(in + 1, bn_of(in + 1)) == ceil_div(in, bn_of(in));
      GemmDesc gt = g;
      gt.N = ones_free ? in + 1 : in;
      gt.splits = dw_splits(out, in, M, true);
      gt.ldc = rup(gt.N, 4);  // 16 B partial rows (TMA store)
      if (tc && out >= 64 && tc_eligible(gt)) {
        const int sp = tc_num_splits(M, gt.splits);
        gt.splits = sp;
        UL_TRY(gemm_tc(gt, -1, s));
        const int64_t blocks = ceil_div(out * gt.ldc, 32);
        reduce_dw_kernel<<<(unsigned)blocks, 256, 0, s>>>(
            ws, sp, out, in, gt.ldc, grads + v.w_off[i],
            ones_free ? grads + v.b_off[i] : nullptr);
        UL_TRY(check_launch("reduce_dw_kernel"));
        if (!ones_free) {
          // 256-row chunks (8 warps x 32 rows, 4 loads in flight each), <= 256 chunks
          const int64_t chunks = ceil_div(M, 256) < 256 ? ceil_div(M, 256) : 256;
          const int64_t rows_per = ceil_div(M, chunks);
          float* part = ws + (int64_t)sp * out * gt.ldc;
          colsum_kernel<<<dim3((unsigned)ceil_div(out, 32), (unsigned)chunks), 256, 0, s>>>(
              dh, lddh, M, out, rows_per, part);
          UL_TRY(check_launch("colsum_kernel"));
          UL_TRY(reduce_splits(part, (int)chunks, out, grads + v.b_off[i], out, out, s));
        }
      } else {
        const int sp = gemm_num_splits(M, dw_splits(out, in, M, false));
        g.N = in;
        g.splits = sp;
        g.ldc = in;
        g.rowsum = ws + (int64_t)sp * out * in;
        UL_TRY(gemm_f32(g, s));
        UL_TRY(reduce_splits(ws, sp, out * in, grads + v.w_off[i], in, in, s));
        UL_TRY(reduce_splits(g.rowsum, sp, out, grads + v.b_off[i], out, out, s));
      }
    }
    if (i == 0) {
      if (dx == nullptr) break;
      GemmDesc g{};
      g.M = M; g.N = dx_ncols; g.K = out;
      g.A = dh; g.lda = lddh; g.B = params + v.w_off[0] + dx_col0; g.ldb = in;
      g.C = dx; g.ldc = lddx;
      g.a_kmajor = true; g.b_kmajor = false; g.epi = kEpiStore; g.splits = 1;
      UL_TRY(gemm_f32(g, s));
      break;
    }
    // dh_prev = (dh W) * elu'(h_{i-1})
    float* nxt = dh_buf[ping];
    ping ^= 1;
    GemmDesc g{};
    g.M = M; g.N = in; g.K = out;
    g.A = dh; g.lda = lddh;
    g.C = nxt; g.ldc = act_ld((int)in);
    g.aux = act_ptr(v, acts, M, i - 1); g.ldaux = act_ld((int)in);
    g.a_kmajor = true; g.b_kmajor = false; g.epi = kEpiEluGrad; g.splits = 1;
    const bool tc_here = tc && out >= 32;
    if (tc_here) {
      g.B = wp + v.wp_off[i];
      g.ldb = rup(in, 4);
    } else {
      g.B = params + v.w_off[i];
      g.ldb = in;
    }
    UL_TRY(run_gemm(g, tc_here, -1, s));
    dh = nxt;
    lddh = act_ld((int)in);
  }
  return UL_OK;
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

extern "C" int ul_mlp_forward(const ul_net_desc* net, const float* params, const float* wstage,
                              int backend, const float* x, int64_t ldx, int64_t M, float* acts,
                              float* out, int64_t ld_out, void* stream) {
  ul::NetView v;
  UL_TRY(ul::make_view(net, &v));
  UL_CHECK_ARG(M >= 0, "forward: negative batch");
  UL_CHECK_ARG(ldx >= v.dims[0], "forward: ldx %lld < input_dim %d", (long long)ldx, v.dims[0]);
  UL_CHECK_ARG(backend == 0 || backend == 1, "forward: backend must be 0 (fp32) or 1 (tf32)");
  return ul::mlp_forward(v, params, wstage, backend, x, ldx, M, acts, out, ld_out,
                         ul::as_stream(stream));
}

extern "C" int ul_mlp_backward(const ul_net_desc* net, const float* params, const float* wstage,
                               int backend, const float* x, int64_t ldx, int x_has_ones, int64_t M,
                               const float* acts, const float* dout, int64_t ld_dout,
                               float* grads, float* dx, int64_t lddx, float* work, void* stream) {
  ul::NetView v;
  UL_TRY(ul::make_view(net, &v));
  UL_CHECK_ARG(M >= 0, "backward: negative batch");
  UL_CHECK_ARG(backend == 0 || backend == 1, "backward: backend must be 0 (fp32) or 1 (tf32)");
  return ul::mlp_backward(v, params, wstage, backend, x, ldx, x_has_ones != 0, M, acts, dout,
                          ld_dout, grads, dx, lddx, 0, v.dims[0], true, true, work,
                          ul::as_stream(stream));
}
