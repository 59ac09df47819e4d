// Cross-translation-unit declarations inside libunilite_b200 (not part of the ABI).
#pragma once
#include "common.cuh"

namespace ul {

// ---------------------------------------------------------------- optimizer
struct SegTable {
  float* g[UL_MAX_SEG];
  float* p[UL_MAX_SEG];
  float* m[UL_MAX_SEG];
  float* v[UL_MAX_SEG];
  int64_t n[UL_MAX_SEG];
  int nseg;
};
// PPO per-step loss finalisation folded into the optimizer's prepare kernel
// (its last CTA runs it before the divergence latch reads ctl->loss_bad)
struct LossFinalize {
  const float* loss;     // [pol, val, kl] sums (after the optional all-reduce)
  const float* log_std;  // actor log_std (entropy)
  int A;
  double n, vcoef, ecoef;
  int last_in_epoch;
  ul_ppo_stats* st;
};
// Staged weight copies refreshed by the Adam step itself (the tensor-core
// MLP's operand layout): W_l of segment s at dst + dst_off[l], rows of ld
struct StageOut {
  void* dst[UL_MAX_SEG];
  int dtype;  // kF32 / kBf16 (same for every segment)
  int nl[UL_MAX_SEG];
  int64_t w_off[UL_MAX_SEG][UL_MAX_LAYERS];
  int64_t dst_off[UL_MAX_SEG][UL_MAX_LAYERS];
  int rows[UL_MAX_SEG][UL_MAX_LAYERS], cols[UL_MAX_SEG][UL_MAX_LAYERS], ld[UL_MAX_SEG][UL_MAX_LAYERS];
};
int launch_prepare(const SegTable& st, ul_opt_ctl* ctl, cudaStream_t s,
                   const LossFinalize* lf = nullptr);
int launch_apply(const SegTable& st, ul_opt_ctl* ctl, int write_grads, int do_adam,
                 cudaStream_t s, const StageOut* so = nullptr);

// --------------------------------------------------------------------- GEMM
// C[M,N] = sum_k A(m,k) B(k,n), fp32.
//   A(m,k) = A[m*lda + k] if a_kmajor else A[k*lda + m]
//   B(k,n) = B[n*ldb + k] if b_kmajor else B[k*ldb + n]
enum Epilogue : int {
  kEpiStore = 0,     // C = acc
  kEpiBias = 1,      // C = acc + bias[n]
  kEpiBiasElu = 2,   // C = elu(acc + bias[n])
  kEpiEluGrad = 3,   // C = acc * (min(aux[m,n],0)+1)
  kEpiBiasLn = 4,    // C = acc + bias[n] as bf16 rows (a LayerNorm layer's pre-LN activation)
  kEpiLnFull = 5,    // kEpiBiasLn + the whole LayerNorm in the epilogue: row statistics
                     // across a cluster of N-tile CTAs (DSMEM), h = elu(LN(a) g + beta)
};

// operand storage of a GEMM / activation buffer
enum DType : int {
  kF32 = 0,   // fp32 (SIMT fp32 or tcgen05 kind::tf32)
  kBf16 = 1,  // bf16 (tcgen05 kind::f16), fp32 accumulation
};

struct GemmDesc {
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
  bool a_kmajor, b_kmajor;
  int epi;
  // split-K over K: when splits > 1, C must be a workspace of splits*M*N
  // floats (partial tiles, ld = N) and a reduction pass follows.
  int splits;
  // optional: per-row sums of A over K (db of a dW GEMM), written per split
  // into rowsum[z*M + m]
  float* rowsum;
  // >= 0: the epilogue also writes C[m, ones_col] = 1 (activation ones column)
  int ones_col = -1;
  // kBf16: A, B (and aux / C of the ELU epilogues) hold bf16 despite the
  // float* fields; only the tensor-core path accepts it
  int dtype = kF32;
  // tensor-core ELU-gradient epilogue only (N <= kCsumMaxN): also emit
  // per-CTA column sums of the output, csum_part[cta][round_up(N,4)]; the
  // launch stores its CTA count in *csum_nz (the bias gradient of the layer
  // below, reduced later with a ReduceJob)
  float* csum_part = nullptr;
  int* csum_nz = nullptr;
  // fp32 operands through the tf32 tensor cores as 3xTF32 (hi/lo split,
  // hi*hi + hi*lo + lo*hi): the exact-fp32 parity back end on tcgen05
  bool x3 = false;
  // kEpiLnFull only: C receives the pre-LN rows a (bf16), ln_h the layer's
  // output h = elu((a - mean) rstd g + beta) (bf16, ld ldh, 1.0 in column
  // ln_h_ones when >= 0), ln_stats the per-row (mean, rstd) float2
  void* ln_h = nullptr;
  int64_t ldh = 0;
  const float* ln_g = nullptr;
  const float* ln_beta = nullptr;
  float* ln_stats = nullptr;
  int ln_h_ones = -1;
};
constexpr int kCsumMaxN = 512;
constexpr int kLnFullMaxN = 1024;  // widest LayerNorm row the fused epilogue takes (4 N tiles)
// widest input-gradient column slice the skinny dX path takes (SAC dQ/da)
constexpr int kSkinnyDxMax = 32;
int gemm_f32(const GemmDesc& d, cudaStream_t s);
// number of K splits gemm_f32 actually launches for a requested split count
int gemm_num_splits(int64_t K, int splits);
// out[j] (+)= sum_z ws[z*len + j], j < len
int reduce_splits(const float* ws, int splits, int64_t len, float* out, int64_t ld_rows,
                  int64_t row_len, cudaStream_t s);

// Fixed-order reduction of block / split partials: out = sum_z src[z*len + j].
// kind 0 (split-K dW): j -> (r, c) = divmod(j, ldp); c < in -> gw[r*in + c],
//   c == in -> gb[r] (ones-column bias), c > in padding.
// kind 1 (segments): [0,n0) -> o0, [n0,n0+n1) -> o1, [n0+n1,n0+n1+n2) -> o2.
// len must be a multiple of 4; null destinations are skipped.
struct ReduceJob {
  const float* src;
  int nz;
  int kind;
  int64_t len;
  int64_t ldp, in;
  float* gw;
  float* gb;
  int64_t n0, n1, n2;
  float *o0, *o1, *o2;
};
constexpr int kMaxReduceJobs = 32;

// Diagnostics only (tools/step_ablate.py): UL_ABLATE bit mask drops pieces of
// every PPO step to time the rest -- 1 gather, 2 Adam apply, 4 the fused
// output stage, 8 the forward, 16 the dX GEMMs, 32 the batched dW GEMMs,
// 64 the gradient reduction.  Results are meaningless when set.
inline int ablate_mask() {
  static int m = -1;
  if (m < 0) {
    const char* e = getenv("UL_ABLATE");
    m = e ? atoi(e) : 0;
  }
  return m;
}

// Optional fold of the K13 prepare pass into the reduction that produces the
// final gradients (single-process PPO step): every value the reduction
// stores inside [base, base + n0) (segment 0) or [base + n0, base + n0 + n1)
// (segment 1) also enters a per-block (sum g^2, non-finite) partial; the
// last block runs the prepare tail (opt_tail.cuh).  Valid only when the
// reduction writes EVERY element of both segments that can be nonzero (the
// bf16 fused-head PPO step: all dW / db / dlog_std values come out of it).
struct SqFold {
  int on;
  const float* base;
  int64_t n0, n1;
  double* part;      // [blocks][2]
  int* bad;          // [blocks][2]
  int cap;           // blocks the partial arrays hold
  unsigned int* ticket;
  ul_opt_ctl* ctl;
  LossFinalize lf;
};

// dW GEMMs of a backward pass collected for one batched tensor-core launch
// (gemm_tc_batch) + one reduction pass of their split partials and the
// pass's other deferred partial sets (run_deferred_dw, mlp.cu)
struct DeferredDw {
  static constexpr int kMax = 16;
  GemmDesc dw[kMax];
  int max_splits[kMax];  // split count each layer's workspace region holds
  int dw_job[kMax];      // jobs[] index of each dW's reduction
  int ndw = 0;
  ReduceJob jobs[3 * kMax];
  int nj = 0;
  const SqFold* fold = nullptr;  // fold the prepare pass into the reduction
  bool folded = false;           // (out) the reduction ran the prepare tail
  void add(const GemmDesc& g, const ReduceJob& j);
};
int run_deferred_dw(DeferredDw& D, cudaStream_t s);  // = the two below
int run_deferred_dw_gemms(DeferredDw& D, cudaStream_t s);
int run_deferred_dw_reduce(DeferredDw& D, cudaStream_t s);
bool deferred_dw_enabled();  // UL_DEFER_DW (default on)
// independent tensor-core GEMMs, batched into as few launches as compatible
int gemm_tc_batch(const GemmDesc* d, int n, cudaStream_t s);
// stacked bias+ELU layers of up to 2 networks in one launch (gemm_tc.cu)
int gemm_tc_chain(const GemmDesc* d, int nets, int L, cudaStream_t s);

// ------------------------------------------------------------------ MLP
struct NetView {
  int n_layers;
  int dims[UL_MAX_LAYERS + 1];
  int64_t w_off[UL_MAX_LAYERS], b_off[UL_MAX_LAYERS], logstd_off, total;
  int64_t wp_off[UL_MAX_LAYERS], wp_total;  // staged (16 B-row) weight layout
  int64_t wb_off[UL_MAX_LAYERS];            // bf16 staged layout (ld round_up(in, 8))
  int ln;                                   // LayerNorm on hidden layers
  int64_t g_off[UL_MAX_LAYERS], beta_off[UL_MAX_LAYERS];
};
// LayerNorm rows (ln.cu): a [M, D] fp32 (GEMM output) -> h (dtype) = elu(LN(a) g + beta)
// a: pre-LN rows, fp32 or (a_bf16) bf16 (the bf16 GEMM's kEpiBiasLn output)
int ln_forward(const void* a, int64_t lda, int64_t M, int D, const float* g, const float* beta,
               float* stats, void* h, int64_t ldh, int ones_col, int dtype, cudaStream_t s,
               bool a_bf16 = false);
// dn -> da in place; partial sums of dg | dbeta | colsum(da) described by *job
int ln_backward(void* dn, int64_t ldd, const void* a, int64_t lda, const float* stats,
                const float* g, int64_t M, int D, float* part, int dtype, float* gg, float* gbeta,
                float* gb, ReduceJob* job, cudaStream_t s, bool a_bf16 = false);
int64_t ln_part_floats(int64_t M, int D);
// pre-LayerNorm rows a_i [M, round_up(D,4)] fp32 and stats [M][2] of hidden layer i
void ln_bufs(const NetView& v, const float* acts, int64_t M, int i, float** a, int64_t* lda,
             float** stats);
int make_view(const ul_net_desc* d, NetView* v);
// hidden activation row stride (elements): round_up(d + 1, 4) fp32 /
// round_up(d + 1, 8) bf16 -- 16-byte rows plus the ones column
int64_t act_ld(int d, int dtype = kF32);
int64_t act_floats(const NetView& v, int64_t M);
const float* act_ptr(const NetView& v, const float* acts, int64_t M, int i, int dtype = kF32);
int64_t bwd_work_floats(const NetView& v, int64_t M);
int stage_weights(const NetView& v, const float* params, float* wp, cudaStream_t s);
// backend 0: fp32 SIMT; 1: tcgen05 tf32 (wp = staged weights, may be null -> SIMT);
// 2: tcgen05 bf16 -- x, the hidden activations and the backward's hidden
// gradients are bf16 (rows of act_ld(d, kBf16)), params / grads / outputs fp32
inline int backend_dtype(int backend) { return backend == 2 ? kBf16 : kF32; }
// backend 3: tcgen05 kind::tf32 on 3xTF32-split fp32 operands (exact-fp32 parity)
constexpr int kBackendTf32x3 = 3;
// scratch of the 3xTF32 split operands: grown on demand outside graph
// capture; plans reserve their bound at creation
int x3_reserve(size_t floats);
size_t x3_bound(const NetView& v, int64_t M);
int stage_weights_dt(const NetView& v, const float* params, void* wp, int dtype, cudaStream_t s);
// n networks' staged rows in one launch
int stage_weights_multi(int n, const NetView* const* v, const float* const* params,
                        void* const* wp, int dtype, cudaStream_t s);

// ------------------------------------------------------------------ gather
// ul_gather_rows with an optional per-desc fp32 -> bf16 conversion (cvt)
int gather_rows(int ndesc, const void* const* src, void* const* dst, const int64_t* src_stride,
                const int64_t* dst_stride, const int64_t* row_bytes, const int64_t* ones_byte,
                const int* cvt, const int64_t* idx, int64_t n, int64_t modulo, int64_t lo,
                int64_t hi, int* err, cudaStream_t stream,
                int64_t cap_blocks = 0);
int mlp_forward(const NetView& v, const float* params, const float* wp, int backend,
                const float* x, int64_t ldx, int64_t M, float* acts, float* out, int64_t ld_out,
                cudaStream_t s);
// One network's operands for a (possibly paired) MLP pass: forward uses
// x/acts/out, backward additionally dout..work.
constexpr int kMaxNets = 4;  // networks advanced in lockstep by mlp_forward_n
struct MlpNet {
  const NetView* v;
  const float* params;
  const float* wp;  // staged weights (tensor-core back ends), else null
  const float* x;
  int64_t ldx;
  bool x_has_ones;
  float* acts;
  float* out;
  int64_t ld_out;
  const float* dout;
  int64_t ld_dout;
  float* grads;
  float* dx;
  int64_t lddx;
  int dx_col0, dx_ncols;
  bool want_dw, zero_logstd;
  float* work;
  // output layer handled outside (the fused PPO output stage): the forward
  // stops at the last hidden layer; the backward starts from dout = dZ of the
  // layer below, held in the work area's first gradient buffer
  // (bwd_head_dz), with that layer's db already produced when head_db_below
  bool head_external = false;
  bool head_db_below = false;
};
// first hidden-gradient buffer of a backward work area (the external head's
// dZ) and the head partial region (skinny_part_floats of the output layer)
float* bwd_head_dz(const NetView& v, float* work, int64_t M);
float* bwd_head_part(const NetView& v, float* work, int64_t M);
// whether the layer below the output layer needs colsum(dZ) for its db (no
// free ones column in its dW GEMM)
bool head_needs_colsum(const MlpNet& N);
// n = 1 or 2 networks in lockstep (grouped tensor-core launches on s; network
// 1's small kernels on `side` between fork/join events when side != null)
// fused forward of the hidden-layer chain (fused_mlp.cu): bf16, widths % 64,
// <= 512, no LayerNorm, up to two networks in one persistent launch
bool fused_fwd_ok(const MlpNet* nets, int n, int dtype);
int fused_forward(const MlpNet* nets, int n, int64_t M, cudaStream_t s);
int mlp_forward_n(const MlpNet* nets, int n, int backend, int64_t M, cudaStream_t s,
                  cudaStream_t side, cudaEvent_t fork, cudaEvent_t join);
// dd: collector for deferred dW GEMMs (bf16 path) shared between calls -- the
// caller runs run_deferred_dw after joining; null: the pass runs its own.
int mlp_backward_n(const MlpNet* nets, int n, int backend, int64_t M, cudaStream_t s,
                   cudaStream_t side, cudaEvent_t fork, cudaEvent_t join,
                   DeferredDw* dd = nullptr);
// dx_cols: compute dX only for input columns [dx_col0, dx_col0 + dx_ncols) (SAC dQ/da);
// want_dw = false skips dW/db (pure input-gradient pass).  x_has_ones: column
// dims[0] of x holds 1.0 (lets the tensor-core dW of layer 0 produce db).
int mlp_backward(const NetView& v, const float* params, const float* wp, int backend,
                 const float* x, int64_t ldx, bool x_has_ones, int64_t M, const float* acts,
                 const float* dout, int64_t ld_dout, float* grads, float* dx, int64_t lddx,
                 int dx_col0, int dx_ncols, bool want_dw, bool zero_logstd, float* work,
                 cudaStream_t s);

}  // namespace ul
