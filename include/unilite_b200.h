/* libunilite_b200 -- C ABI of the B200-native UniLab learner hot path.
 *
 * The reference (arxiv/paper_2605_30313, package `unilite`) has no FFI: its
 * boundary is the Python function/class API re-exported by
 * R:tensornet/__init__.py, R:algos/__init__.py, R:replaypath/__init__.py and
 * R:runtime/__init__.py (R: = /root/reference/pkg/src/unilite/).  Every entry
 * point below replaces one of those Python functions (cited per function);
 * the Python package `paper_2605_30313_b200` binds them with ctypes and keeps
 * the reference names/signatures.
 *
 * Conventions
 *   - all tensor pointers are DEVICE pointers unless named `host_*`;
 *   - `stream` is a cudaStream_t passed as void*; every call is asynchronous
 *     on that stream unless documented otherwise;
 *   - float32 storage, row-major, explicit leading dimensions (`ld*`, in
 *     elements); [T, N] arrays are t-major (element (t, n) at t*N + n);
 *   - flags are uint8 (0/1); indices are int64;
 *   - return value is a status code; on error ul_last_error() holds a message
 *     (thread local).  No C++ exception crosses this boundary.
 */
#ifndef UNILITE_B200_H
#define UNILITE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define UL_ABI_VERSION 1

/* status codes -> Python exception in the shim */
#define UL_OK 0
#define UL_ERR_VALUE 1      /* ValueError            */
#define UL_ERR_INDEX 2      /* IndexError            */
#define UL_ERR_DIVERGENCE 3 /* DivergenceError       */
#define UL_ERR_SLOT 4       /* SlotStateError        */
#define UL_ERR_CUDA 5       /* RuntimeError (CUDA)   */

const char* ul_last_error(void);
int ul_version(void);
int ul_device_count(int* count);
int ul_stream_sync(void* stream);
int ul_memcpy_async(void* dst, const void* src, int64_t bytes, void* stream);
/* async byte fill of device memory (cudaMemsetAsync) */
int ul_memset_async(void* dst, int value, int64_t bytes, void* stream);
/* strided 2-D async copy (row pitch change, e.g. 235 -> 236 floats) */
int ul_memcpy2d_async(void* dst, int64_t dpitch, const void* src, int64_t spitch,
                      int64_t width_bytes, int64_t rows, void* stream);
int ul_host_alloc_pinned(void** ptr, int64_t bytes);
int ul_host_free_pinned(void* ptr);
int ul_event_create(void** ev);
int ul_event_destroy(void* ev);
int ul_event_record(void* ev, void* stream);
int ul_stream_wait_event(void* stream, void* ev);
int ul_event_query(void* ev, int* done);
int ul_event_sync(void* ev);

/* ------------------------------------------------------------------ K1/K2 */
/* GAE reverse scan.  Replaces R:algos/estimators.py:29-63 (+ _next_values
 * :15-26).  truncation_values may be NULL (reference default None).
 * f64 arithmetic, f32 outputs adv/ret [T, N]. */
int ul_gae_f32(const float* rewards, const float* values, const uint8_t* terminated,
               const uint8_t* truncated, const float* truncation_values, const float* bootstrap,
               int64_t T, int64_t N, double gamma, double lam, float* adv, float* ret,
               void* stream);

/* V-trace reverse scan.  Replaces R:algos/estimators.py:66-122.  truncated and
 * truncation_values may be NULL.  Outputs vs, pg_adv [T, N]. */
int ul_vtrace_f32(const float* behavior_logp, const float* target_logp, const float* rewards,
                  const float* values, const uint8_t* terminated, const uint8_t* truncated,
                  const float* truncation_values, const float* bootstrap, int64_t T, int64_t N,
                  double gamma, double rho_bar, double c_bar, float* vs, float* pg_adv,
                  void* stream);

/* --------------------------------------------------------------- K12/K13 */
#define UL_MAX_SEG 4
#define UL_PREP_BLOCKS 296
/* Device-resident optimizer control record (allocate ul_opt_ctl_bytes() of
 * device memory, initialise on the host with ul_opt_ctl_init, upload). */
typedef struct ul_opt_ctl {
  double lr[UL_MAX_SEG];        /* per-segment learning rate            */
  double beta1, beta2, eps;     /* Adam hyper-parameters                */
  double max_norm;              /* joint clip threshold, <= 0 disables  */
  int64_t t[UL_MAX_SEG];        /* Adam step counters (device-updated)  */
  double norm;                  /* pre-clip joint norm of the last call */
  double factor;                /* clip factor applied by the last call */
  double sumsq[UL_MAX_SEG];
  int32_t seg_bad[UL_MAX_SEG];  /* non-finite gradients seen           */
  int32_t seg_update[UL_MAX_SEG];
  int32_t loss_bad;             /* set by loss heads, cleared per step  */
  int32_t diverged;             /* sticky DivergenceError latch         */
  int32_t steps;                /* prepare calls so far                 */
  int32_t fail_step;            /* first failing step, -1 if none       */
  uint32_t ticket;              /* internal last-block counter          */
  int32_t pad0;
  double part[UL_PREP_BLOCKS][UL_MAX_SEG]; /* internal partials */
  int32_t part_bad[UL_PREP_BLOCKS][UL_MAX_SEG];
} ul_opt_ctl;

int64_t ul_opt_ctl_bytes(void);
int ul_opt_ctl_init(ul_opt_ctl* host_ctl, int nseg, const double* lr, double beta1,
                    double beta2, double eps, double max_norm);

/* Joint global-norm clip of nseg gradient segments, in place.  Replaces
 * R:tensornet/adam.py:30-40; the pre-clip norm lands in ctl->norm. */
int ul_clip_global_norm(float* const* grads, const int64_t* sizes, int nseg, ul_opt_ctl* ctl,
                        void* stream);

/* Adam (+ optional joint clip via ctl->max_norm, + finiteness latch).
 * Replaces R:tensornet/adam.py:43-80 (run over several segments it is the
 * PPO step's clip_global_norm([actor, critic]) + two adam_step calls,
 * R:algos/ppo.py:181-185). */
int ul_adam_step(float* const* params, float* const* grads, float* const* m, float* const* v,
                 const int64_t* sizes, int nseg, ul_opt_ctl* ctl, int write_clipped_grads,
                 void* stream);

/* Polyak target update target <- (1-tau) target + tau online over a flat
 * parameter vector.  Replaces R:algos/sac.py:100-108. */
int ul_polyak(float* target, const float* online, int64_t n, double tau, void* stream);

/* ------------------------------------------------------------- K7/K8 MLP */
#define UL_MAX_LAYERS 8
/* A dense ELU MLP (R:tensornet/mlp.py:16-76): dims = (in, h1, ..., out),
 * parameters in ONE flat float32 buffer in ModelParams.flat order
 * (W0 (out x in, row-major), b0, W1, b1, ..., log_std). */
typedef struct ul_net_desc {
  int32_t n_layers;
  int32_t dims[UL_MAX_LAYERS + 1];
  /* 1: LayerNorm (gain g, shift beta; eps 1e-5) between every hidden layer's
   * affine map and its ELU -- an extension for cfg3's critics, not in the
   * reference.  Params per hidden layer become W, b, g, beta; hidden widths
   * must be multiples of 4. */
  int32_t layer_norm;
} ul_net_desc;

/* number of floats of the flat parameter vector (incl. log_std) */
int64_t ul_net_param_count(const ul_net_desc* net);
/* activation cache floats for a batch of M rows (hidden layers only; layer
 * i's rows have pitch round_up(d_i + 1, 4): 16 B rows + a ones column) */
int64_t ul_mlp_act_floats(const ul_net_desc* net, int64_t M);
/* backward workspace floats for a batch of M rows */
int64_t ul_mlp_bwd_work_floats(const ul_net_desc* net, int64_t M);
/* staged-weight floats (tensor-core path: W rows padded to 16 B; the bf16
 * staging of UL_GEMM_BF16 fits in the same buffer) */
int64_t ul_mlp_wstage_floats(const ul_net_desc* net);
/* copy the flat W_i into the staged 16 B-row layout (call after every update) */
int ul_stage_weights(const ul_net_desc* net, const float* params, float* wstage, void* stream);

/* GEMM back ends for the MLP passes */
#define UL_GEMM_FP32 0 /* SIMT fp32 FFMA: the exact-fp32 parity path            */
#define UL_GEMM_TF32 1 /* tcgen05.mma kind::tf32 + TMEM + TMA (needs wstage)    */
#define UL_GEMM_BF16 2 /* tcgen05.mma kind::f16 (bf16 operands, fp32 accumulate):
                        * x, hidden activations and hidden gradients stored bf16
                        * (rows of round_up(d + 1, 8)); params, grads, outputs
                        * and the upstream gradient stay fp32 (1e-2 tolerance) */
#define UL_GEMM_TF32X3 3 /* tcgen05 kind::tf32 over 3xTF32-split fp32 operands
                          * (hi*hi + hi*lo + lo*hi as one GEMM over a tripled K):
                          * the fp32-parity path on the tensor cores */
/* activation row pitch (elements) of a hidden layer of width d for a back end */
int64_t ul_mlp_act_ld(int d, int backend);
/* stage W for a back end (UL_GEMM_BF16 writes bf16 rows of round_up(in, 8)) */
int ul_stage_weights_ex(const ul_net_desc* net, const float* params, void* wstage, int backend,
                        void* stream);

/* Forward: out[M, out] (ld_out) = MLP(x[M, in] (ldx)); hidden activations are
 * cached in `acts` (ul_mlp_act_floats).  Replaces R:tensornet/mlp.py:153-172. */
int ul_mlp_forward(const ul_net_desc* net, const float* params, const float* wstage, int backend,
                   const float* x, int64_t ldx, int64_t M, float* acts, float* out,
                   int64_t ld_out, void* stream);

/* Two independent networks over the same M rows (APPO's target recompute:
 * the actor on obs rows, the critic on critic_obs rows) in lockstep, one
 * grouped tensor-core launch per layer; per network identical to
 * ul_mlp_forward.  Replaces the pair of forwards at R:algos/appo.py:35-39. */
int ul_mlp_forward2(const ul_net_desc* net_a, const float* params_a, const float* wstage_a,
                    const float* x_a, int64_t ldx_a, float* acts_a, float* out_a, int64_t ld_out_a,
                    const ul_net_desc* net_b, const float* params_b, const float* wstage_b,
                    const float* x_b, int64_t ldx_b, float* acts_b, float* out_b, int64_t ld_out_b,
                    int backend, int64_t M, void* stream);

/* Backward from the upstream gradient dout[M, out] (ld_dout): writes the flat
 * gradient vector `grads` (log_std slot zeroed) and, if dx != NULL, the input
 * gradient dx[M, in] (lddx).  x_has_ones: column `in` of x holds 1.0 (lets
 * the tensor-core dW of layer 0 emit db).  Replaces R:tensornet/mlp.py:175-198. */
int ul_mlp_backward(const ul_net_desc* net, const float* params, const float* wstage, int backend,
                    const float* x, int64_t ldx, int x_has_ones, int64_t M, const float* acts,
                    const float* dout, int64_t ld_dout, float* grads, float* dx, int64_t lddx,
                    float* work, void* stream);

/* Plain fp32 GEMM C = op(A) op(B) (+bias/ELU epilogues), exposed for tests.
 * layout bit0: A is K-major ([M,K] row-major) else M-major ([K,M]);
 * layout bit1: B is K-major ([N,K] row-major) else N-major ([K,N]).
 * epi: 0 store, 1 +bias, 2 ELU(+bias), 3 *(min(aux,0)+1). */
int ul_gemm_f32(int layout, int epi, int64_t M, int64_t N, int64_t K, const float* A,
                int64_t lda, const float* B, int64_t ldb, float* C, int64_t ldc,
                const float* bias, const float* aux, int64_t ldaux, void* stream);

/* Same contract on the tcgen05 tensor-core kernel.  dtype 0: fp32 operands
 * (kind::tf32, fp32 out; M >= 128, N >= 64, K >= 32); dtype 1: bf16 operands
 * (kind::f16; epilogues 2 and 3 read/write bf16, 0 and 1 write fp32; any
 * shape).  16 B-aligned operands and row pitches; splits > 1 writes split-K
 * partials [splits][M][ldc] at C. */
int ul_gemm_tc(int layout, int epi, int64_t M, int64_t N, int64_t K, const void* A, int64_t lda,
               const void* B, int64_t ldb, void* C, int64_t ldc, const float* bias,
               const void* aux, int64_t ldaux, int splits, int dtype, void* stream);

/* Diagnostics (no reference counterpart): with UL_TC_TRACE=1 in the
 * environment every tcgen05 GEMM launch records CTA 0's event timestamps and
 * per-role wait-cycle sums; ul_tc_trace copies the kTraceSlots (160) u64
 * slots to host_out, ul_tc_trace_reset zeroes them (tools/trace_gemm.py). */
int ul_tc_trace(unsigned long long* host_out);
int ul_tc_trace_reset(void);

/* ------------------------------------------------- K4 / K5 / K6 data path */
/* Gather rows of up to 12 arrays sharing one index vector (PPO minibatch
 * copies of R:algos/ppo.py:161-176; replay sample copy of
 * R:replaypath/storage.py:106-110).  Strides / row widths in BYTES.  Rows
 * outside [lo, hi) are skipped and set *err (device int, may be NULL);
 * modulo > 0 maps absolute replay indices to ring slots.  ones_byte (may be
 * NULL): per desc, byte offset of a float overwritten with 1.0 in every
 * gathered row (-1 = none; the MLP's bias column). */
int ul_gather_rows(int ndesc, const void* const* src, void* const* dst,
                   const int64_t* src_stride, const int64_t* dst_stride, const int64_t* row_bytes,
                   const int64_t* ones_byte, const int64_t* idx, int64_t n, int64_t modulo,
                   int64_t lo, int64_t hi, int* err, void* stream);
/* ul_gather_rows + a per-desc conversion flag: cvt[d] = 1 turns fp32 source
 * rows into bf16 destination rows (row_bytes / ones_byte count SOURCE bytes;
 * the bf16 staging of a PPO segment's observation rows). */
/* fp32 rows [rows, lds] (4-byte aligned, e.g. unpadded H2D landing rows) ->
 * bf16 rows [rows, ldd] (ldd % 8 == 0): columns >= width zero, column
 * ones_col (>= 0) set to 1.0 -- the once-per-segment bf16 observation staging. */
int ul_rows_to_bf16(const float* src, int64_t lds, int width, void* dst, int64_t ldd,
                    int64_t rows, int ones_col, void* stream);
int ul_gather_rows_cvt(int ndesc, const void* const* src, void* const* dst,
                       const int64_t* src_stride, const int64_t* dst_stride,
                       const int64_t* row_bytes, const int64_t* ones_byte, const int* cvt,
                       const int64_t* idx, int64_t n, void* stream);

/* Replay ring insert (R:replaypath/storage.py:76-104): n rows of `width`
 * floats at absolute index `head`; rows may be pinned-host or device memory.
 * n >= cap keeps only the last cap rows (each at its own absolute slot). */
int ul_ring_insert(float* ring, int64_t cap, int64_t width, int64_t head, const float* rows,
                   int64_t n, void* stream);

/* float64 -> float32 narrowing of k <= 8 device arrays in one launch (the
 * rollout segment's float64 per-step scalars, landed by a raw H2D) */
int ul_narrow_f64(int k, const double* const* src, float* const* dst, const int64_t* n,
                  void* stream);

/* Device permutation of [0, n) (performance mode only; NOT the numpy Philox
 * shuffle of R:algos/ppo.py:162). */
int ul_device_permutation(int64_t n, uint64_t key, int64_t* out, void* stream);
/* count (<= 16) permutations of [0, n) in one launch, one per host key:
 * out + e * ld holds the permutation of key e (the per-epoch minibatch orders). */
int ul_device_permutations(int64_t n, int count, const uint64_t* host_keys, int64_t* out,
                           int64_t ld, void* stream);

/* ------------------------------------------- FlashSAC collector transforms */
/* Device ReturnStdNormalizer.normalize + NStepPacker.push + replay insert
 * (R:algos/estimators.py:153-207, R:replaypath/storage.py:17-46; SURVEY.md
 * 8(f) item 3).  state = ul_nstep_state_bytes(...) zeroed bytes; inputs for
 * one env step are device arrays (obs/next_obs [N,d], act [N,a], r [N] f32,
 * term/trunc [N] u8); emitted codec rows land at ring[(head + i) % cap]
 * (pitch ldr floats) in the reference's env-major order; *count_out (device
 * or pinned) = rows written.  norm_gamma <= 0: no reward normalisation. */
int64_t ul_nstep_state_bytes(int n_envs, int n, int obs_dim, int act_dim);
int ul_nstep_push(void* state, int n_envs, int n, int obs_dim, int act_dim, double gamma,
                  double norm_gamma, double g_max, double eps, const float* obs, const float* act,
                  const float* r, const float* next_obs, const uint8_t* term,
                  const uint8_t* trunc, float* ring, int64_t cap, int64_t ldr, int64_t head,
                  int64_t* count_out, void* stream);
/* normaliser (count, mean, m2, std) -> out[4] */
int ul_nstep_norm_stats(void* state, int n_envs, int n, int obs_dim, int act_dim, double* out,
                        void* stream);

/* ------------------------------------------------------------ K3 normaliser */
/* state = float64 [1 + 2D]: count, mean[D], var[D]
 * (R:tensornet/normalizer.py:14-25).  work = ul_norm_work_bytes(D) bytes of
 * zero-initialised device memory. */
int64_t ul_norm_work_bytes(int64_t D);
/* Normalizer.update (R:tensornet/normalizer.py:27-45) */
int ul_norm_update(const float* x, int64_t B, int64_t D, int64_t ldx, double* state, void* work,
                   int frozen, void* stream);
/* Normalizer.apply (R:tensornet/normalizer.py:47-49) */
int ul_norm_apply(const float* x, int64_t B, int64_t D, int64_t ldx, const double* state,
                  float* out, int64_t ldo, void* stream);

/* Diagonal Gaussian log-prob summed over A action dims
 * (R:tensornet/distributions.py:11-18); out[n] float32. */
int ul_gaussian_logp(const float* mean, int64_t ld_mean, const float* log_std,
                     const float* action, int64_t ld_act, int64_t n, int A, float* out,
                     void* stream);

/* --------------------------------------------------- PPO / APPO update plan */
#define UL_MAX_ACT 64
typedef struct ul_ppo_stats {
  double policy_sum, value_sum, entropy_sum, kl_epoch_sum, kl_last;
  int64_t steps;
} ul_ppo_stats;

typedef struct ul_ppo_plan_desc {
  ul_net_desc actor, critic;
  int64_t rows;                     /* T*N transitions per segment            */
  int64_t ld_obs, ld_cobs, ld_act;  /* row strides of the bound device arrays */
  int32_t epochs, minibatches;
  double clip_param, entropy_coef, value_loss_coef;
  int32_t use_clipped_value_loss;
  double max_grad_norm;
  int32_t world_size, rank;         /* data-parallel minibatch sharding       */
  int32_t raw_advantages;           /* 1: advantages already normalised       */
  int32_t local_shards;             /* 0: every rank holds the whole segment and
                                       takes rows [rank*mb/G, (rank+1)*mb/G) of
                                       each permuted minibatch; 1: each rank owns
                                       its own segment rows (weak scaling) and a
                                       global minibatch is the union of the
                                       ranks' local minibatches              */
  int32_t gemm_backend;             /* UL_GEMM_FP32 / _TF32 / _BF16 / _TF32X3 */
  int32_t obs_bf16;                 /* 1: obs / cobs bindings hold bf16 rows (ld_obs /
                                       ld_cobs in elements, the ones column already
                                       set); UL_GEMM_BF16 only                */
} ul_ppo_plan_desc;

typedef struct ul_ppo_bindings {
  const float* obs;   /* [rows, ld_obs]  */
  const float* cobs;  /* [rows, ld_cobs] */
  const float* act;   /* [rows, ld_act]  */
  const float* blogp; /* [rows] behaviour log-prob          */
  const float* adv;   /* [rows] advantages (pg_adv for APPO) */
  const float* ret;   /* [rows] returns (vs for APPO)       */
  const float* oldv;  /* [rows] old values                  */
  float* actor_params;
  float* critic_params;
  float* actor_m;
  float* actor_v;
  float* critic_m;
  float* critic_v;
  const int64_t* perm; /* [epochs, rows] minibatch permutations */
  float* reduce_buf;   /* optional caller-owned all-reduce buffer of
                          ul_ppo_plan_reduce_buffer() floats, NULL = internal */
} ul_ppo_bindings;

typedef struct ul_ppo_result {
  double policy_loss, value_loss, entropy, kl, grad_norm;
  int64_t t_actor, t_critic;
  int32_t diverged, fail_step;
} ul_ppo_result;

/* The epoch x minibatch loop of R:algos/ppo.py:136-199 as a native plan:
 * per step gather -> actor/critic forward -> loss head -> backward ->
 * [all-reduce of the plan's gradient buffer] -> loss check, joint clip,
 * Adam(actor), Adam(critic).  Whole updates replay as one CUDA graph. */
int ul_ppo_plan_create(const ul_ppo_plan_desc* desc, void** plan);
int ul_ppo_plan_destroy(void* plan);
int ul_ppo_plan_bind(void* plan, const ul_ppo_bindings* b);
/* upload lr / step counters, reset stats, advantage statistics */
int ul_ppo_plan_begin(void* plan, double lr_actor, double lr_critic, int64_t t_actor,
                      int64_t t_critic, void* stream);
/* Data-parallel "local" shards: this rank's raw advantage sums [sum A,
 * sum A^2, n] after begin (3 doubles into dst), and the (mean, std) of the
 * loss head from the all-reduced sums (normalize_advantages over the union
 * of the ranks' rows, R:algos/ppo.py:132-133). */
int ul_ppo_plan_adv_sums(void* plan, double* dst, void* stream);
int ul_ppo_plan_adv_finalize(void* plan, const double* sums, void* stream);
int ul_ppo_plan_step_grads(void* plan, int epoch, int k, void* stream);
int ul_ppo_plan_step_apply(void* plan, int epoch, int k, void* stream);
/* contiguous [actor grads | critic grads | 3 loss partials] buffer that a
 * data-parallel caller all-reduces (sum) between step_grads and step_apply */
int ul_ppo_plan_reduce_buffer(void* plan, float** ptr, int64_t* n);
/* begin + every step (graph-captured when use_graph) */
int ul_ppo_plan_run(void* plan, double lr_actor, double lr_critic, int64_t t_actor,
                    int64_t t_critic, int use_graph, void* stream);
/* ul_ppo_plan_run (graph) enqueued behind `prev`'s update on the same stream
 * before the host has read prev's statistics: the Adam step counters and the
 * divergence latch continue from prev's device controller (prev may be plan). */
int ul_ppo_plan_run_after(void* plan, const void* prev, double lr_actor, double lr_critic,
                          void* stream);
/* Enqueue the D2H of the update's result records behind it; the next
 * ul_ppo_plan_finish then waits for those records only (not the stream). */
int ul_ppo_plan_collect(void* plan, void* stream);
/* One epoch of ul_ppo_plan_run as its own CUDA graph (epoch 0 also uploads the
 * controller and stages the weights): lets the caller upload epoch e + 1's
 * host permutation while epoch e runs.  Epochs must run 0, 1, ... in order. */
int ul_ppo_plan_run_epoch(void* plan, int epoch, double lr_actor, double lr_critic,
                          int64_t t_actor, int64_t t_critic, void* stream);
/* D2H of the statistics + stream sync; UL_ERR_DIVERGENCE if a step diverged */
int ul_ppo_plan_finish(void* plan, ul_ppo_result* out, void* stream);
/* kernels per update (graph kernel nodes) and algorithmic GEMM FLOPs per update */
int ul_ppo_plan_counts(void* plan, int64_t* kernels_per_update, double* gemm_flops_per_update);
/* One un-graphed update with CUDA events around every kernel class:
 * ms[0] MLP passes (GEMMs), ms[1] gather, ms[2] heads/finalize, ms[3] optimizer,
 * ms[4] all, ms[5] the MLP backward part of ms[0], of which ms[6] the dX chains and
 * ms[7] the batched dW launch (the rest: the deferred reduction).  ms holds 8 doubles.
 * Synchronises the stream. */
int ul_ppo_plan_profile(void* plan, double lr_actor, double lr_critic, int64_t t_actor,
                        int64_t t_critic, double* ms, void* stream);

/* ------------------------------------------ SAC / FastSAC / FlashSAC plan */
/* Device-resident SAC scalars: log_alpha and its ScalarAdam state
 * (R:algos/sac.py:35-53), plus the last update's loss terms. */
typedef struct ul_sac_ctl {
  double log_alpha, a_m, a_v, a_t, alpha_lr;
  double critic_loss, actor_loss, alpha_loss, logp_sum;
  int32_t diverged;      /* 0 ok, 1 critic side, 2 actor / alpha side (first failure) */
  int32_t fail_update;   /* index of the first diverged update of a run, -1 none  */
} ul_sac_ctl;

typedef struct ul_sac_plan_desc {
  ul_net_desc actor;  /* obs -> act                                   */
  ul_net_desc critic; /* obs+act -> 1 (q1, q2 and both targets)        */
  int64_t batch;
  int32_t obs_dim, act_dim;
  double gamma, tau, target_entropy, max_grad_norm;
  int32_t gemm_backend;
  int32_t world_size; /* data-parallel ranks: `batch` is this rank's share, losses
                       * and gradients are scaled by batch * world_size (0 = 1) */
} ul_sac_plan_desc;

typedef struct ul_sac_bindings {
  float *actor, *actor_m, *actor_v;
  float *q1, *q1_m, *q1_v;
  float *q2, *q2_m, *q2_v;
  float *q1t, *q2t;
  /* optional caller-owned all-reduce buffers (NULL = plan-owned):
   * critic_red [2*Pq + 4] = [g_q1 | g_q2 | critic loss part], actor_red
   * [Pa + 4] = [g_a | actor loss part | sum log pi] */
  float *critic_red, *actor_red;
} ul_sac_bindings;

/* ------------------------------------------- per-call SAC / Gaussian API */
/* Kernels behind the reference's per-call functions (the fused update is the
 * plan below).  Reductions write per-block partials into `work`
 * (ul_api_work_doubles() doubles, zeroed once by the caller; its last slot
 * is the replay-safe last-block ticket). */
int64_t ul_api_work_doubles(void);
/* gaussian_dist / squashed_log_prob (R:tensornet/distributions.py:29-70),
 * float64.  mode 0: plain sample (x = eps), 1: plain evaluation (x = action),
 * 2: squashed sample (x = eps), 3: squashed evaluation (x = action, clipped
 * to +-(1 - 1e-6), u = atanh), 4: squashed log-prob of given (u = x, a = a_in).
 * sample / u_out [n, A] (may be NULL), logp [n]. */
int ul_gaussian_dist(const double* mean, int64_t ldm, const double* log_std, const double* x,
                     int64_t ldx, const double* a_in, int64_t n, int A, int mode, double* sample,
                     double* u_out, double* logp, void* stream);
/* sample_squashed (R:tensornet/distributions.py:73-84) in float32 arithmetic:
 * u = mean + exp(log_std) eps, a = tanh(u), logp [n] */
int ul_sample_squashed(const float* mean, int64_t ldm, const float* log_std, const float* eps,
                       int64_t lde, int64_t n, int A, float* a, float* u, float* logp,
                       void* stream);
/* critic_target's y = r + gamma^n_used (1 - term)(min(q1t, q2t) - alpha logp)
 * (R:algos/sac.py:111-125), float64 */
int ul_sac_soft_target(const double* r, const double* term, const double* nused,
                       const float* q1t, const float* q2t, const float* logp, double log_alpha,
                       double gamma, int64_t n, double* y, void* stream);
/* critic_loss_and_grads head (R:algos/sac.py:128-136): *loss = mean((q-y)^2),
 * dq = 2 (q - y) / n cast to float32 (device scalar / vector) */
int ul_sac_mse_head(const float* q, const double* y, int64_t n, float* dq, double* loss,
                    double* work, void* stream);
/* actor_loss_and_grads pick (R:algos/sac.py:194-205): *loss = mean(alpha
 * logp - min(q1, q2)), d1 = [q1 <= q2], d2 = 1 - d1 */
int ul_sac_pick_head(const float* q1, const float* q2, const float* logp, int64_t n,
                     double log_alpha, float* d1, float* d2, double* loss, double* work,
                     void* stream);
/* actor gradient head (R:algos/sac.py:207-217): dQ/da = dq1 + dq2 (rows of
 * ldq, the action columns); dmean [n, A]; dlog_std [A] is ADDED to */
int ul_sac_actor_head(const float* a, const float* eps, const float* dq1, const float* dq2,
                      int64_t ldq, const float* log_std, int64_t n, int A, double log_alpha,
                      float* dmean, float* dlog_std, double* work, void* stream);
/* *out = sum_i (x[i] + shift), float64 (alpha_loss_and_grad's mean) */
int ul_sum_f64(const float* x, int64_t n, double shift, double* out, double* work, void* stream);

/* sac_update (R:algos/sac.py:139-178) as a native plan.  Batches come as
 * codec rows (R:replaypath/storage.py:17-46) gathered from a device replay
 * ring or a staged batch. */
int ul_sac_plan_create(const ul_sac_plan_desc* desc, void** plan);
int ul_sac_plan_destroy(void* plan);
int ul_sac_plan_bind(void* plan, const ul_sac_bindings* b);
/* rows[(idx[i] % modulo)] (pitch in floats); idx NULL = rows 0..B-1 */
int ul_sac_plan_load_rows(void* plan, const float* rows, int64_t pitch, const int64_t* idx,
                          int64_t modulo, int64_t lo, int64_t hi, int* err, void* stream);
/* upload alpha state + per-network (lr, t): order actor, q1, q2 (async, no
 * host sync: pinned staging per record) */
int ul_sac_plan_begin(void* plan, const ul_sac_ctl* host_ctl, const double* lrs,
                      const int64_t* ts, void* stream);
/* room for runs of up to n updates: noise [n][2][B][A] float32 (per update:
 * eps of the target, eps of the actor step) and per-update statistics */
int ul_sac_plan_reserve(void* plan, int n_updates);
/* noise buffer (reserved updates x [2, B, A]); fill it from the host (parity
 * mode: the reference draw order) or on the device */
int ul_sac_plan_noise_ptr(void* plan, float** eps);
int ul_sac_plan_device_noise(void* plan, uint64_t key, uint64_t counter, void* stream);
/* n consecutive sac_update calls on the loaded batch (FlashSAC's
 * updates_per_step loop, R:runtime/sac_runner.py:313-321) as ONE CUDA graph
 * launch: update u takes the actor / alpha step when (update_count0 + u + 1)
 * % policy_frequency == 0.  Everything stays on the device between updates;
 * the first divergence latches every later step off (the reference raises). */
int ul_sac_plan_run(void* plan, int n_updates, int64_t update_count0, int policy_frequency,
                    void* stream);
int ul_sac_plan_update(void* plan, int do_actor, void* stream);
/* The same update split at its two data-parallel exchange points (SURVEY
 * 8(e)): critic_grads -> all-reduce(critic buffer) -> critic_apply ->
 * [actor_grads -> all-reduce(actor buffer) -> actor_apply] -> polyak.
 * ul_sac_plan_update == the sequence without exchanges. */
int ul_sac_plan_reduce_buffers(void* plan, float** critic, int64_t* n_critic, float** actor,
                               int64_t* n_actor);
int ul_sac_plan_critic_grads(void* plan, void* stream);
int ul_sac_plan_critic_apply(void* plan, void* stream);
int ul_sac_plan_actor_grads(void* plan, void* stream);
int ul_sac_plan_actor_apply(void* plan, void* stream);
int ul_sac_plan_polyak(void* plan, void* stream);
/* D2H of the control records (+ one sync): ts = step counters (actor, q1,
 * q2); stats (may be NULL): n x [critic_loss, actor_loss, alpha_loss, alpha]
 * of the last run (NaN where an update took no actor step) */
int ul_sac_plan_finish(void* plan, ul_sac_ctl* out, int64_t* ts, double* stats, int n,
                       void* stream);

#ifdef __cplusplus
}
#endif
#endif /* UNILITE_B200_H */
