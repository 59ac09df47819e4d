#include <cuda_bf16.h>
// Native PPO/APPO update plan: the epoch x minibatch loop of R:algos/ppo.py:136-199.
//
// A plan owns every per-step device buffer (minibatch staging, activation
// caches, gradient/all-reduce buffer, loss partials, optimizer control) so a
// whole update is a fixed sequence of launches on fixed pointers; it is
// captured once into a CUDA graph and replayed per update (one launch, no
// host round trip until the statistics are read back).  Per step:
//   gather (K4) -> actor fwd, critic fwd (K7) -> PPO head (K9) ->
//   actor bwd, critic bwd (K8) -> [caller all-reduce] -> loss finalize ->
//   joint clip + Adam(actor) + Adam(critic) (K13).
#include <stdlib.h>

#include <new>

#include "learner.cuh"

namespace ul {
namespace {


struct PpoPlan {
  ul_ppo_plan_desc d{};
  NetView va{}, vc{};
  int A = 0;
  int64_t rows = 0, mb = 0, mb_local = 0;
  int64_t ld_mo = 0, ld_mc = 0, ld_ma = 0;  // minibatch staging row strides (elements)
  int dt = kF32;                            // MLP activation / input storage
  int64_t Pa = 0, Pc = 0;
  // device arena
  char* arena = nullptr;
  float *mb_obs = nullptr, *mb_cobs = nullptr, *mb_act = nullptr, *mb_scal = nullptr;
  float *acts_a = nullptr, *acts_c = nullptr, *out_a = nullptr, *out_c = nullptr;
  float *dmean = nullptr, *dv = nullptr, *work = nullptr, *work_c = nullptr, *red = nullptr,
        *red_own = nullptr;
  float *wst_a = nullptr, *wst_c = nullptr;  // staged (16 B-row) weights, tensor-core path
  double *head_part = nullptr, *adv_stats = nullptr, *adv_part = nullptr;
  unsigned int* tickets = nullptr;  // [0] head, [1] adv stats, [2] folded prepare
  // K13 prepare folded into the step's gradient reduction (single process,
  // fused-head bf16 step; UL_FOLD_PREP=0 disables): block partials
  static constexpr int kFoldCap = 8192;
  double* fold_part = nullptr;
  int* fold_bad = nullptr;
  bool fold_on = false;
  bool prep_folded = false;  // the last step_grads ran the prepare tail
  ul_opt_ctl* ctl_d = nullptr;
  ul_ppo_stats* st_d = nullptr;
  // pinned mirrors
  ul_opt_ctl* ctl_h = nullptr;
  ul_ppo_stats* st_h = nullptr;
  ul_ppo_bindings b{};
  bool bound = false;
  cudaStream_t cap_stream = nullptr;
  cudaStream_t side = nullptr;  // critic branch (fork/join inside each step)
  cudaEvent_t ev_in = nullptr, ev_out = nullptr, ev_fork = nullptr, ev_join = nullptr;
  // ul_ppo_plan_collect: result records D2H'd behind the update, ev_res marks them
  cudaEvent_t ev_res = nullptr;
  bool collected = false;
  // the next minibatch's gather runs on the side stream under this step's
  // optimizer (and all-reduce) -- ev_gfork / ev_gjoin bracket it
  cudaEvent_t ev_gfork = nullptr, ev_gjoin = nullptr;
  bool gathered_ahead = false;
  cudaGraphExec_t graph = nullptr;
  int64_t graph_kernels = 0;
  // per-epoch graphs (parity mode: the host draws epoch e + 1's permutation
  // while epoch e runs); epoch 0's also stages the weights
  static constexpr int kMaxEpochGraphs = 32;
  cudaGraphExec_t egraph[kMaxEpochGraphs] = {};
  bool epoch_mode = false;  // capturing / running one epoch per graph
  // optional per-phase CUDA-event profiling (ul_ppo_plan_profile)
  struct Prof {
    static constexpr int kMax = 4096;
    cudaEvent_t ev[kMax];
    int cat[kMax];
    int n = 0;
    bool on = false;
  };
  Prof* prof = nullptr;
};

// record a phase boundary: the interval ending here belongs to class `cat`
inline void mark(PpoPlan* p, int cat, cudaStream_t s) {
  if (!p->prof || !p->prof->on || p->prof->n >= PpoPlan::Prof::kMax) return;
  auto* pr = p->prof;
  cudaEventRecord(pr->ev[pr->n], s);
  pr->cat[pr->n] = cat;
  pr->n++;
}

size_t ctl_header_bytes() { return offsetof(ul_opt_ctl, part); }

int alloc_plan(PpoPlan* p) {
  const int64_t ml = p->mb_local;
  size_t off = 0;
  auto carve = [&](size_t bytes) {
    size_t o = off;
    off += (bytes + 255) & ~size_t(255);
    return o;
  };
  const size_t o_obs = carve(sizeof(float) * ml * p->ld_mo);
  const size_t o_cobs = carve(sizeof(float) * ml * p->ld_mc);
  const size_t o_act = carve(sizeof(float) * ml * p->ld_ma);
  const size_t o_scal = carve(sizeof(float) * ml * 4);
  const size_t o_acta = carve(sizeof(float) * act_floats(p->va, ml));
  const size_t o_actc = carve(sizeof(float) * act_floats(p->vc, ml));
  const size_t o_outa = carve(sizeof(float) * ml * p->A);
  const size_t o_outc = carve(sizeof(float) * ml);
  const size_t o_dmean = carve(sizeof(float) * ml * p->A);
  const size_t o_dv = carve(sizeof(float) * ml);
  const int64_t wa = bwd_work_floats(p->va, ml), wc = bwd_work_floats(p->vc, ml);
  const size_t o_work = carve(sizeof(float) * wa);
  const size_t o_workc = carve(sizeof(float) * wc);
  const size_t o_red = carve(sizeof(float) * (p->Pa + p->Pc + 4));
  const size_t o_hp = carve(sizeof(double) * ppo_head_partial_doubles(ml, p->A));
  const size_t o_as = carve(sizeof(double) * 8);  // mean, std, S1, S2, n
  const size_t o_ap = carve(sizeof(double) * 2 * kAdvStatBlocks);
  const size_t o_tk = carve(sizeof(unsigned int) * 8);
  const size_t o_ctl = carve(sizeof(ul_opt_ctl));
  const size_t o_st = carve(sizeof(ul_ppo_stats));
  const size_t o_fp = carve(sizeof(double) * 2 * PpoPlan::kFoldCap);
  const size_t o_fb = carve(sizeof(int) * 2 * PpoPlan::kFoldCap);
  const size_t o_wa = carve(sizeof(float) * p->va.wp_total);
  const size_t o_wc = carve(sizeof(float) * p->vc.wp_total);
  UL_CUDA(cudaMalloc(&p->arena, off));
  UL_CUDA(cudaMemset(p->arena, 0, off));
  char* a = p->arena;
  p->mb_obs = (float*)(a + o_obs);
  p->mb_cobs = (float*)(a + o_cobs);
  p->mb_act = (float*)(a + o_act);
  p->mb_scal = (float*)(a + o_scal);
  p->acts_a = (float*)(a + o_acta);
  p->acts_c = (float*)(a + o_actc);
  p->out_a = (float*)(a + o_outa);
  p->out_c = (float*)(a + o_outc);
  p->dmean = (float*)(a + o_dmean);
  p->dv = (float*)(a + o_dv);
  p->work = (float*)(a + o_work);
  p->work_c = (float*)(a + o_workc);
  p->red_own = (float*)(a + o_red);
  p->red = p->red_own;
  p->head_part = (double*)(a + o_hp);
  p->adv_stats = (double*)(a + o_as);
  p->adv_part = (double*)(a + o_ap);
  p->tickets = (unsigned int*)(a + o_tk);
  p->ctl_d = (ul_opt_ctl*)(a + o_ctl);
  p->st_d = (ul_ppo_stats*)(a + o_st);
  p->fold_part = (double*)(a + o_fp);
  p->fold_bad = (int*)(a + o_fb);
  p->wst_a = (float*)(a + o_wa);
  p->wst_c = (float*)(a + o_wc);
  UL_CUDA(cudaHostAlloc(&p->ctl_h, sizeof(ul_opt_ctl), cudaHostAllocPortable));
  UL_CUDA(cudaHostAlloc(&p->st_h, sizeof(ul_ppo_stats), cudaHostAllocPortable));
  UL_CUDA(cudaStreamCreateWithFlags(&p->cap_stream, cudaStreamNonBlocking));
  UL_CUDA(cudaEventCreateWithFlags(&p->ev_in, cudaEventDisableTiming));
  UL_CUDA(cudaEventCreateWithFlags(&p->ev_res, cudaEventDisableTiming));
  UL_CUDA(cudaEventCreateWithFlags(&p->ev_out, cudaEventDisableTiming));
  UL_CUDA(cudaStreamCreateWithFlags(&p->side, cudaStreamNonBlocking));
  UL_CUDA(cudaEventCreateWithFlags(&p->ev_fork, cudaEventDisableTiming));
  UL_CUDA(cudaEventCreateWithFlags(&p->ev_gfork, cudaEventDisableTiming));
  UL_CUDA(cudaEventCreateWithFlags(&p->ev_gjoin, cudaEventDisableTiming));
  UL_CUDA(cudaEventCreateWithFlags(&p->ev_join, cudaEventDisableTiming));
  return UL_OK;
}

void free_plan(PpoPlan* p) {
  if (p->prof) {
    for (int i = 0; i < PpoPlan::Prof::kMax; ++i) cudaEventDestroy(p->prof->ev[i]);
    delete p->prof;
  }
  if (p->graph) cudaGraphExecDestroy(p->graph);
  for (int e = 0; e < PpoPlan::kMaxEpochGraphs; ++e)
    if (p->egraph[e]) cudaGraphExecDestroy(p->egraph[e]);
  if (p->arena) cudaFree(p->arena);
  if (p->ctl_h) cudaFreeHost(p->ctl_h);
  if (p->st_h) cudaFreeHost(p->st_h);
  if (p->cap_stream) cudaStreamDestroy(p->cap_stream);
  if (p->ev_in) cudaEventDestroy(p->ev_in);
  if (p->ev_res) cudaEventDestroy(p->ev_res);
  if (p->ev_out) cudaEventDestroy(p->ev_out);
  if (p->side) cudaStreamDestroy(p->side);
  if (p->ev_fork) cudaEventDestroy(p->ev_fork);
  if (p->ev_gfork) cudaEventDestroy(p->ev_gfork);
  if (p->ev_gjoin) cudaEventDestroy(p->ev_gjoin);
  if (p->ev_join) cudaEventDestroy(p->ev_join);
}

// Both networks' MLP pass.  Grouped: lockstep layers with one tensor-core
// launch per layer for both networks (default for the forward: twice the
// tiles per launch, better wave quantisation).  Otherwise the critic runs on
// the side stream concurrently with the actor (its kernels fill the gaps and
// tails of the actor's); default for the backward, whose dW GEMMs of both
// networks are deferred into one batched launch either way.
// UL_GROUP=0/1 forces both; UL_GROUP_FWD / UL_GROUP_BWD each pass.
// dd (backward, may be null): deferred-dW collector, possibly pre-seeded with
// the fused output stage's partial reductions
int gather_ahead(PpoPlan* p, int e, int k, cudaStream_t s);

int mlp_pass(PpoPlan* p, MlpNet* nets, int be, int64_t ml, cudaStream_t s, bool fwd,
             DeferredDw* dd = nullptr, int ahead_e = -1, int ahead_k = -1) {
  static int g_fwd = -1, g_bwd = -1;
  if (g_fwd < 0) {
    auto env = [](const char* n, int def) {
      const char* e = getenv(n);
      return e ? (atoi(e) != 0 ? 1 : 0) : def;
    };
    const int both = env("UL_GROUP", -1);
    g_fwd = both >= 0 ? both : env("UL_GROUP_FWD", 1);
    g_bwd = both >= 0 ? both : env("UL_GROUP_BWD", 0);
  }
  // 3xTF32: the split-operand scratch is shared, so every GEMM of the pass
  // stays on one stream (the grouped drivers; small kernels still fork)
  const bool x3 = be == kBackendTf32x3;
  if (fwd && (g_fwd || x3))
    return mlp_forward_n(nets, 2, be, ml, s, p->side, p->ev_fork, p->ev_join);
  DeferredDw own;
  DeferredDw* D = dd ? dd : &own;
  if (!fwd && (g_bwd || x3)) {
    UL_TRY(mlp_backward_n(nets, 2, be, ml, s, p->side, p->ev_fork, p->ev_join, D));
    mark(p, 6, s);
    UL_TRY(run_deferred_dw_gemms(*D, s));
    mark(p, 7, s);
    // the minibatch staging is free once the dW GEMMs have read it: the next
    // step's gather runs beside the reduction and the optimizer
    if (ahead_e >= 0) UL_TRY(gather_ahead(p, ahead_e, ahead_k, s));
    return run_deferred_dw_reduce(*D, s);
  }
  if (!fwd && (ablate_mask() & 128)) {  // (diagnostic: both dX chains on s, no fork / join)
    UL_TRY(mlp_backward_n(nets + 1, 1, be, ml, s, nullptr, nullptr, nullptr, D));
    UL_TRY(mlp_backward_n(nets, 1, be, ml, s, nullptr, nullptr, nullptr, D));
    UL_TRY(run_deferred_dw_gemms(*D, s));
    if (ahead_e >= 0) UL_TRY(gather_ahead(p, ahead_e, ahead_k, s));
    return run_deferred_dw_reduce(*D, s);
  }
  UL_CUDA(cudaEventRecord(p->ev_fork, s));
  UL_CUDA(cudaStreamWaitEvent(p->side, p->ev_fork, 0));
  if (fwd) {
    UL_TRY(mlp_forward_n(nets + 1, 1, be, ml, p->side, nullptr, nullptr, nullptr));
    UL_TRY(mlp_forward_n(nets, 1, be, ml, s, nullptr, nullptr, nullptr));
  } else {
    // bf16: both networks' dW GEMMs are collected and run as one batched
    // launch (+ one reduction) after the two dX chains join
    UL_TRY(mlp_backward_n(nets + 1, 1, be, ml, p->side, nullptr, nullptr, nullptr, D));
    UL_TRY(mlp_backward_n(nets, 1, be, ml, s, nullptr, nullptr, nullptr, D));
  }
  UL_CUDA(cudaEventRecord(p->ev_join, p->side));
  UL_CUDA(cudaStreamWaitEvent(s, p->ev_join, 0));
  if (fwd) return UL_OK;
  mark(p, 6, s);  // (profiling) dX chains of both networks
  UL_TRY(run_deferred_dw_gemms(*D, s));
  mark(p, 7, s);  // the batched dW launch
  if (ahead_e >= 0) UL_TRY(gather_ahead(p, ahead_e, ahead_k, s));
  return run_deferred_dw_reduce(*D, s);
}

void fill_stage_out(const PpoPlan* p, StageOut* so) {
  const NetView* vs[2] = {&p->va, &p->vc};
  float* dst[2] = {p->wst_a, p->wst_c};
  so->dtype = p->dt;
  for (int sg = 0; sg < 2; ++sg) {
    const NetView& v = *vs[sg];
    so->dst[sg] = dst[sg];
    so->nl[sg] = v.n_layers;
    for (int l = 0; l < v.n_layers; ++l) {
      so->w_off[sg][l] = v.w_off[l];
      so->dst_off[sg][l] = p->dt == kBf16 ? v.wb_off[l] : v.wp_off[l];
      so->rows[sg][l] = v.dims[l + 1];
      so->cols[sg][l] = v.dims[l];
      so->ld[sg][l] = (v.dims[l] + (p->dt == kBf16 ? 7 : 3)) / (p->dt == kBf16 ? 8 : 4) *
                      (p->dt == kBf16 ? 8 : 4);
    }
  }
}

// device part of begin: stats reset + advantage statistics + staged weights
// (graph-capturable)
int begin_device(PpoPlan* p, cudaStream_t s) {
  p->gathered_ahead = false;
  if (p->d.gemm_backend >= 1) {
    UL_TRY(stage_weights_dt(p->va, p->b.actor_params, p->wst_a, p->dt, s));
    UL_TRY(stage_weights_dt(p->vc, p->b.critic_params, p->wst_c, p->dt, s));
  }
  UL_CUDA(cudaMemsetAsync(p->st_d, 0, sizeof(ul_ppo_stats), s));
  // critic log_std never receives a gradient (R:algos/ppo.py:119); keep its slot zero
  UL_CUDA(cudaMemsetAsync(p->red + p->Pa + p->vc.logstd_off, 0, sizeof(float), s));
  if (p->d.raw_advantages) return UL_OK;
  return launch_adv_stats(p->b.adv, p->rows, p->adv_part, p->tickets + 1, p->adv_stats, s);
}

// The controller header travels as a kernel parameter, not a memcpy: an H2D
// copy on the compute stream would queue on the copy engine behind the next
// segment's ~190 MB of staging copies and hold the update back until they
// drain.  src (may be dst itself, or null): an update chained behind another
// one without a host round trip keeps that controller's Adam step counters
// and divergence latch (read on the device, in stream order).
struct CtlHeader {
  uint32_t w[offsetof(ul_opt_ctl, part) / sizeof(uint32_t)];
};

__global__ void ctl_load_kernel(ul_opt_ctl* dst, const __grid_constant__ CtlHeader h,
                                const ul_opt_ctl* src) {
  int64_t t0 = 0, t1 = 0;
  int32_t div = 0, fail = 0;
  if (src) {
    t0 = src->t[0];
    t1 = src->t[1];
    div = src->diverged;
    fail = src->fail_step;
  }
  uint32_t* d = reinterpret_cast<uint32_t*>(dst);
  for (int i = 0; i < (int)(sizeof(h.w) / sizeof(uint32_t)); ++i) d[i] = h.w[i];
  if (src) {
    dst->t[0] = t0;
    dst->t[1] = t1;
    dst->diverged = div;
    dst->fail_step = fail;
  }
}

int load_ctl(PpoPlan* p, double lr_a, double lr_c, int64_t t_a, int64_t t_c, const PpoPlan* prev,
             cudaStream_t s) {
  // (built in a host-local record: p->ctl_h may still be receiving an earlier
  // update's collected results)
  const double lr[2] = {lr_a, lr_c};
  static thread_local ul_opt_ctl c;
  UL_TRY(ul_opt_ctl_init(&c, 2, lr, 0.9, 0.999, 1e-8, p->d.max_grad_norm));
  c.t[0] = t_a;
  c.t[1] = t_c;
  CtlHeader h;
  memcpy(&h, &c, sizeof(h));
  ctl_load_kernel<<<1, 1, 0, s>>>(p->ctl_d, h, prev ? prev->ctl_d : nullptr);
  return check_launch("ctl_load_kernel");
}

int upload_ctl(PpoPlan* p, double lr_a, double lr_c, int64_t t_a, int64_t t_c, cudaStream_t s) {
  return load_ctl(p, lr_a, lr_c, t_a, t_c, nullptr, s);
}

int upload_ctl_chained(PpoPlan* p, const PpoPlan* prev, double lr_a, double lr_c,
                       cudaStream_t s) {
  return load_ctl(p, lr_a, lr_c, 0, 0, prev, s);
}

// K4: minibatch (e, k)'s rows of the 7 per-row arrays in one gather launch
int step_gather(PpoPlan* p, int e, int k, cudaStream_t s, bool ahead = false) {
  const ul_ppo_bindings& b = p->b;
  const int64_t ml = p->mb_local;
  const int64_t* idx = p->d.local_shards
                           ? b.perm + (int64_t)e * p->rows + (int64_t)k * ml
                           : b.perm + (int64_t)e * p->rows + (int64_t)k * p->mb + p->d.rank * ml;
  const bool bf = p->dt == kBf16;
  // K4: one gather launch for the 7 per-row arrays; the obs / critic-obs
  // pad column is set to 1.0 (the tensor-core dW's bias column).  Segment
  // rows may be unpadded (ld == width, the H2D landing layout): the ones
  // unit is then read one float past the row (the segment buffers carry a
  // 16-byte tail) and replaced.
  const void* src[7] = {b.obs, b.cobs, b.act, b.blogp, b.adv, b.ret, b.oldv};
  void* dst[7] = {p->mb_obs, p->mb_cobs, p->mb_act, p->mb_scal, p->mb_scal + ml,
                  p->mb_scal + 2 * ml, p->mb_scal + 3 * ml};
  // (bf16 path: the two network inputs are converted to bf16 rows on the way)
  const int64_t xb = bf ? 2 : 4;
  // (bf16 segment rows: already converted, padded and carrying the ones
  // column -- copied as whole 16-byte units, half the bytes of fp32 rows)
  const int64_t sb = p->d.obs_bf16 ? 2 : 4;
  const int64_t sst[7] = {sb * p->d.ld_obs, sb * p->d.ld_cobs, 4 * p->d.ld_act, 4, 4, 4, 4};
  const int64_t dstr[7] = {xb * p->ld_mo, xb * p->ld_mc, 4 * p->ld_ma, 4, 4, 4, 4};
  const int64_t od = p->va.dims[0], cd = p->vc.dims[0];
  const bool ones_o = p->ld_mo > od, ones_c = p->ld_mc > cd;
  // (a padded segment row is read whole -- 16-byte units when it allows;
  // an unpadded one plus the ones unit)
  auto row_b = [](bool ones, int64_t d, int64_t ld, int64_t ldm) {
    return 4 * (!ones ? d : ld > d ? (ld < ldm ? ld : ldm) : d + 1);
  };
  const bool sbf = p->d.obs_bf16 != 0;
  const int64_t rb[7] = {sbf ? 2 * p->ld_mo : row_b(ones_o, od, p->d.ld_obs, p->ld_mo),
                         sbf ? 2 * p->ld_mc : row_b(ones_c, cd, p->d.ld_cobs, p->ld_mc),
                         4 * p->ld_ma, 4, 4, 4, 4};
  const int64_t ones[7] = {ones_o && !sbf ? 4 * od : -1, ones_c && !sbf ? 4 * cd : -1,
                           -1, -1, -1, -1, -1};
  const int cvt[7] = {bf && !sbf ? 1 : 0, bf && !sbf ? 1 : 0, 0, 0, 0, 0, 0};
  // the gather-ahead on the side stream takes at most 2 CTAs per SM, so it
  // steals fewer SMs from the optimizer kernels it overlaps (measured 0.8 %
  // per update; UL_GATHER_AHEAD_BPS overrides)
  static int64_t ahead_cap = -1;
  if (ahead_cap < 0) {
    const char* e2 = getenv("UL_GATHER_AHEAD_BPS");
    ahead_cap = (int64_t)(e2 ? atoi(e2) : 2) * kNumSMs;
  }
  return gather_rows(7, src, dst, sst, dstr, rb, ones, cvt, idx, ml, 0, 0, p->rows, nullptr, s,
                     ahead ? ahead_cap : 0);
}

// After step (e, k)'s backward the minibatch staging is free: gather the next
// step's rows on the side stream, where it runs under this step's optimizer
// kernels (and the all-reduce in data-parallel runs) instead of before the
// next forward.  UL_GATHER_AHEAD=0 disables.
int gather_ahead(PpoPlan* p, int e, int k, cudaStream_t s) {
  static int on = -1;
  if (on < 0) {
    const char* v = getenv("UL_GATHER_AHEAD");
    on = v ? atoi(v) != 0 : 1;
  }
  int ne = e, nk = k + 1;
  if (nk == p->d.minibatches) {
    nk = 0;
    ++ne;
  }
  // (one graph per epoch: the next epoch's permutation is not uploaded yet)
  if (!on || (ablate_mask() & 1) || ne >= p->d.epochs || (p->epoch_mode && ne != e)) return UL_OK;
  if (ablate_mask() & 256) {  // (diagnostic: the gather on s, no fork / join)
    UL_TRY(step_gather(p, ne, nk, s, true));
    p->gathered_ahead = true;
    return UL_OK;
  }
  UL_CUDA(cudaEventRecord(p->ev_gfork, s));
  UL_CUDA(cudaStreamWaitEvent(p->side, p->ev_gfork, 0));
  UL_TRY(step_gather(p, ne, nk, p->side, true));
  UL_CUDA(cudaEventRecord(p->ev_gjoin, p->side));
  p->gathered_ahead = true;
  return UL_OK;
}

// the loss bookkeeping of step (., k) for the prepare tail
LossFinalize loss_finalize_of(const PpoPlan* p, int k) {
  LossFinalize lf{};
  lf.loss = p->red + p->Pa + p->Pc;
  lf.log_std = p->b.actor_params + p->va.logstd_off;
  lf.A = p->A;
  lf.n = (double)p->mb;
  lf.vcoef = p->d.value_loss_coef;
  lf.ecoef = p->d.entropy_coef;
  lf.last_in_epoch = k == p->d.minibatches - 1;
  lf.st = p->st_d;
  return lf;
}

int step_grads(PpoPlan* p, int e, int k, cudaStream_t s) {
  p->prep_folded = false;
  const ul_ppo_bindings& b = p->b;
  const int64_t ml = p->mb_local;
  const bool tc = p->d.gemm_backend >= 1;
  const int64_t od = p->va.dims[0], cd = p->vc.dims[0];
  const bool ones_o = p->ld_mo > od, ones_c = p->ld_mc > cd;
  if (p->gathered_ahead) {  // gathered on the side stream under the previous step
    if (!(ablate_mask() & 256)) UL_CUDA(cudaStreamWaitEvent(s, p->ev_gjoin, 0));
    p->gathered_ahead = false;
  } else if (!(ablate_mask() & 1)) {
    UL_TRY(step_gather(p, e, k, s));
  }
  mark(p, 1, s);
  // K7 forwards of both networks in lockstep: one grouped tensor-core launch
  // per layer, the critic's small kernels on the side stream.  Weights
  // changed at the previous Adam step: the tensor-core path restages them.
  const int be = p->d.gemm_backend;
  // (staged tensor-core weights: written at update begin, then refreshed by
  // every Adam step -- see step_apply)
  MlpNet nets[2] = {};
  nets[0].v = &p->va;
  nets[0].params = b.actor_params;
  nets[0].wp = tc ? p->wst_a : nullptr;
  nets[0].x = p->mb_obs;
  nets[0].ldx = p->ld_mo;
  nets[0].x_has_ones = ones_o;
  nets[0].acts = p->acts_a;
  nets[0].out = p->out_a;
  nets[0].ld_out = p->A;
  nets[0].dout = p->dmean;
  nets[0].ld_dout = p->A;
  nets[0].grads = p->red;
  nets[0].want_dw = true;
  nets[0].zero_logstd = false;  // the head writes the actor's log_std gradient
  nets[0].work = p->work;
  nets[1].v = &p->vc;
  nets[1].params = b.critic_params;
  nets[1].wp = tc ? p->wst_c : nullptr;
  nets[1].x = p->mb_cobs;
  nets[1].ldx = p->ld_mc;
  nets[1].x_has_ones = ones_c;
  nets[1].acts = p->acts_c;
  nets[1].out = p->out_c;
  nets[1].ld_out = 1;
  nets[1].dout = p->dv;
  nets[1].ld_dout = 1;
  nets[1].grads = p->red + p->Pa;
  nets[1].want_dw = true;
  nets[1].zero_logstd = true;  // critic log_std never receives a gradient
  nets[1].work = p->work_c;
  // Fused output stage (bf16, deferred dW): both skinny output layers'
  // forward + backward and the K9 head in one kernel (ppo_fused.cu)
  static int fused_env = -1;
  if (fused_env < 0) {
    const char* e = getenv("UL_FUSED_HEAD");
    fused_env = e ? atoi(e) != 0 : 1;
  }
  const int nla = p->va.n_layers, nlc = p->vc.n_layers;
  const bool fused = fused_env && be == 2 && tc && nla >= 2 && nlc >= 2 && !p->va.ln &&
                     !p->vc.ln && p->vc.dims[nlc] == 1 &&
                     ppo_fused_ok(p->A, p->va.dims[nla - 1], p->vc.dims[nlc - 1]) &&
                     deferred_dw_enabled();
  if (fused) {
    for (int k = 0; k < 2; ++k) {
      const NetView& v = k ? p->vc : p->va;
      nets[k].head_external = true;
      nets[k].dout = bwd_head_dz(v, nets[k].work, ml);
      nets[k].ld_dout = act_ld(v.dims[v.n_layers - 1], p->dt);
      nets[k].head_db_below = head_needs_colsum(nets[k]);
    }
  }
  if (!(ablate_mask() & 8)) UL_TRY(mlp_pass(p, nets, be, ml, s, true));
  mark(p, 0, s);
  if (fused) {
    PpoFusedArgs f{};
    PpoHeadArgs& h = f.h;
    h.n_local = ml;
    h.n_global = (double)p->mb;
    h.A = p->A;
    h.log_std = b.actor_params + p->va.logstd_off;
    h.act = p->mb_act;
    h.ld_act = p->ld_ma;
    h.blogp = p->mb_scal;
    h.adv = p->mb_scal + ml;
    h.ret = p->mb_scal + 2 * ml;
    h.oldv = p->mb_scal + 3 * ml;
    h.adv_stats = p->d.raw_advantages ? nullptr : p->adv_stats;
    h.clip = p->d.clip_param;
    h.vcoef = p->d.value_loss_coef;
    h.clipped_v = p->d.use_clipped_value_loss;
    h.part = p->head_part;
    h.ticket = p->tickets;
    h.dlogstd_out = p->red + p->va.logstd_off;
    h.loss_out = p->red + p->Pa + p->Pc;
    h.ent_coef_add = p->d.rank == 0 ? -p->d.entropy_coef : 0.0;
    const NetView& va = p->va;
    const NetView& vc = p->vc;
    f.Ka = va.dims[nla - 1];
    f.Kc = vc.dims[nlc - 1];
    f.ha = act_ptr(va, p->acts_a, ml, nla - 2, p->dt);
    f.ldha = act_ld(f.Ka, p->dt);
    f.hc = act_ptr(vc, p->acts_c, ml, nlc - 2, p->dt);
    f.ldhc = act_ld(f.Kc, p->dt);
    f.Wa = b.actor_params + va.w_off[nla - 1];
    f.ba = b.actor_params + va.b_off[nla - 1];
    f.wba = reinterpret_cast<const __nv_bfloat16*>(p->wst_a) + va.wb_off[nla - 1];
    f.ldwb = (f.Ka + 7) / 8 * 8;
    f.Wc = b.critic_params + vc.w_off[nlc - 1];
    f.bc = b.critic_params + vc.b_off[nlc - 1];
    f.dha = const_cast<float*>(nets[0].dout);
    f.lddha = nets[0].ld_dout;
    f.dhc = const_cast<float*>(nets[1].dout);
    f.lddhc = nets[1].ld_dout;
    f.csa = nets[0].head_db_below;
    f.csc = nets[1].head_db_below;
    f.parta = bwd_head_part(va, nets[0].work, ml);
    f.plena = ceil_div((int64_t)p->A * f.Ka + p->A + f.Ka, 4) * 4;
    f.gwa = nets[0].grads + va.w_off[nla - 1];
    f.gba = nets[0].grads + va.b_off[nla - 1];
    f.gcsa = f.csa ? nets[0].grads + va.b_off[nla - 2] : nullptr;
    f.partc = bwd_head_part(vc, nets[1].work, ml);
    f.plenc = ceil_div((int64_t)f.Kc + 1 + f.Kc, 4) * 4;
    f.gwc = nets[1].grads + vc.w_off[nlc - 1];
    f.gbc = nets[1].grads + vc.b_off[nlc - 1];
    f.gcsc = f.csc ? nets[1].grads + vc.b_off[nlc - 2] : nullptr;
    f.lossp = reinterpret_cast<float*>(p->head_part);  // (doubles region, ample as floats)
    f.lossld = ceil_div(3 + p->A, 4) * 4;
    DeferredDw dd;
    if (!(ablate_mask() & 4)) UL_TRY(launch_ppo_fused(f, p->dt, dd.jobs, &dd.nj, s));
    mark(p, 2, s);
    // single process: the reduction that writes the final gradients also
    // takes their joint norm / finiteness and runs the prepare tail (every
    // element of both segments is written by it on this path; the critic's
    // log_std slot stays zero)
    SqFold fold{};
    if (p->fold_on && p->d.world_size <= 1) {
      fold.on = 1;
      fold.base = p->red;
      fold.n0 = p->Pa;
      fold.n1 = p->Pc;
      fold.part = p->fold_part;
      fold.bad = p->fold_bad;
      fold.cap = PpoPlan::kFoldCap;
      fold.ticket = p->tickets + 2;
      fold.ctl = p->ctl_d;
      fold.lf = loss_finalize_of(p, k);
      dd.fold = &fold;
    }
    UL_TRY(mlp_pass(p, nets, be, ml, s, false, &dd, e, k));
    p->prep_folded = dd.folded;
    if (fold.on && !dd.folded && getenv("UL_FOLD_DEBUG"))
      fprintf(stderr, "[ul] step (%d, %d): prepare not folded\n", e, k);
    mark(p, 5, s);
    return UL_OK;
  }
  // K9 head
  PpoHeadArgs h{};
  h.n_local = ml;
  h.n_global = (double)p->mb;
  h.A = p->A;
  h.mean = p->out_a;
  h.ld_mean = p->A;
  h.log_std = b.actor_params + p->va.logstd_off;
  h.act = p->mb_act;
  h.ld_act = p->ld_ma;
  h.blogp = p->mb_scal;
  h.adv = p->mb_scal + ml;
  h.ret = p->mb_scal + 2 * ml;
  h.oldv = p->mb_scal + 3 * ml;
  h.v = p->out_c;
  h.ld_v = 1;
  h.adv_stats = p->d.raw_advantages ? nullptr : p->adv_stats;
  h.clip = p->d.clip_param;
  h.vcoef = p->d.value_loss_coef;
  h.clipped_v = p->d.use_clipped_value_loss;
  h.dmean = p->dmean;
  h.ld_dmean = p->A;
  h.dv = p->dv;
  h.part = p->head_part;
  h.ticket = p->tickets;
  h.dlogstd_out = p->red + p->va.logstd_off;
  h.loss_out = p->red + p->Pa + p->Pc;
  h.ent_coef_add = p->d.rank == 0 ? -p->d.entropy_coef : 0.0;
  UL_TRY(launch_ppo_head(h, s));
  mark(p, 2, s);
  // K8 backwards of both networks into the contiguous all-reduce buffer
  UL_TRY(mlp_pass(p, nets, be, ml, s, false));
  mark(p, 5, s);
  return gather_ahead(p, e, k, s);
}

int step_apply(PpoPlan* p, int e, int k, cudaStream_t s) {
  (void)e;
  const ul_ppo_bindings& b = p->b;
  const LossFinalize lf = loss_finalize_of(p, k);
  SegTable st{};
  st.nseg = 2;
  st.g[0] = p->red;
  st.g[1] = p->red + p->Pa;
  st.p[0] = b.actor_params;
  st.p[1] = b.critic_params;
  st.m[0] = b.actor_m;
  st.m[1] = b.critic_m;
  st.v[0] = b.actor_v;
  st.v[1] = b.critic_v;
  st.n[0] = p->Pa;
  st.n[1] = p->Pc;
  // joint clip + loss finalisation, then Adam (which also refreshes the
  // staged tensor-core weights for the next step)
  StageOut so{};
  const bool tc = p->d.gemm_backend >= 1;
  if (tc) fill_stage_out(p, &so);
  // (folded: the step's gradient reduction already ran the prepare tail)
  if (!p->prep_folded) UL_TRY(launch_prepare(st, p->ctl_d, s, &lf));
  p->prep_folded = false;
  if (!(ablate_mask() & 2)) UL_TRY(launch_apply(st, p->ctl_d, 0, 1, s, tc ? &so : nullptr));
  mark(p, 3, s);
  return UL_OK;
}

int all_steps(PpoPlan* p, cudaStream_t s) {
  UL_TRY(begin_device(p, s));
  for (int e = 0; e < p->d.epochs; ++e)
    for (int k = 0; k < p->d.minibatches; ++k) {
      UL_TRY(step_grads(p, e, k, s));
      UL_TRY(step_apply(p, e, k, s));
    }
  return UL_OK;
}

}  // namespace
}  // namespace ul

using ul::PpoPlan;

extern "C" int ul_ppo_plan_create(const ul_ppo_plan_desc* desc, void** plan) {
  UL_CHECK_ARG(desc && plan, "ppo plan: null argument");
  PpoPlan* p = new (std::nothrow) PpoPlan();
  UL_CHECK_ARG(p != nullptr, "ppo plan: out of host memory");
  p->d = *desc;
  {
    const char* e = getenv("UL_FOLD_PREP");  // read per plan (tests compare both)
    p->fold_on = e ? atoi(e) != 0 : true;
  }
  int st = ul::make_view(&desc->actor, &p->va);
  if (st == UL_OK) st = ul::make_view(&desc->critic, &p->vc);
  if (st != UL_OK) {
    delete p;
    return st;
  }
  p->A = p->va.dims[p->va.n_layers];
  p->rows = desc->rows;
  const int ws = desc->world_size < 1 ? 1 : desc->world_size;
  auto fail = [&](const char* msg) {
    ul::set_error("%s", msg);
    delete p;
    return UL_ERR_VALUE;
  };
  if (p->vc.dims[p->vc.n_layers] != 1) return fail("ppo plan: critic output must be 1");
  if (p->A > UL_MAX_ACT) return fail("ppo plan: action dim above UL_MAX_ACT");
  if (desc->minibatches < 1 || desc->epochs < 0) return fail("ppo plan: bad epochs/minibatches");
  if (desc->rows % desc->minibatches != 0) {
    ul::set_error("minibatches %d must divide batch size %lld", desc->minibatches,
                  (long long)desc->rows);
    delete p;
    return UL_ERR_VALUE;
  }
  if (desc->rank < 0 || desc->rank >= ws) return fail("ppo plan: bad rank");
  if (desc->local_shards) {
    p->mb_local = desc->rows / desc->minibatches;
    p->mb = p->mb_local * ws;
  } else {
    p->mb = desc->rows / desc->minibatches;
    if (p->mb % ws != 0) return fail("ppo plan: world_size must divide the minibatch");
    p->mb_local = p->mb / ws;
  }
  if (desc->ld_obs < p->va.dims[0] || desc->ld_cobs < p->vc.dims[0] || desc->ld_act < p->A)
    return fail("ppo plan: leading dimension below feature width");
  if (desc->obs_bf16 && desc->gemm_backend != 2)
    return fail("ppo plan: bf16 observation rows need the bf16 back end");
  if (desc->gemm_backend < 0 || desc->gemm_backend > 3)
    return fail("ppo plan: gemm_backend must be UL_GEMM_FP32, _TF32, _BF16 or _TF32X3");
  p->dt = ul::backend_dtype(desc->gemm_backend);
  if (desc->gemm_backend == ul::kBackendTf32x3) {  // split scratch before any graph capture
    const size_t a = ul::x3_bound(p->va, p->mb_local), c = ul::x3_bound(p->vc, p->mb_local);
    st = ul::x3_reserve(a > c ? a : c);
    if (st != UL_OK) {
      delete p;
      return st;
    }
  }
  // minibatch staging rows: the feature width + the ones column, padded to
  // 16-byte TMA rows (bf16: round_up(d + 1, 8) elements, fp32: round_up(d + 1, 4)),
  // whatever the segment's own row pitch
  {
    const int64_t od = p->va.dims[0], cd = p->vc.dims[0];
    const int64_t q = p->dt == ul::kBf16 ? 8 : 4;
    p->ld_mo = (od + 1 + q - 1) / q * q;
    p->ld_mc = (cd + 1 + q - 1) / q * q;
    if (desc->obs_bf16 && (desc->ld_obs != p->ld_mo || desc->ld_cobs != p->ld_mc))
      return fail("ppo plan: bf16 observation rows must be round_up(d + 1, 8) wide");
  }
  p->ld_ma = desc->ld_act;
  p->Pa = p->va.total;
  p->Pc = p->vc.total;
  st = ul::alloc_plan(p);
  if (st != UL_OK) {
    ul::free_plan(p);
    delete p;
    return st;
  }
  *plan = p;
  return UL_OK;
}

extern "C" int ul_ppo_plan_destroy(void* plan) {
  PpoPlan* p = (PpoPlan*)plan;
  if (!p) return UL_OK;
  ul::free_plan(p);
  delete p;
  return UL_OK;
}

extern "C" int ul_ppo_plan_bind(void* plan, const ul_ppo_bindings* b) {
  PpoPlan* p = (PpoPlan*)plan;
  UL_CHECK_ARG(p && b, "ppo plan: null argument");
  const bool same = p->bound && memcmp(&p->b, b, sizeof(*b)) == 0;
  if (!same)
    for (int e = 0; e < PpoPlan::kMaxEpochGraphs; ++e)
      if (p->egraph[e]) {
        cudaGraphExecDestroy(p->egraph[e]);
        p->egraph[e] = nullptr;
      }
  if (!same && p->graph) {
    cudaGraphExecDestroy(p->graph);
    p->graph = nullptr;
  }
  p->b = *b;
  p->bound = true;
  p->red = b->reduce_buf ? b->reduce_buf : p->red_own;
  return UL_OK;
}

extern "C" int ul_ppo_plan_begin(void* plan, double lr_actor, double lr_critic, int64_t t_actor,
                                 int64_t t_critic, void* stream) {
  PpoPlan* p = (PpoPlan*)plan;
  UL_CHECK_ARG(p && p->bound, "ppo plan: not bound");
  cudaStream_t s = ul::as_stream(stream);
  UL_TRY(ul::upload_ctl(p, lr_actor, lr_critic, t_actor, t_critic, s));
  return ul::begin_device(p, s);
}

// Global advantage statistics across data-parallel ranks that own different
// rows ("local" shards, weak scaling): the begin step leaves this rank's raw
// sums [sum A, sum A^2, n] behind; the caller all-reduces them and finalize
// turns the global sums into the (mean, population std) the loss head reads
// -- normalize_advantages over the union of the ranks' segments
// (R:algos/ppo.py:132-133, :156).
extern "C" int ul_ppo_plan_adv_sums(void* plan, double* dst, void* stream) {
  PpoPlan* p = (PpoPlan*)plan;
  UL_CHECK_ARG(p && dst, "ppo plan: null argument");
  UL_CUDA(cudaMemcpyAsync(dst, p->adv_stats + 2, 3 * sizeof(double), cudaMemcpyDeviceToDevice,
                          ul::as_stream(stream)));
  return UL_OK;
}

extern "C" int ul_ppo_plan_adv_finalize(void* plan, const double* sums, void* stream) {
  PpoPlan* p = (PpoPlan*)plan;
  UL_CHECK_ARG(p && sums, "ppo plan: null argument");
  return ul::launch_adv_finalize(sums, p->adv_stats, ul::as_stream(stream));
}

extern "C" int ul_ppo_plan_step_grads(void* plan, int epoch, int k, void* stream) {
  PpoPlan* p = (PpoPlan*)plan;
  UL_CHECK_ARG(p && p->bound, "ppo plan: not bound");
  UL_CHECK_ARG(epoch >= 0 && epoch < p->d.epochs && k >= 0 && k < p->d.minibatches,
               "ppo plan: step out of range");
  return ul::step_grads(p, epoch, k, ul::as_stream(stream));
}

extern "C" int ul_ppo_plan_step_apply(void* plan, int epoch, int k, void* stream) {
  PpoPlan* p = (PpoPlan*)plan;
  UL_CHECK_ARG(p && p->bound, "ppo plan: not bound");
  return ul::step_apply(p, epoch, k, ul::as_stream(stream));
}

extern "C" int ul_ppo_plan_reduce_buffer(void* plan, float** ptr, int64_t* n) {
  PpoPlan* p = (PpoPlan*)plan;
  UL_CHECK_ARG(p && ptr && n, "ppo plan: null argument");
  *ptr = p->red;
  *n = p->Pa + p->Pc + 3;
  return UL_OK;
}

namespace ul {
namespace {
int run_graph(PpoPlan* p, cudaStream_t s);
}  // namespace
}  // namespace ul

extern "C" int ul_ppo_plan_run(void* plan, double lr_actor, double lr_critic, int64_t t_actor,
                               int64_t t_critic, int use_graph, void* stream) {
  PpoPlan* p = (PpoPlan*)plan;
  UL_CHECK_ARG(p && p->bound, "ppo plan: not bound");
  cudaStream_t s = ul::as_stream(stream);
  UL_TRY(ul::upload_ctl(p, lr_actor, lr_critic, t_actor, t_critic, s));
  if (!use_graph) return ul::all_steps(p, s);
  return ul::run_graph(p, s);
}

// ul_ppo_plan_run (graph) chained behind `prev`'s update on the same stream:
// the Adam step counters and the divergence latch continue from prev's
// controller on the device, so the host may enqueue this update before it
// has read prev's statistics.
extern "C" int ul_ppo_plan_run_after(void* plan, const void* prev, double lr_actor,
                                     double lr_critic, void* stream) {
  PpoPlan* p = (PpoPlan*)plan;
  const PpoPlan* q = (const PpoPlan*)prev;
  UL_CHECK_ARG(p && p->bound && q && q->ctl_d, "ppo plan: not bound / null previous plan");
  cudaStream_t s = ul::as_stream(stream);
  UL_TRY(ul::upload_ctl_chained(p, q, lr_actor, lr_critic, s));
  return ul::run_graph(p, s);
}

// enqueue the D2H of the update's result records behind it (ev_res); the
// next ul_ppo_plan_finish waits on that event instead of the whole stream,
// so later updates may already be queued behind this one
extern "C" int ul_ppo_plan_collect(void* plan, void* stream) {
  PpoPlan* p = (PpoPlan*)plan;
  UL_CHECK_ARG(p && p->bound, "ppo plan: not bound");
  cudaStream_t s = ul::as_stream(stream);
  UL_CUDA(cudaMemcpyAsync(p->ctl_h, p->ctl_d, ul::ctl_header_bytes(), cudaMemcpyDeviceToHost, s));
  UL_CUDA(cudaMemcpyAsync(p->st_h, p->st_d, sizeof(ul_ppo_stats), cudaMemcpyDeviceToHost, s));
  UL_CUDA(cudaEventRecord(p->ev_res, s));
  p->collected = true;
  return UL_OK;
}

namespace ul {
namespace {
int run_graph(PpoPlan* p, cudaStream_t s) {
  // run on the plan's capture stream, ordered after / before the caller's stream
  UL_CUDA(cudaEventRecord(p->ev_in, s));
  UL_CUDA(cudaStreamWaitEvent(p->cap_stream, p->ev_in, 0));
  if (!p->graph) {
    cudaGraph_t g;
    UL_CUDA(cudaStreamBeginCapture(p->cap_stream, cudaStreamCaptureModeThreadLocal));
    int st = ul::all_steps(p, p->cap_stream);
    cudaError_t ce = cudaStreamEndCapture(p->cap_stream, &g);
    if (st != UL_OK) return st;
    UL_CUDA(ce);
    size_t nn = 0;
    cudaGraphGetNodes(g, nullptr, &nn);
    cudaGraphNode_t* nodes = (cudaGraphNode_t*)malloc(sizeof(cudaGraphNode_t) * (nn ? nn : 1));
    cudaGraphGetNodes(g, nodes, &nn);
    p->graph_kernels = 0;
    for (size_t i = 0; i < nn; ++i) {
      cudaGraphNodeType t;
      cudaGraphNodeGetType(nodes[i], &t);
      if (t == cudaGraphNodeTypeKernel) p->graph_kernels++;
    }
    free(nodes);
    ce = cudaGraphInstantiate(&p->graph, g, 0);
    cudaGraphDestroy(g);
    UL_CUDA(ce);
  }
  UL_CUDA(cudaGraphLaunch(p->graph, p->cap_stream));
  UL_CUDA(cudaEventRecord(p->ev_out, p->cap_stream));
  UL_CUDA(cudaStreamWaitEvent(s, p->ev_out, 0));
  return UL_OK;
}
}  // namespace
}  // namespace ul

// One epoch of the update as its own CUDA graph (parity mode with host
// permutations: the caller uploads epoch e's permutation, launches epoch e,
// and draws epoch e + 1's while it runs).  Epoch 0 uploads the controller and
// stages the weights first.
extern "C" int ul_ppo_plan_run_epoch(void* plan, int epoch, double lr_actor, double lr_critic,
                                     int64_t t_actor, int64_t t_critic, void* stream) {
  PpoPlan* p = (PpoPlan*)plan;
  UL_CHECK_ARG(p && p->bound, "ppo plan: not bound");
  UL_CHECK_ARG(epoch >= 0 && epoch < p->d.epochs && epoch < PpoPlan::kMaxEpochGraphs,
               "ppo plan: epoch %d outside [0, %d)", epoch, p->d.epochs);
  cudaStream_t s = ul::as_stream(stream);
  if (epoch == 0) UL_TRY(ul::upload_ctl(p, lr_actor, lr_critic, t_actor, t_critic, s));
  UL_CUDA(cudaEventRecord(p->ev_in, s));
  UL_CUDA(cudaStreamWaitEvent(p->cap_stream, p->ev_in, 0));
  if (!p->egraph[epoch]) {
    cudaGraph_t g;
    p->epoch_mode = true;
    UL_CUDA(cudaStreamBeginCapture(p->cap_stream, cudaStreamCaptureModeThreadLocal));
    int st = epoch == 0 ? ul::begin_device(p, p->cap_stream) : UL_OK;
    for (int k = 0; k < p->d.minibatches && st == UL_OK; ++k) {
      st = ul::step_grads(p, epoch, k, p->cap_stream);
      if (st == UL_OK) st = ul::step_apply(p, epoch, k, p->cap_stream);
    }
    cudaError_t ce = cudaStreamEndCapture(p->cap_stream, &g);
    p->epoch_mode = false;
    if (st != UL_OK) return st;
    UL_CUDA(ce);
    ce = cudaGraphInstantiate(&p->egraph[epoch], g, 0);
    cudaGraphDestroy(g);
    UL_CUDA(ce);
  }
  UL_CUDA(cudaGraphLaunch(p->egraph[epoch], p->cap_stream));
  UL_CUDA(cudaEventRecord(p->ev_out, p->cap_stream));
  UL_CUDA(cudaStreamWaitEvent(s, p->ev_out, 0));
  return UL_OK;
}

extern "C" int ul_ppo_plan_finish(void* plan, ul_ppo_result* out, void* stream) {
  PpoPlan* p = (PpoPlan*)plan;
  UL_CHECK_ARG(p && out, "ppo plan: null argument");
  cudaStream_t s = ul::as_stream(stream);
  if (p->collected) {  // (ul_ppo_plan_collect) only this update's records
    p->collected = false;
    UL_CUDA(cudaEventSynchronize(p->ev_res));
  } else {
    UL_CUDA(cudaMemcpyAsync(p->ctl_h, p->ctl_d, ul::ctl_header_bytes(), cudaMemcpyDeviceToHost, s));
    UL_CUDA(cudaMemcpyAsync(p->st_h, p->st_d, sizeof(ul_ppo_stats), cudaMemcpyDeviceToHost, s));
    UL_CUDA(cudaStreamSynchronize(s));
  }
  const double nb = (double)p->d.epochs * p->d.minibatches;
  const ul_ppo_stats& st = *p->st_h;
  out->policy_loss = nb > 0 ? st.policy_sum / nb : 0.0;
  out->value_loss = nb > 0 ? st.value_sum / nb : 0.0;
  out->entropy = nb > 0 ? st.entropy_sum / nb : 0.0;
  out->kl = p->d.epochs > 0 ? st.kl_epoch_sum / p->d.epochs : 0.0;
  out->grad_norm = p->ctl_h->steps > 0 ? p->ctl_h->norm : 0.0;
  out->t_actor = p->ctl_h->t[0];
  out->t_critic = p->ctl_h->t[1];
  out->diverged = p->ctl_h->diverged;
  out->fail_step = p->ctl_h->fail_step;
  if (out->diverged) {
    ul::set_error("non-finite PPO loss or gradients at step %d", out->fail_step);
    return UL_ERR_DIVERGENCE;
  }
  return UL_OK;
}

extern "C" int ul_ppo_plan_counts(void* plan, int64_t* kernels_per_update,
                                  double* gemm_flops_per_update) {
  PpoPlan* p = (PpoPlan*)plan;
  UL_CHECK_ARG(p && kernels_per_update && gemm_flops_per_update, "ppo plan: null argument");
  *kernels_per_update = p->graph_kernels;
  // algorithmic FLOPs: forward + dW of every layer, dX of every layer but the first
  double f = 0.0;
  for (const ul::NetView* v : {&p->va, &p->vc}) {
    double macs = 0.0, first = (double)v->dims[0] * v->dims[1];
    for (int i = 0; i < v->n_layers; ++i) macs += (double)v->dims[i] * v->dims[i + 1];
    f += 2.0 * (double)p->mb_local * (macs + macs + (macs - first));
  }
  *gemm_flops_per_update = f * p->d.epochs * p->d.minibatches;
  return UL_OK;
}

extern "C" int ul_ppo_plan_profile(void* plan, double lr_actor, double lr_critic, int64_t t_actor,
                                   int64_t t_critic, double* ms, void* stream) {
  PpoPlan* p = (PpoPlan*)plan;
  UL_CHECK_ARG(p && p->bound && ms, "ppo plan: not bound");
  cudaStream_t s = ul::as_stream(stream);
  if (!p->prof) {
    p->prof = new PpoPlan::Prof();
    for (int i = 0; i < PpoPlan::Prof::kMax; ++i) UL_CUDA(cudaEventCreate(&p->prof->ev[i]));
  }
  p->prof->n = 0;
  p->prof->on = true;
  UL_TRY(ul::upload_ctl(p, lr_actor, lr_critic, t_actor, t_critic, s));
  UL_TRY(ul::begin_device(p, s));
  ul::mark(p, 4, s);
  int st = UL_OK;
  for (int e = 0; e < p->d.epochs && st == UL_OK; ++e)
    for (int k = 0; k < p->d.minibatches && st == UL_OK; ++k) {
      st = ul::step_grads(p, e, k, s);
      if (st == UL_OK) st = ul::step_apply(p, e, k, s);
    }
  p->prof->on = false;
  UL_TRY(st);
  UL_CUDA(cudaStreamSynchronize(s));
  for (int c = 0; c < 8; ++c) ms[c] = 0.0;
  for (int i = 1; i < p->prof->n; ++i) {
    float t = 0.f;
    UL_CUDA(cudaEventElapsedTime(&t, p->prof->ev[i - 1], p->prof->ev[i]));
    const int c = p->prof->cat[i];
    if (c >= 0 && c < 4) ms[c] += t;
    if (c >= 5 && c <= 7) {  // MLP backward: counted with the GEMMs, in total and by part
      ms[0] += t;
      ms[5] += t;
      if (c >= 6) ms[c] += t;
    }
    ms[4] += t;
  }
  return UL_OK;
}
