// K10 SAC soft target, K11 SAC critic / actor / alpha heads, and the native
// SAC update plan (FastSAC = reference algo "sac", FlashSAC = "flashsac").
//
// Replaces R:algos/sac.py:35-53 (ScalarAdam), :100-108 (soft_update),
// :111-125 (critic_target), :128-136 (critic_loss_and_grads), :139-178
// (sac_update), :181-221 (actor_loss_and_grads), :224-229
// (alpha_loss_and_grad), :232-249 (_actor_and_alpha_step) and
// R:tensornet/distributions.py:66-84 (squashed sample / log-prob).
// One update, in the reference order:
//   target:  actor fwd(next_obs) -> squash(eps1) -> q1t/q2t fwd -> y (f64)
//   critics: q1, q2 fwd -> MSE head -> q1, q2 bwd -> Adam(q1), Adam(q2)
//   [actor every policy_frequency updates]: actor fwd(obs) -> squash(eps2)
//            -> q1, q2 fwd (UPDATED critics) -> argmin pick -> q1/q2 dX only
//            over the action columns -> actor head -> actor bwd -> Adam(actor)
//            -> alpha ScalarAdam (f64, device)
//   Polyak q1t <- q1, q2t <- q2 (incl. log_std)
// The replay batch arrives as codec rows (obs | action | r | next_obs | term |
// n_used, R:replaypath/storage.py:17-46) gathered straight from the device
// replay ring (K6) into the critic / actor / target input matrices.
#include <cuda_bf16.h>

#include <new>

#include "learner.cuh"

namespace ul {
namespace {

constexpr double kLog2Pi = 1.8378770664093453;

// ---------------------------------------------------------------- kernels
// a = tanh(mean + std*eps) (f32 like the reference), logp = Gaussian(u) -
// sum log1p(-a^2 + 1e-6); a is written into dst[:, col0:col0+A] (a critic
// input matrix, fp32 or bf16 rows) and, optionally, a_out (for the actor
// gradient).
template <typename T>
__global__ void __launch_bounds__(256) squash_kernel(
    const float* __restrict__ mean, int64_t ldm, const float* __restrict__ log_std,
    const float* __restrict__ eps, int64_t lde, int64_t n, int A, T* __restrict__ dst, int64_t ldd,
    int col0, float* __restrict__ a_out, float* __restrict__ logp) {
  // warp per row, lane per action dimension (A <= UL_MAX_ACT = 64: two
  // passes of 32 lanes); the f64 log-prob terms meet in a warp sum
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n; i += nw) {
    double lp = 0.0;
    for (int j = lane; j < A; j += 32) {
      const float ls = log_std[j];
      const float sd = expf(ls);
      const float m = mean[i * ldm + j];
      const float u = __fadd_rn(m, __fmul_rn(sd, eps[i * lde + j]));
      const float a = tanhf(u);
      const double z = ((double)u - (double)m) / (double)sd;
      lp += -(double)ls - 0.5 * kLog2Pi - 0.5 * z * z;
      lp -= log1p(-(double)a * (double)a + 1e-6);
      dst[i * ldd + col0 + j] = (T)a;
      if (a_out) a_out[i * A + j] = a;
    }
    lp = warp_sum(lp);
    if (lane == 0) logp[i] = (float)lp;
  }
}

// Codec rows (obs | act | r | next_obs | term | n_used, R:replaypath/
// storage.py:17-46) -> the plan's network inputs in their GEMM dtype:
// qin = [obs | act | 1], obs = [obs | 1], qa = [obs | (a_pi)], qn =
// [next_obs | (a')] and the fp32 scalars.  One warp per row, lanes across
// the row (one coalesced read of its bytes); idx (may be NULL) addresses the
// ring by absolute index (% modulo), rows outside [lo, hi) are skipped and
// flag *err.
template <typename T>
__global__ void __launch_bounds__(256) sac_load_kernel(
    const float* __restrict__ rows, int64_t pitch, const int64_t* __restrict__ idx,
    int64_t modulo, int64_t lo, int64_t hi, int* err, int64_t B, int D, int A,
    T* __restrict__ qin, int64_t ldq, T* __restrict__ obs, int64_t ldo, T* __restrict__ qa,
    T* __restrict__ qn, float* __restrict__ rew, float* __restrict__ term,
    float* __restrict__ nused) {
  pdl_trigger();
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const T one = (T)1.0f;
  for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < B; r += warps) {
    int64_t slot = r;
    if (idx) {
      const int64_t a = idx[r];
      if (a < lo || a >= hi) {
        if (lane == 0 && err) *err = 1;
        continue;
      }
      slot = modulo > 0 ? a % modulo : a;
    }
    const float* src = rows + slot * pitch;
    T* qi = qin + r * ldq;
    T* ob = obs + r * ldo;
    T* qar = qa + r * ldq;
    T* qnr = qn + r * ldq;
    for (int j = lane; j < D; j += 32) {
      const T o = (T)src[j];
      qi[j] = o;
      ob[j] = o;
      qar[j] = o;
      qnr[j] = (T)src[D + A + 1 + j];
    }
    for (int j = lane; j < A; j += 32) qi[D + j] = (T)src[D + j];
    if (lane == 0) {
      qi[D + A] = one;
      ob[D] = one;
      rew[r] = src[D + A];
      term[r] = src[2 * D + A + 1];
      nused[r] = src[2 * D + A + 2];
    }
  }
}

// y = r + gamma^n_used (1 - term) (min(q1t, q2t) - alpha logp)  (float64)
__global__ void sac_target_kernel(const float* __restrict__ r, const float* __restrict__ term,
                                  const float* __restrict__ nused, const float* __restrict__ q1t,
                                  const float* __restrict__ q2t, const float* __restrict__ logp,
                                  const ul_sac_ctl* __restrict__ ctl, double gamma, int64_t n,
                                  double* __restrict__ y) {
  const double alpha = exp(ctl->log_alpha);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const double keep = term[i] > 0.5f ? 0.0 : 1.0;
    const double soft = fmin((double)q1t[i], (double)q2t[i]) - alpha * (double)logp[i];
    y[i] = (double)r[i] + pow(gamma, (double)(int64_t)nused[i]) * keep * soft;
  }
}

// twin-critic MSE head: dq_k = 2 (q_k - y)/B ; loss_k = mean (q_k - y)^2
__global__ void __launch_bounds__(256) critic_head_kernel(const float* __restrict__ q1,
                                                          const float* __restrict__ q2,
                                                          const double* __restrict__ y, int64_t n,
                                                          double inv_n, float* __restrict__ dq1,
                                                          float* __restrict__ dq2, double* part,
                                                          unsigned int* ticket, ul_sac_ctl* ctl,
                                                          float* loss_slot, double* rec) {
  __shared__ double scratch[32];
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double l1 = 0.0, l2 = 0.0;
  if (i < n) {
    const double e1 = (double)q1[i] - y[i], e2 = (double)q2[i] - y[i];
    l1 = e1 * e1;
    l2 = e2 * e2;
    dq1[i] = (float)(2.0 * e1 * inv_n);
    dq2[i] = (float)(2.0 * e2 * inv_n);
  }
  double r1 = block_sum(l1, scratch);
  double r2 = block_sum(l2, scratch);
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = r1;
    part[2 * blockIdx.x + 1] = r2;
  }
  if (!last_block_ticket(ticket, gridDim.x)) return;
  if (threadIdx.x == 0) {
    double s1 = 0.0, s2 = 0.0;
    for (unsigned b = 0; b < gridDim.x; ++b) {
      s1 += part[2 * b];
      s2 += part[2 * b + 1];
    }
    ctl->critic_loss = s1 * inv_n + s2 * inv_n;
    // data-parallel: this rank's share, all-reduced with the critic gradients
    if (loss_slot) loss_slot[0] = (float)ctl->critic_loss;
    if (rec) {  // per-update statistics of a run: critic loss, alpha before
      rec[0] = ctl->critic_loss;
      rec[3] = exp(ctl->log_alpha);
    }
  }
}

// actor-step pick head: pick = (q1 <= q2), loss = mean(alpha logp - min q)
__global__ void __launch_bounds__(256) pick_head_kernel(const float* __restrict__ q1,
                                                        const float* __restrict__ q2,
                                                        const float* __restrict__ logp, int64_t n,
                                                        double n_global, float* __restrict__ d1,
                                                        float* __restrict__ d2, double* part,
                                                        unsigned int* ticket, ul_sac_ctl* ctl,
                                                        float* slots, double* rec) {
  __shared__ double scratch[32];
  const double alpha = exp(ctl->log_alpha);
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double l = 0.0, lp = 0.0;
  if (i < n) {
    const float a = q1[i], b = q2[i];
    const bool pick = a <= b;
    d1[i] = pick ? 1.f : 0.f;
    d2[i] = pick ? 0.f : 1.f;
    l = alpha * (double)logp[i] - (double)fminf(a, b);
    lp = (double)logp[i];
  }
  double r1 = block_sum(l, scratch);
  double r2 = block_sum(lp, scratch);
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = r1;
    part[2 * blockIdx.x + 1] = r2;
  }
  if (!last_block_ticket(ticket, gridDim.x)) return;
  if (threadIdx.x == 0) {
    double s1 = 0.0, s2 = 0.0;
    for (unsigned b = 0; b < gridDim.x; ++b) {
      s1 += part[2 * b];
      s2 += part[2 * b + 1];
    }
    ctl->actor_loss = s1 / n_global;
    ctl->logp_sum = s2;
    if (rec) rec[1] = ctl->actor_loss;
    if (slots) {  // data-parallel shares, all-reduced with the actor gradients
      slots[0] = (float)ctl->actor_loss;
      slots[1] = (float)s2;
    }
  }
}

// data-parallel: take the all-reduced loss / log-prob sums back into ctl
__global__ void sac_reduced_scalars_kernel(ul_sac_ctl* ctl, const float* cslot,
                                           const float* aslots) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  if (cslot) ctl->critic_loss = (double)cslot[0];
  if (aslots) {
    ctl->actor_loss = (double)aslots[0];
    ctl->logp_sum = (double)aslots[1];
  }
}

// actor gradient head (R:algos/sac.py:207-217): dmean, dlog_std
__global__ void __launch_bounds__(256) actor_head_kernel(
    const float* __restrict__ a, const float* __restrict__ eps, int64_t lde,
    const float* __restrict__ din1, const float* __restrict__ din2, int64_t ldin,
    const float* __restrict__ log_std, int64_t n, double n_global, int A,
    const ul_sac_ctl* __restrict__ ctl, float* __restrict__ dmean, double* part,
    unsigned int* ticket, float* __restrict__ dls_out) {
  __shared__ double scratch[32];
  const double alpha = exp(ctl->log_alpha);
  const double inv_n = 1.0 / n_global;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double* pp = part + (int64_t)blockIdx.x * A;
  for (int j = 0; j < A; ++j) {
    double t = 0.0;
    if (i < n) {
      const double av = (double)a[i * A + j];
      const double oma = 1.0 - av * av;
      const double dlogp_du = 2.0 * av * oma / (oma + 1e-6);
      const double dq = (double)din1[i * ldin + j] + (double)din2[i * ldin + j];
      const double du_dls = exp((double)log_std[j]) * (double)eps[i * lde + j];
      dmean[i * A + j] = (float)((alpha * dlogp_du - dq * oma) * inv_n);
      t = (alpha * (-1.0 + dlogp_du * du_dls) - dq * oma * du_dls) * inv_n;
    }
    const double r = block_sum(t, scratch);
    if (threadIdx.x == 0) pp[j] = r;
  }
  if (!last_block_ticket(ticket, gridDim.x)) return;
  for (int j = threadIdx.x; j < A; j += blockDim.x) {
    double s = 0.0;
    for (unsigned b = 0; b < gridDim.x; ++b) s += part[(int64_t)b * A + j];
    dls_out[j] = (float)s;
  }
}

// ScalarAdam on log_alpha (R:algos/sac.py:35-53, :224-229, :245-249); skipped
// once any step of the run diverged (the reference raised before it)
__global__ void alpha_step_kernel(ul_sac_ctl* ctl, const ul_opt_ctl* oc_a, double n,
                                  double target_entropy, double* rec) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  if (oc_a->diverged || ctl->diverged) return;
  const double excess = ctl->logp_sum / n + target_entropy;
  const double la = ctl->log_alpha;
  ctl->alpha_loss = -la * excess;
  const double g = -excess;
  if (!isfinite(g)) {
    ctl->diverged = 2;
    return;
  }
  ctl->a_t += 1.0;
  const double b1 = 0.9, b2 = 0.999;
  ctl->a_m = b1 * ctl->a_m + (1.0 - b1) * g;
  ctl->a_v = b2 * ctl->a_v + (1.0 - b2) * g * g;
  const double mh = ctl->a_m / (1.0 - pow(b1, ctl->a_t));
  const double vh = ctl->a_v / (1.0 - pow(b2, ctl->a_t));
  ctl->log_alpha = la - ctl->alpha_lr * mh / (sqrt(vh) + 1e-8);
  if (rec) {
    rec[2] = ctl->alpha_loss;
    rec[3] = exp(ctl->log_alpha);
  }
}

// Divergence latch between the phases of a run.  side 1 (after the critic
// Adam steps): a latched critic controller or a non-finite critic loss;
// side 2 (after the actor step): the actor controller or alpha.  The first
// failure is recorded (ctl->diverged = side, fail_update = u) and every
// controller is latched so no later step of the run mutates anything
// (R:algos/sac.py:158-163 / :238-241 raise at that point).
__global__ void sac_latch_kernel(ul_sac_ctl* ctl, ul_opt_ctl* oc_a, ul_opt_ctl* oc_q1,
                                 ul_opt_ctl* oc_q2, int side, int u) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const bool crit = oc_q1->diverged || oc_q2->diverged || !isfinite(ctl->critic_loss);
  const bool act = side == 2 && (oc_a->diverged || ctl->diverged == 2 ||
                                 !isfinite(ctl->actor_loss));
  if (ctl->diverged == 0 && (crit || act)) {
    ctl->diverged = crit ? 1 : 2;
    ctl->fail_update = u;
  }
  if (ctl->diverged) {
    oc_a->diverged = 1;
    oc_q1->diverged = 1;
    oc_q2->diverged = 1;
  }
}

// Polyak of both target critics in one launch (R:algos/sac.py:100-108,
// :176-177): t *= (1 - tau); t += tau * o with two f32 roundings each (the
// numpy order); skipped once the run diverged.
__global__ void polyak2_kernel(float* __restrict__ t1, const float* __restrict__ o1,
                               float* __restrict__ t2, const float* __restrict__ o2, int64_t n4,
                               int64_t n, float keep, float tau,
                               const ul_opt_ctl* __restrict__ guard) {
  pdl_trigger();
  pdl_wait();
  if (guard && guard->diverged) return;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  float4* a4 = reinterpret_cast<float4*>(t1);
  float4* b4 = reinterpret_cast<float4*>(t2);
  const float4* c4 = reinterpret_cast<const float4*>(o1);
  const float4* d4 = reinterpret_cast<const float4*>(o2);
  auto mix = [&](float4 t, float4 o) {
    return make_float4(__fadd_rn(__fmul_rn(t.x, keep), __fmul_rn(tau, o.x)),
                       __fadd_rn(__fmul_rn(t.y, keep), __fmul_rn(tau, o.y)),
                       __fadd_rn(__fmul_rn(t.z, keep), __fmul_rn(tau, o.z)),
                       __fadd_rn(__fmul_rn(t.w, keep), __fmul_rn(tau, o.w)));
  };
  for (int64_t i = i0; i < n4; i += stride) {
    const float4 a = a4[i], b = b4[i], c = __ldg(c4 + i), d = __ldg(d4 + i);
    a4[i] = mix(a, c);
    b4[i] = mix(b, d);
  }
  for (int64_t i = 4 * n4 + i0; i < n; i += stride) {
    t1[i] = __fadd_rn(__fmul_rn(t1[i], keep), __fmul_rn(tau, o1[i]));
    t2[i] = __fadd_rn(__fmul_rn(t2[i], keep), __fmul_rn(tau, o2[i]));
  }
}

// device standard normals (performance mode): Philox4x32-10 + Box-Muller
__device__ __forceinline__ void philox(uint32_t (&c)[4], uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint64_t p0 = (uint64_t)0xD2511F53u * c[0];
    const uint64_t p1 = (uint64_t)0xCD9E8D57u * c[2];
    const uint32_t h0 = (uint32_t)(p0 >> 32), l0 = (uint32_t)p0;
    const uint32_t h1 = (uint32_t)(p1 >> 32), l1 = (uint32_t)p1;
    c[0] = h1 ^ c[1] ^ k0;
    c[1] = l1;
    c[2] = h0 ^ c[3] ^ k1;
    c[3] = l0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
}

__global__ void normal_kernel(float* out, int64_t n, uint64_t key, uint64_t counter) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q * 4 < n; q += stride) {
    uint32_t c[4] = {(uint32_t)q, (uint32_t)(q >> 32), (uint32_t)counter,
                     (uint32_t)(counter >> 32)};
    philox(c, (uint32_t)key, (uint32_t)(key >> 32));
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const float u1 = ((float)c[2 * h] + 1.0f) * 2.3283064e-10f;  // (0, 1]
      const float u2 = (float)c[2 * h + 1] * 2.3283064e-10f;
      const float rr = sqrtf(-2.f * logf(u1));
      float s, co;
      sincospif(2.f * u2, &s, &co);
      const int64_t o = q * 4 + 2 * h;
      if (o < n) out[o] = rr * co;
      if (o + 1 < n) out[o + 1] = rr * s;
    }
  }
}

__global__ void fill_f64_kernel(double* dst, int n, double v) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[i] = v;
}

int fill_f64(double* dst, int n, double v, cudaStream_t s) {
  fill_f64_kernel<<<(n + 127) / 128, 128, 0, s>>>(dst, n, v);
  return check_launch("fill_f64_kernel");
}

int grid_for(int64_t n) {
  int64_t b = ceil_div(n > 0 ? n : 1, 256);
  return (int)(b > 8 * kNumSMs ? 8 * kNumSMs : b);
}

// ------------------------------------------------------------------- plan
struct SacGraph {
  int n = 0;
  uint64_t mask = 0;  // bit u: update u takes the actor step
  cudaGraphExec_t exec = nullptr;
};

struct SacPlan {
  ul_sac_plan_desc d{};
  NetView va{}, vq{};
  int D = 0, A = 0;
  int dt = kF32;  // dtype of the network inputs / activations (bf16 back end: kBf16)
  int64_t B = 0, ldq = 0, ldo = 0, Pa = 0, Pq = 0;
  char* arena = nullptr;
  void *qin = nullptr, *qn = nullptr, *qa = nullptr, *obs = nullptr;
  float *rew = nullptr, *term = nullptr, *nused = nullptr;
  float *acts_a = nullptr, *acts_q1 = nullptr, *acts_q2 = nullptr;
  float *acts_q1t = nullptr, *acts_q2t = nullptr;  // (the 4-network grouped forward)
  float *mean = nullptr, *a_pi = nullptr, *logp = nullptr, *q1o = nullptr, *q2o = nullptr,
        *q1t = nullptr, *q2t = nullptr, *dq1 = nullptr, *dq2 = nullptr, *din1 = nullptr,
        *din2 = nullptr, *dmean = nullptr;
  double* y = nullptr;
  float *g_a = nullptr, *g_q1 = nullptr, *g_q2 = nullptr, *work = nullptr;
  float* work2 = nullptr;  // q2's backward workspace (the twin critics run grouped)
  float *gq_own = nullptr, *ga_own = nullptr;  // plan-owned reduce buffers
  int world = 1;
  double n_global = 0.0;
  float *ws_a = nullptr, *ws_q1 = nullptr, *ws_q2 = nullptr, *ws_q1t = nullptr, *ws_q2t = nullptr;
  // per-update noise [n_cap][2][B][A] and statistics [n_cap][4]
  int n_cap = 0;
  float* eps = nullptr;
  double* stats = nullptr;
  int u = 0;  // update index of the phase being issued (noise / stats slot)
  double* part = nullptr;
  unsigned int* tickets = nullptr;
  ul_opt_ctl *oc_a = nullptr, *oc_q1 = nullptr, *oc_q2 = nullptr;
  ul_opt_ctl* oc_h = nullptr;  // pinned staging, 3 records (actor, q1, q2)
  ul_sac_ctl* ctl = nullptr;
  ul_sac_ctl* ctl_h = nullptr;
  ul_sac_bindings b{};
  bool bound = false;
  cudaStream_t cap = nullptr;  // capture / replay stream of the run graphs
  cudaEvent_t ev_in = nullptr, ev_out = nullptr;
  static constexpr int kMaxGraphs = 16;
  SacGraph graphs[kMaxGraphs];
  int n_graphs = 0;
};

// The twin critics as ONE grouped pass (one tcgen05 launch per layer for
// both networks, one batched dW launch): x rows shared, per-network params,
// staged weights, activation caches, outputs.  UL_SAC_GROUP=0: one network
// at a time; 2 (default 1): the target critics' and the online critics'
// forwards as one 4-network pass (own activation caches for the targets)
int sac_group() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("UL_SAC_GROUP");
    on = e ? atoi(e) : 1;
  }
  return on;
}

int alloc_sac(SacPlan* p) {
  size_t off = 0;
  auto carve = [&](size_t bytes) {
    size_t o = off;
    off += (bytes + 255) & ~size_t(255);
    return o;
  };
  const int64_t B = p->B;
  const int64_t wa = bwd_work_floats(p->va, B), wq = bwd_work_floats(p->vq, B);
  // input matrices sized for fp32 rows (bf16 rows are narrower)
  const int64_t ldq32 = act_ld(p->D + p->A), ldo32 = act_ld(p->D);
  size_t o[42];
  int k = 0;
  o[k++] = carve(4 * B * ldq32);                  // 0 qin
  o[k++] = carve(4 * B * ldq32);                  // 1 qn
  o[k++] = carve(4 * B * ldq32);                  // 2 qa
  o[k++] = carve(4 * B * ldo32);                  // 3 obs
  o[k++] = carve(4 * B);                          // 4 rew
  o[k++] = carve(4 * B);                          // 5 term
  o[k++] = carve(4 * B);                          // 6 nused
  o[k++] = carve(4 * act_floats(p->va, B));       // 7
  o[k++] = carve(4 * act_floats(p->vq, B));       // 8
  o[k++] = carve(4 * act_floats(p->vq, B));       // 9
  o[k++] = carve(4 * B * p->A);                   // 10 mean
  o[k++] = carve(4 * B * p->A);                   // 11 a_pi
  o[k++] = carve(4 * B);                          // 12 logp
  o[k++] = carve(4 * B);                          // 13 q1o
  o[k++] = carve(4 * B);                          // 14 q2o
  o[k++] = carve(4 * B);                          // 15 q1t
  o[k++] = carve(4 * B);                          // 16 q2t
  o[k++] = carve(4 * B);                          // 17 dq1
  o[k++] = carve(4 * B);                          // 18 dq2
  o[k++] = carve(4 * B * p->A);                   // 19 din1
  o[k++] = carve(4 * B * p->A);                   // 20 din2
  o[k++] = carve(4 * B * p->A);                   // 21 dmean
  o[k++] = carve(8 * B);                          // 22 y
  o[k++] = carve(4 * (p->Pa + 8));                // 23 g_a | actor slots
  o[k++] = carve(4 * (2 * p->Pq + 8));            // 24 g_q1 | g_q2 | critic slot
  o[k++] = carve(4 * wq);                         // 25 work2 (q2's backward)
  o[k++] = carve(4 * (wa > wq ? wa : wq));        // 26 work
  o[k++] = carve(4 * p->va.wp_total);             // 27
  o[k++] = carve(4 * p->vq.wp_total);             // 28
  o[k++] = carve(4 * p->vq.wp_total);             // 29
  o[k++] = carve(4 * p->vq.wp_total);             // 30
  o[k++] = carve(4 * p->vq.wp_total);             // 31
  o[k++] = carve(8);                              // 32 (noise: ul_sac_plan_reserve)
  o[k++] = carve(8 * (ceil_div(B, 256) * (UL_MAX_ACT + 2) + 64));  // 33 part
  o[k++] = carve(4 * 16);                         // 34 tickets
  o[k++] = carve(sizeof(ul_opt_ctl));             // 35
  o[k++] = carve(sizeof(ul_opt_ctl));             // 36
  o[k++] = carve(sizeof(ul_opt_ctl));             // 37
  o[k++] = carve(sizeof(ul_sac_ctl));             // 38
  const bool four = sac_group() >= 2;
  o[k++] = carve(four ? 4 * act_floats(p->vq, B) : 0);  // 39 acts_q1t
  o[k++] = carve(four ? 4 * act_floats(p->vq, B) : 0);  // 40 acts_q2t
  UL_CUDA(cudaMalloc(&p->arena, off));
  UL_CUDA(cudaMemset(p->arena, 0, off));
  char* a = p->arena;
  p->qin = a + o[0];
  p->qn = a + o[1];
  p->qa = a + o[2];
  p->obs = a + o[3];
  float** fp[] = {&p->rew, &p->term, &p->nused, &p->acts_a, &p->acts_q1, &p->acts_q2, &p->mean,
                  &p->a_pi, &p->logp, &p->q1o, &p->q2o, &p->q1t, &p->q2t, &p->dq1, &p->dq2,
                  &p->din1, &p->din2, &p->dmean};
  for (int i = 0; i < 18; ++i) *fp[i] = (float*)(a + o[4 + i]);
  p->y = (double*)(a + o[22]);
  p->ga_own = (float*)(a + o[23]);
  p->gq_own = (float*)(a + o[24]);
  p->g_a = p->ga_own;
  p->g_q1 = p->gq_own;
  p->g_q2 = p->gq_own + p->Pq;
  p->work = (float*)(a + o[26]);
  p->work2 = (float*)(a + o[25]);
  p->ws_a = (float*)(a + o[27]);
  p->ws_q1 = (float*)(a + o[28]);
  p->ws_q2 = (float*)(a + o[29]);
  p->ws_q1t = (float*)(a + o[30]);
  p->ws_q2t = (float*)(a + o[31]);
  p->part = (double*)(a + o[33]);
  p->tickets = (unsigned int*)(a + o[34]);
  p->oc_a = (ul_opt_ctl*)(a + o[35]);
  p->oc_q1 = (ul_opt_ctl*)(a + o[36]);
  p->oc_q2 = (ul_opt_ctl*)(a + o[37]);
  p->ctl = (ul_sac_ctl*)(a + o[38]);
  p->acts_q1t = four ? (float*)(a + o[39]) : nullptr;
  p->acts_q2t = four ? (float*)(a + o[40]) : nullptr;
  UL_CUDA(cudaHostAlloc(&p->oc_h, 3 * sizeof(ul_opt_ctl), cudaHostAllocPortable));
  UL_CUDA(cudaHostAlloc(&p->ctl_h, sizeof(ul_sac_ctl), cudaHostAllocPortable));
  UL_CUDA(cudaStreamCreateWithFlags(&p->cap, cudaStreamNonBlocking));
  UL_CUDA(cudaEventCreateWithFlags(&p->ev_in, cudaEventDisableTiming));
  UL_CUDA(cudaEventCreateWithFlags(&p->ev_out, cudaEventDisableTiming));
  return UL_OK;
}

void drop_graphs(SacPlan* p) {
  for (int i = 0; i < p->n_graphs; ++i)
    if (p->graphs[i].exec) cudaGraphExecDestroy(p->graphs[i].exec);
  p->n_graphs = 0;
}

void free_sac(SacPlan* p) {
  drop_graphs(p);
  if (p->arena) cudaFree(p->arena);
  if (p->eps) cudaFree(p->eps);
  if (p->stats) cudaFree(p->stats);
  if (p->oc_h) cudaFreeHost(p->oc_h);
  if (p->ctl_h) cudaFreeHost(p->ctl_h);
  if (p->cap) cudaStreamDestroy(p->cap);
  if (p->ev_in) cudaEventDestroy(p->ev_in);
  if (p->ev_out) cudaEventDestroy(p->ev_out);
}

size_t ctl_hdr() { return offsetof(ul_opt_ctl, part); }


int critics_forward(const SacPlan* p, int be, const float* x, const float* w1, const float* ws1,
                    float* out1, const float* w2, const float* ws2, float* out2, cudaStream_t s) {
  if (!sac_group()) {
    UL_TRY(mlp_forward(p->vq, w1, ws1, be, x, p->ldq, p->B, p->acts_q1, out1, 1, s));
    return mlp_forward(p->vq, w2, ws2, be, x, p->ldq, p->B, p->acts_q2, out2, 1, s);
  }
  MlpNet n[2] = {};
  for (int k = 0; k < 2; ++k) {
    n[k].v = &p->vq;
    n[k].params = k ? w2 : w1;
    n[k].wp = be >= 1 ? (k ? ws2 : ws1) : nullptr;
    n[k].x = x;
    n[k].ldx = p->ldq;
    n[k].acts = k ? p->acts_q2 : p->acts_q1;
    n[k].out = k ? out2 : out1;
    n[k].ld_out = 1;
  }
  return mlp_forward_n(n, 2, be, p->B, s, nullptr, nullptr, nullptr);
}

// target critics on the next rows (xt) and online critics on the current
// rows (x) as one 4-network lockstep pass (UL_SAC_GROUP=2)
int critics_forward4(const SacPlan* p, int be, const float* xt, const float* x,
                     cudaStream_t s) {
  const ul_sac_bindings& b = p->b;
  const float* w[4] = {b.q1t, b.q2t, b.q1, b.q2};
  const float* ws[4] = {p->ws_q1t, p->ws_q2t, p->ws_q1, p->ws_q2};
  float* acts[4] = {p->acts_q1t, p->acts_q2t, p->acts_q1, p->acts_q2};
  float* out[4] = {p->q1t, p->q2t, p->q1o, p->q2o};
  MlpNet n[4] = {};
  for (int k = 0; k < 4; ++k) {
    n[k].v = &p->vq;
    n[k].params = w[k];
    n[k].wp = be >= 1 ? ws[k] : nullptr;
    n[k].x = k < 2 ? xt : x;
    n[k].ldx = p->ldq;
    n[k].acts = acts[k];
    n[k].out = out[k];
    n[k].ld_out = 1;
  }
  return mlp_forward_n(n, 4, be, p->B, s, nullptr, nullptr, nullptr);
}

// backward of both online critics from dq1 / dq2: parameter gradients
// (grads1/2, want_dw) or the input gradient over columns [dx_col0, + dx_ncols)
int critics_backward(const SacPlan* p, int be, const float* x, bool x_has_ones, bool want_dw,
                     float* grads1, float* grads2, float* din1, float* din2, int dx_col0,
                     int dx_ncols, bool zero_logstd, cudaStream_t s) {
  const ul_sac_bindings& b = p->b;
  if (!sac_group()) {
    UL_TRY(mlp_backward(p->vq, b.q1, p->ws_q1, be, x, p->ldq, x_has_ones, p->B, p->acts_q1,
                        p->dq1, 1, grads1, din1, din1 ? p->A : 0, dx_col0, dx_ncols, want_dw,
                        zero_logstd, p->work, s));
    return mlp_backward(p->vq, b.q2, p->ws_q2, be, x, p->ldq, x_has_ones, p->B, p->acts_q2,
                        p->dq2, 1, grads2, din2, din2 ? p->A : 0, dx_col0, dx_ncols, want_dw,
                        zero_logstd, p->work, s);
  }
  MlpNet n[2] = {};
  for (int k = 0; k < 2; ++k) {
    n[k].v = &p->vq;
    n[k].params = k ? b.q2 : b.q1;
    n[k].wp = be >= 1 ? (k ? p->ws_q2 : p->ws_q1) : nullptr;
    n[k].x = x;
    n[k].ldx = p->ldq;
    n[k].x_has_ones = x_has_ones;
    n[k].acts = k ? p->acts_q2 : p->acts_q1;
    n[k].dout = k ? p->dq2 : p->dq1;
    n[k].ld_dout = 1;
    n[k].grads = k ? grads2 : grads1;
    n[k].dx = k ? din2 : din1;
    n[k].lddx = (k ? din2 : din1) ? p->A : 0;
    n[k].dx_col0 = dx_col0;
    n[k].dx_ncols = dx_ncols;
    n[k].want_dw = want_dw;
    n[k].zero_logstd = zero_logstd;
    n[k].work = k ? p->work2 : p->work;
  }
  return mlp_backward_n(n, 2, be, p->B, s, nullptr, nullptr, nullptr, nullptr);
}

int adam_one(float* params, float* grads, float* m, float* v, int64_t n, ul_opt_ctl* oc,
             cudaStream_t s) {
  SegTable st{};
  st.nseg = 1;
  st.g[0] = grads;
  st.p[0] = params;
  st.m[0] = m;
  st.v[0] = v;
  st.n[0] = n;
  UL_TRY(launch_prepare(st, oc, s));
  return launch_apply(st, oc, 0, 1, s);
}

int launch_squash(SacPlan* p, const float* eps, void* dst, float* a_out, cudaStream_t s) {
  const float* ls = p->b.actor + p->va.logstd_off;
  const int64_t B = p->B;
  int64_t blocks = ceil_div(B, 8);  // 8 rows (warps) per block
  blocks = blocks > 16 * kNumSMs ? 16 * kNumSMs : blocks;
  if (p->dt == kBf16)
    squash_kernel<__nv_bfloat16><<<(unsigned)blocks, 256, 0, s>>>(
        p->mean, p->A, ls, eps, p->A, B, p->A, (__nv_bfloat16*)dst, p->ldq, p->D, a_out, p->logp);
  else
    squash_kernel<float><<<(unsigned)blocks, 256, 0, s>>>(p->mean, p->A, ls, eps, p->A, B, p->A,
                                                          (float*)dst, p->ldq, p->D, a_out,
                                                          p->logp);
  return check_launch("squash_kernel");
}

double* rec_of(SacPlan* p) { return p->stats ? p->stats + 4 * (int64_t)p->u : nullptr; }
const float* eps_of(SacPlan* p, int which) {
  return p->eps + ((int64_t)p->u * 2 + which) * p->B * p->A;
}

}  // namespace
}  // namespace ul

using ul::SacPlan;

extern "C" int ul_sac_plan_create(const ul_sac_plan_desc* desc, void** plan) {
  UL_CHECK_ARG(desc && plan, "sac plan: null argument");
  SacPlan* p = new (std::nothrow) SacPlan();
  UL_CHECK_ARG(p, "sac plan: out of host memory");
  p->d = *desc;
  int st = ul::make_view(&desc->actor, &p->va);
  if (st == UL_OK) st = ul::make_view(&desc->critic, &p->vq);
  if (st != UL_OK) {
    delete p;
    return st;
  }
  p->D = desc->obs_dim;
  p->A = desc->act_dim;
  p->B = desc->batch;
  auto fail = [&](const char* m) {
    ul::set_error("%s", m);
    delete p;
    return UL_ERR_VALUE;
  };
  if (p->B < 2) return fail("sac_update needs a batch of at least 2 rows");
  if (p->va.dims[0] != p->D || p->va.dims[p->va.n_layers] != p->A)
    return fail("sac plan: actor dims do not match obs/act");
  if (p->vq.dims[0] != p->D + p->A || p->vq.dims[p->vq.n_layers] != 1)
    return fail("sac plan: critic must map obs+act -> 1");
  if (p->A > UL_MAX_ACT) return fail("sac plan: action dim above UL_MAX_ACT");
  if (desc->gemm_backend < 0 || desc->gemm_backend > 3)
    return fail("sac plan: gemm_backend must be 0 (fp32), 1 (tf32), 2 (bf16) or 3 (3xTF32)");
  if (desc->gemm_backend == ul::kBackendTf32x3) {
    const size_t a = ul::x3_bound(p->va, p->B), q = ul::x3_bound(p->vq, p->B);
    if (ul::x3_reserve(a > q ? a : q) != UL_OK) {
      delete p;
      return UL_ERR_CUDA;
    }
  }
  p->dt = ul::backend_dtype(desc->gemm_backend);
  p->ldq = ul::act_ld(p->D + p->A, p->dt);
  p->ldo = ul::act_ld(p->D, p->dt);
  p->world = desc->world_size > 1 ? desc->world_size : 1;
  p->n_global = (double)p->B * p->world;
  p->Pa = p->va.total;
  p->Pq = p->vq.total;
  st = ul::alloc_sac(p);
  if (st == UL_OK) st = ul_sac_plan_reserve(p, 1);
  if (st != UL_OK) {
    ul::free_sac(p);
    delete p;
    return st;
  }
  *plan = p;
  return UL_OK;
}

extern "C" int ul_sac_plan_destroy(void* plan) {
  SacPlan* p = (SacPlan*)plan;
  if (!p) return UL_OK;
  ul::free_sac(p);
  delete p;
  return UL_OK;
}

extern "C" int ul_sac_plan_reserve(void* plan, int n_updates) {
  SacPlan* p = (SacPlan*)plan;
  UL_CHECK_ARG(p && n_updates >= 1 && n_updates <= 64, "sac plan: reserve 1..64 updates");
  if (n_updates <= p->n_cap) return UL_OK;
  UL_CUDA(cudaDeviceSynchronize());  // the old buffers may still be read
  ul::drop_graphs(p);                // (graphs hold the old pointers)
  if (p->eps) cudaFree(p->eps);
  if (p->stats) cudaFree(p->stats);
  p->eps = nullptr;
  p->stats = nullptr;
  UL_CUDA(cudaMalloc(&p->eps, sizeof(float) * 2 * (size_t)n_updates * p->B * p->A));
  UL_CUDA(cudaMemset(p->eps, 0, sizeof(float) * 2 * (size_t)n_updates * p->B * p->A));
  UL_CUDA(cudaMalloc(&p->stats, sizeof(double) * 4 * (size_t)n_updates));
  p->n_cap = n_updates;
  return UL_OK;
}

extern "C" int ul_sac_plan_bind(void* plan, const ul_sac_bindings* b) {
  SacPlan* p = (SacPlan*)plan;
  UL_CHECK_ARG(p && b, "sac plan: null argument");
  const bool same = p->bound && memcmp(&p->b, b, sizeof(*b)) == 0;
  if (!same) ul::drop_graphs(p);  // graphs bake the parameter pointers
  p->b = *b;
  p->bound = true;
  float* gq = b->critic_red ? b->critic_red : p->gq_own;
  p->g_q1 = gq;
  p->g_q2 = gq + p->Pq;
  p->g_a = b->actor_red ? b->actor_red : p->ga_own;
  return UL_OK;
}

// Load a batch of codec rows (obs | act | r | next_obs | term | n_used):
// rows[idx[i] % modulo] for device ring rows (idx may be NULL for rows
// 0..B-1), written in the back end's input dtype by one kernel.
extern "C" int ul_sac_plan_load_rows(void* plan, const float* rows, int64_t pitch,
                                     const int64_t* idx, int64_t modulo, int64_t lo, int64_t hi,
                                     int* err, void* stream) {
  SacPlan* p = (SacPlan*)plan;
  UL_CHECK_ARG(p, "sac plan: null");
  const int64_t width = 2 * (int64_t)p->D + p->A + 3;
  UL_CHECK_ARG(pitch >= width, "sac plan: row pitch below codec width");
  cudaStream_t s = ul::as_stream(stream);
  int64_t blocks = ul::ceil_div(p->B, 8);
  blocks = blocks > 8 * ul::kNumSMs ? 8 * ul::kNumSMs : blocks;
  if (p->dt == ul::kBf16) {
    using T = __nv_bfloat16;
    return ul::launch_pdl("sac_load_kernel", ul::sac_load_kernel<T>, dim3((unsigned)blocks),
                          dim3(256), 0, s, rows, pitch, idx, modulo, lo, hi, err, p->B, p->D,
                          p->A, (T*)p->qin, p->ldq, (T*)p->obs, p->ldo, (T*)p->qa, (T*)p->qn,
                          p->rew, p->term, p->nused);
  }
  return ul::launch_pdl("sac_load_kernel", ul::sac_load_kernel<float>, dim3((unsigned)blocks),
                        dim3(256), 0, s, rows, pitch, idx, modulo, lo, hi, err, p->B, p->D, p->A,
                        (float*)p->qin, p->ldq, (float*)p->obs, p->ldo, (float*)p->qa,
                        (float*)p->qn, p->rew, p->term, p->nused);
}

// Upload the optimizer / alpha control state (host values -> device):
// asynchronous, one pinned staging record each (the previous finish synced).
extern "C" int ul_sac_plan_begin(void* plan, const ul_sac_ctl* host_ctl, const double* lrs,
                                 const int64_t* ts, void* stream) {
  SacPlan* p = (SacPlan*)plan;
  UL_CHECK_ARG(p && p->bound && host_ctl && lrs && ts, "sac plan: not bound");
  cudaStream_t s = ul::as_stream(stream);
  *p->ctl_h = *host_ctl;
  p->ctl_h->diverged = 0;
  p->ctl_h->fail_update = -1;
  UL_CUDA(cudaMemcpyAsync(p->ctl, p->ctl_h, sizeof(ul_sac_ctl), cudaMemcpyHostToDevice, s));
  ul_opt_ctl* dst[3] = {p->oc_a, p->oc_q1, p->oc_q2};
  for (int k = 0; k < 3; ++k) {
    const double lr = lrs[k];
    UL_TRY(ul_opt_ctl_init(p->oc_h + k, 1, &lr, 0.9, 0.999, 1e-8, p->d.max_grad_norm));
    p->oc_h[k].t[0] = ts[k];
    UL_CUDA(cudaMemcpyAsync(dst[k], p->oc_h + k, ul::ctl_hdr(), cudaMemcpyHostToDevice, s));
  }
  return UL_OK;
}

// Fill the whole reserved noise buffer [n_cap][2][B][A] on the device
// (performance mode).
extern "C" int ul_sac_plan_device_noise(void* plan, uint64_t key, uint64_t counter,
                                        void* stream) {
  SacPlan* p = (SacPlan*)plan;
  UL_CHECK_ARG(p, "sac plan: null");
  const int64_t n = 2 * (int64_t)p->n_cap * p->B * p->A;
  ul::normal_kernel<<<ul::grid_for(ul::ceil_div(n, 4)), 256, 0, ul::as_stream(stream)>>>(
      p->eps, n, key, counter);
  return ul::check_launch("normal_kernel");
}

extern "C" int ul_sac_plan_noise_ptr(void* plan, float** eps) {
  SacPlan* p = (SacPlan*)plan;
  UL_CHECK_ARG(p && eps, "sac plan: null");
  *eps = p->eps;
  return UL_OK;
}

namespace ul {
namespace {

int stage_critics(SacPlan* p, cudaStream_t s) {
  const NetView* v[2] = {&p->vq, &p->vq};
  const float* src[2] = {p->b.q1, p->b.q2};
  void* dst[2] = {p->ws_q1, p->ws_q2};
  return stage_weights_multi(2, v, src, dst, backend_dtype(p->d.gemm_backend), s);
}

// phase 1: staged weights, soft target, critic forwards + MSE head + critic
// backwards into [g_q1 | g_q2 | loss share]
int sac_critic_grads(SacPlan* p, cudaStream_t s) {
  const ul_sac_bindings& b = p->b;
  const int be = p->d.gemm_backend;
  const int64_t B = p->B, A = p->A;
  const float* qin = (const float*)p->qin;  // (rows of the back end's dtype)
  const float* qn = (const float*)p->qn;
  if (be != 0) {  // tensor-core back ends read 16-B-row staged (tf32 / bf16) weights:
    // all five networks in one launch
    const NetView* v[5] = {&p->va, &p->vq, &p->vq, &p->vq, &p->vq};
    const float* src[5] = {b.actor, b.q1, b.q2, b.q1t, b.q2t};
    void* dst[5] = {p->ws_a, p->ws_q1, p->ws_q2, p->ws_q1t, p->ws_q2t};
    UL_TRY(stage_weights_multi(5, v, src, dst, backend_dtype(be), s));
  }
  // ---- K10 target (next_obs rows of qn, actions a' written by the squash)
  UL_TRY(mlp_forward(p->va, b.actor, p->ws_a, be, qn, p->ldq, B, p->acts_a, p->mean, A, s));
  UL_TRY(launch_squash(p, eps_of(p, 0), p->qn, nullptr, s));
  const bool four = p->acts_q1t != nullptr;
  if (four)
    UL_TRY(critics_forward4(p, be, qn, qin, s));
  else
    UL_TRY(critics_forward(p, be, qn, b.q1t, p->ws_q1t, p->q1t, b.q2t, p->ws_q2t, p->q2t, s));
  sac_target_kernel<<<grid_for(B), 256, 0, s>>>(p->rew, p->term, p->nused, p->q1t, p->q2t,
                                               p->logp, p->ctl, p->d.gamma, B, p->y);
  UL_TRY(check_launch("sac_target_kernel"));
  // ---- K11 critics (ones column of qin at D+A feeds the tensor-core db)
  if (!four)
    UL_TRY(critics_forward(p, be, qin, b.q1, p->ws_q1, p->q1o, b.q2, p->ws_q2, p->q2o, s));
  const unsigned nb = (unsigned)ceil_div(B, 256);
  critic_head_kernel<<<nb, 256, 0, s>>>(p->q1o, p->q2o, p->y, B, 1.0 / p->n_global, p->dq1,
                                        p->dq2, p->part, p->tickets, p->ctl,
                                        p->world > 1 ? p->g_q1 + 2 * p->Pq : nullptr, rec_of(p));
  UL_TRY(check_launch("critic_head_kernel"));
  return critics_backward(p, be, qin, true, true, p->g_q1, p->g_q2, nullptr, nullptr, 0, 0, true,
                          s);
}

// phase 2: (reduced loss back into ctl) Adam(q1), Adam(q2), latch
int sac_critic_apply(SacPlan* p, cudaStream_t s) {
  const ul_sac_bindings& b = p->b;
  if (p->world > 1) {
    sac_reduced_scalars_kernel<<<1, 32, 0, s>>>(p->ctl, p->g_q1 + 2 * p->Pq, nullptr);
    UL_TRY(check_launch("sac_reduced_scalars_kernel"));
  }
  UL_TRY(adam_one(b.q1, p->g_q1, b.q1_m, b.q1_v, p->Pq, p->oc_q1, s));
  UL_TRY(adam_one(b.q2, p->g_q2, b.q2_m, b.q2_v, p->Pq, p->oc_q2, s));
  sac_latch_kernel<<<1, 32, 0, s>>>(p->ctl, p->oc_a, p->oc_q1, p->oc_q2, 1, p->u);
  return check_launch("sac_latch_kernel");
}

// phase 3 (actor steps): actor fwd -> squash(eps2) -> UPDATED critics fwd ->
// argmin pick -> critic dX over the action columns -> actor head -> actor
// backward into [g_a | loss share | sum log pi]
int sac_actor_grads(SacPlan* p, cudaStream_t s) {
  const ul_sac_bindings& b = p->b;
  const int be = p->d.gemm_backend;
  const int64_t B = p->B, D = p->D, A = p->A;
  const float* ls = b.actor + p->va.logstd_off;
  const float* qa = (const float*)p->qa;
  const float* obs = (const float*)p->obs;
  if (be != 0) UL_TRY(stage_critics(p, s));  // the critics just took their Adam step
  const float* eps2 = eps_of(p, 1);
  UL_TRY(mlp_forward(p->va, b.actor, p->ws_a, be, obs, p->ldo, B, p->acts_a, p->mean, A, s));
  UL_TRY(launch_squash(p, eps2, p->qa, p->a_pi, s));
  UL_TRY(critics_forward(p, be, qa, b.q1, p->ws_q1, p->q1o, b.q2, p->ws_q2, p->q2o, s));
  const unsigned nb = (unsigned)ceil_div(B, 256);
  pick_head_kernel<<<nb, 256, 0, s>>>(p->q1o, p->q2o, p->logp, B, p->n_global, p->dq1, p->dq2,
                                      p->part, p->tickets + 1, p->ctl,
                                      p->world > 1 ? p->g_a + p->Pa : nullptr, rec_of(p));
  UL_TRY(check_launch("pick_head_kernel"));
  // dQ/da through each critic's input gradient, action columns only (fp32 out)
  UL_TRY(critics_backward(p, be, qa, false, false, nullptr, nullptr, p->din1, p->din2, (int)D,
                          (int)A, false, s));
  actor_head_kernel<<<nb, 256, 0, s>>>(p->a_pi, eps2, A, p->din1, p->din2, A, ls, B, p->n_global,
                                       (int)A, p->ctl, p->dmean, p->part, p->tickets + 2,
                                       p->g_a + p->va.logstd_off);
  UL_TRY(check_launch("actor_head_kernel"));
  return mlp_backward(p->va, b.actor, p->ws_a, be, obs, p->ldo, true, B, p->acts_a, p->dmean,
                      A, p->g_a, nullptr, 0, 0, 0, true, false, p->work, s);
}

// phase 4: (reduced scalars back into ctl) Adam(actor), alpha ScalarAdam, latch
int sac_actor_apply(SacPlan* p, cudaStream_t s) {
  const ul_sac_bindings& b = p->b;
  if (p->world > 1) {
    sac_reduced_scalars_kernel<<<1, 32, 0, s>>>(p->ctl, nullptr, p->g_a + p->Pa);
    UL_TRY(check_launch("sac_reduced_scalars_kernel"));
  }
  UL_TRY(adam_one(b.actor, p->g_a, b.actor_m, b.actor_v, p->Pa, p->oc_a, s));
  alpha_step_kernel<<<1, 32, 0, s>>>(p->ctl, p->oc_a, p->n_global, p->d.target_entropy,
                                     rec_of(p));
  UL_TRY(check_launch("alpha_step_kernel"));
  sac_latch_kernel<<<1, 32, 0, s>>>(p->ctl, p->oc_a, p->oc_q1, p->oc_q2, 2, p->u);
  return check_launch("sac_latch_kernel");
}

// phase 5: Polyak q1t <- q1, q2t <- q2 (R:algos/sac.py:176-177), one launch,
// skipped after a divergence
int sac_polyak(SacPlan* p, cudaStream_t s) {
  const int64_t n = p->Pq;
  const bool vec = ((((uintptr_t)p->b.q1t | (uintptr_t)p->b.q1 | (uintptr_t)p->b.q2t |
                      (uintptr_t)p->b.q2) & 15) == 0);
  const int64_t n4 = vec ? n / 4 : 0;
  int64_t blocks = ceil_div(n4 > 0 ? n4 : n, 256);
  blocks = blocks > 4 * kNumSMs ? 4 * kNumSMs : blocks;
  return launch_pdl("polyak2_kernel", polyak2_kernel, dim3((unsigned)(blocks > 0 ? blocks : 1)),
                    dim3(256), 0, s, p->b.q1t, (const float*)p->b.q1, p->b.q2t,
                    (const float*)p->b.q2, n4, n, (float)(1.0 - p->d.tau), (float)p->d.tau,
                    (const ul_opt_ctl*)p->oc_q1);
}

int one_update(SacPlan* p, int u, bool do_actor, cudaStream_t s) {
  p->u = u;
  UL_TRY(sac_critic_grads(p, s));
  UL_TRY(sac_critic_apply(p, s));
  if (do_actor) {
    UL_TRY(sac_actor_grads(p, s));
    UL_TRY(sac_actor_apply(p, s));
  }
  return sac_polyak(p, s);
}

}  // namespace
}  // namespace ul

// One sac_update (R:algos/sac.py:139-178), issued kernel by kernel.  do_actor:
// update_count % policy_frequency == 0 after the increment.
extern "C" int ul_sac_plan_update(void* plan, int do_actor, void* stream) {
  SacPlan* p = (SacPlan*)plan;
  UL_CHECK_ARG(p && p->bound, "sac plan: not bound");
  cudaStream_t s = ul::as_stream(stream);
  UL_TRY(ul::fill_f64(p->stats, 4, __builtin_nan(""), s));
  return ul::one_update(p, 0, do_actor != 0, s);
}

// n updates as one CUDA graph (cached per (n, actor-step pattern)); the stats
// rows start as NaN so updates without an actor step report none.
extern "C" int ul_sac_plan_run(void* plan, int n_updates, int64_t update_count0,
                               int policy_frequency, void* stream) {
  SacPlan* p = (SacPlan*)plan;
  UL_CHECK_ARG(p && p->bound, "sac plan: not bound");
  UL_CHECK_ARG(n_updates >= 1 && n_updates <= p->n_cap,
               "sac plan: %d updates exceed the reserved %d", n_updates, p->n_cap);
  UL_CHECK_ARG(policy_frequency >= 1, "sac plan: policy_frequency must be >= 1");
  cudaStream_t s = ul::as_stream(stream);
  uint64_t mask = 0;
  for (int u = 0; u < n_updates; ++u)
    if ((update_count0 + u + 1) % policy_frequency == 0) mask |= uint64_t(1) << u;
  ul::SacGraph* g = nullptr;
  for (int i = 0; i < p->n_graphs; ++i)
    if (p->graphs[i].n == n_updates && p->graphs[i].mask == mask) g = &p->graphs[i];
  UL_CUDA(cudaEventRecord(p->ev_in, s));
  UL_CUDA(cudaStreamWaitEvent(p->cap, p->ev_in, 0));
  if (!g) {
    if (p->n_graphs == SacPlan::kMaxGraphs) ul::drop_graphs(p);
    cudaGraph_t gr;
    UL_CUDA(cudaStreamBeginCapture(p->cap, cudaStreamCaptureModeThreadLocal));
    int st = UL_OK;
    const double nanv = __builtin_nan("");
    for (int u = 0; u < n_updates && st == UL_OK; ++u) {
      // NaN-fill the update's stats row (a memset node would need a byte
      // pattern): the heads overwrite what the update produces
      st = ul::fill_f64(p->stats + 4 * u, 4, nanv, p->cap);
      if (st == UL_OK) st = ul::one_update(p, u, (mask >> u) & 1, p->cap);
    }
    cudaError_t ce = cudaStreamEndCapture(p->cap, &gr);
    if (st != UL_OK) return st;
    UL_CUDA(ce);
    g = &p->graphs[p->n_graphs++];
    g->n = n_updates;
    g->mask = mask;
    ce = cudaGraphInstantiate(&g->exec, gr, 0);
    cudaGraphDestroy(gr);
    UL_CUDA(ce);
  }
  UL_CUDA(cudaGraphLaunch(g->exec, p->cap));
  UL_CUDA(cudaEventRecord(p->ev_out, p->cap));
  UL_CUDA(cudaStreamWaitEvent(s, p->ev_out, 0));
  return UL_OK;
}

extern "C" int ul_sac_plan_reduce_buffers(void* plan, float** critic, int64_t* n_critic,
                                          float** actor, int64_t* n_actor) {
  SacPlan* p = (SacPlan*)plan;
  UL_CHECK_ARG(p && critic && n_critic && actor && n_actor, "sac plan: null argument");
  *critic = p->g_q1;
  *n_critic = 2 * p->Pq + 4;
  *actor = p->g_a;
  *n_actor = p->Pa + 4;
  return UL_OK;
}

#define UL_SAC_PHASE(NAME, FN)                                  \
  extern "C" int NAME(void* plan, void* stream) {               \
    SacPlan* p = (SacPlan*)plan;                                \
    UL_CHECK_ARG(p && p->bound, "sac plan: not bound");         \
    p->u = 0;                                                   \
    return ul::FN(p, ul::as_stream(stream));                    \
  }
UL_SAC_PHASE(ul_sac_plan_critic_grads, sac_critic_grads)
UL_SAC_PHASE(ul_sac_plan_critic_apply, sac_critic_apply)
UL_SAC_PHASE(ul_sac_plan_actor_grads, sac_actor_grads)
UL_SAC_PHASE(ul_sac_plan_actor_apply, sac_actor_apply)
UL_SAC_PHASE(ul_sac_plan_polyak, sac_polyak)
#undef UL_SAC_PHASE

// Read back the control records (and the run's per-update statistics) with
// one sync; UL_ERR_DIVERGENCE if any step of the run diverged (out->diverged:
// 1 critic side, 2 actor / alpha side; out->fail_update: which update).
extern "C" int ul_sac_plan_finish(void* plan, ul_sac_ctl* out, int64_t* ts, double* stats,
                                  int n, void* stream) {
  SacPlan* p = (SacPlan*)plan;
  UL_CHECK_ARG(p && out && ts, "sac plan: null");
  UL_CHECK_ARG(!stats || (n >= 0 && n <= p->n_cap), "sac plan: stats rows exceed the reserve");
  cudaStream_t s = ul::as_stream(stream);
  UL_CUDA(cudaMemcpyAsync(p->ctl_h, p->ctl, sizeof(ul_sac_ctl), cudaMemcpyDeviceToHost, s));
  ul_opt_ctl* srcs[3] = {p->oc_a, p->oc_q1, p->oc_q2};
  for (int k = 0; k < 3; ++k)
    UL_CUDA(cudaMemcpyAsync(p->oc_h + k, srcs[k], ul::ctl_hdr(), cudaMemcpyDeviceToHost, s));
  if (stats && n > 0)
    UL_CUDA(cudaMemcpyAsync(stats, p->stats, sizeof(double) * 4 * n, cudaMemcpyDeviceToHost, s));
  UL_CUDA(cudaStreamSynchronize(s));
  for (int k = 0; k < 3; ++k) ts[k] = p->oc_h[k].t[0];
  *out = *p->ctl_h;
  if (out->diverged) {
    ul::set_error(out->diverged == 1 ? "non-finite SAC critic loss or gradients"
                                     : "non-finite SAC actor / alpha loss or gradients");
    return UL_ERR_DIVERGENCE;
  }
  return UL_OK;
}
