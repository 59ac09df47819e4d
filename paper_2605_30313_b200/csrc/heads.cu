// K9 PPO loss head (+ advantage statistics), fused per minibatch row.
//
// Replaces R:algos/ppo.py:70-129 (ppo_loss_and_grads minus the MLP passes),
// R:tensornet/distributions.py:11-26 (gaussian_log_prob / entropy) and
// R:algos/ppo.py:132-133 (normalize_advantages, folded into the head: the
// advantage is normalised on the fly from device-resident (mean, std)).
// One thread per row computes logp, ratio, the clipped surrogate with the
// reference's tie rule (gradient flows iff ratio*A <= clip(ratio)*A), dmean,
// the clipped value loss (gradient iff (v-R)^2 >= (v_clip-R)^2) and dv; the
// row terms (sum min-surrogate, sum value loss, sum KL, dlog_std[A]) are
// block-reduced, and the last CTA folds the per-CTA partials in fixed order
// into the gradient buffer (log_std slot) and the loss-partial slots that the
// data-parallel all-reduce carries.  Per-row math is float64 (the reference's
// ratio/advantage/loss dtype, Appendix B of SURVEY.md).
#include "learner.cuh"

namespace ul {
namespace {

constexpr double kLog2Pi = 1.8378770664093453;

constexpr int kHeadThr = 128, kHeadWarps = kHeadThr / 32;

__global__ void __launch_bounds__(kHeadThr) ppo_head_kernel(PpoHeadArgs a) {
  __shared__ double s_ls[UL_MAX_ACT], s_isd[UL_MAX_ACT];
  __shared__ double red[kHeadWarps][3 + UL_MAX_ACT];
  __shared__ double s_lsum;
  const int A = a.A, nq = 3 + A;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  pdl_trigger();
  pdl_wait();
  // per-dimension constants once per block: log_std and 1/std
  for (int j = threadIdx.x; j < A; j += blockDim.x) {
    const double ls = (double)a.log_std[j];
    s_ls[j] = ls;
    s_isd[j] = exp(-ls);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int j = 0; j < A; ++j) t += s_ls[j];
    s_lsum = t;
  }
  __syncthreads();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool act_row = i < a.n_local;
  double pol = 0.0, val = 0.0, kl = 0.0, dlogp = 0.0;
  const double adv_mean = a.adv_stats ? a.adv_stats[0] : 0.0;
  const double adv_den = a.adv_stats ? a.adv_stats[1] + 1e-8 : 1.0;
  const float* act = a.act + i * a.ld_act;
  const float* mean = a.mean + i * a.ld_mean;
  if (act_row) {
    double zz = 0.0;
    for (int j = 0; j < A; ++j) {
      const double z = ((double)act[j] - (double)mean[j]) * s_isd[j];
      zz += z * z;
    }
    const double logp = -s_lsum - A * (0.5 * kLog2Pi) - 0.5 * zz;
    const double b = (double)a.blogp[i];
    const double adv = ((double)a.adv[i] - adv_mean) / adv_den;
    const double ratio = exp(logp - b);
    const double s1 = ratio * adv;
    const double rc = fmin(fmax(ratio, 1.0 - a.clip), 1.0 + a.clip);
    const double s2 = rc * adv;
    pol = fmin(s1, s2);
    dlogp = (s1 <= s2) ? -adv * ratio / a.n_global : 0.0;
    kl = b - logp;
    // value head (R:algos/ppo.py:107-118)
    const double v = (double)a.v[i * a.ld_v];
    const double R = (double)a.ret[i];
    double dv;
    if (a.clipped_v) {
      const double ov = (double)a.oldv[i];
      const double vc = ov + fmin(fmax(v - ov, -a.clip), a.clip);
      const double lu = (v - R) * (v - R), lc = (vc - R) * (vc - R);
      val = fmax(lu, lc);
      dv = lu >= lc ? 2.0 * (v - R) / a.n_global : 0.0;
    } else {
      val = (v - R) * (v - R);
      dv = 2.0 * (v - R) / a.n_global;
    }
    a.dv[i] = (float)(dv * a.vcoef);
  }
  // row terms, warp-reduced: [pol, val, kl, dls_0 .. dls_{A-1}]
  double r = warp_sum(pol);
  if (lane == 0) red[w][0] = r;
  r = warp_sum(val);
  if (lane == 0) red[w][1] = r;
  r = warp_sum(kl);
  if (lane == 0) red[w][2] = r;
  for (int j = 0; j < A; ++j) {
    double t = 0.0;
    if (act_row) {
      const double z = ((double)act[j] - (double)mean[j]) * s_isd[j];
      a.dmean[i * a.ld_dmean + j] = (float)(dlogp * z * s_isd[j]);
      t = dlogp * (z * z - 1.0);
    }
    t = warp_sum(t);
    if (lane == 0) red[w][3 + j] = t;
  }
  __syncthreads();
  double* part = a.part + (int64_t)blockIdx.x * nq;
  for (int q = threadIdx.x; q < nq; q += blockDim.x) {
    double t = 0.0;
    for (int k = 0; k < kHeadWarps; ++k) t += red[k][q];
    part[q] = t;
  }
  if (!last_block_ticket(a.ticket, gridDim.x)) return;
  // last CTA: fixed-order fold of the per-CTA partials.  8 lanes per term
  // (16 terms per pass), each summing blocks b = l, l + 8, ... with all loads
  // in flight, then a 3-step shuffle tree within the 8 lanes.
  const unsigned nb = gridDim.x;
  for (int q0 = 0; q0 < nq; q0 += kHeadThr / 8) {
    const int q = q0 + (int)(threadIdx.x >> 3), l = threadIdx.x & 7;
    double t = 0.0;
    if (q < nq) {
      for (unsigned b0 = l; b0 < nb; b0 += 64) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const unsigned b = b0 + 8 * u;
          v[u] = b < nb ? a.part[(int64_t)b * nq + q] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) t += v[u];
      }
    }
    t += __shfl_xor_sync(0xffffffffu, t, 1);
    t += __shfl_xor_sync(0xffffffffu, t, 2);
    t += __shfl_xor_sync(0xffffffffu, t, 4);
    if (q < nq && l == 0) {
      if (q < 3) a.loss_out[q] = (float)t;
      else a.dlogstd_out[q - 3] = (float)(t + a.ent_coef_add);
    }
  }
}

// mean / population std of the advantages (normalize_advantages), f64
__global__ void __launch_bounds__(256) adv_stats_kernel(const float* __restrict__ adv, int64_t n,
                                                        double* part, unsigned int* ticket,
                                                        double* out) {
  __shared__ double scratch[32];
  const double c = (double)adv[0];
  double s1 = 0.0, s2 = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const double d = (double)adv[i] - c;
    s1 += d;
    s2 += d * d;
  }
  double r1 = block_sum(s1, scratch);
  double r2 = block_sum(s2, scratch);
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = r1;
    part[2 * blockIdx.x + 1] = r2;
  }
  if (!last_block_ticket(ticket, gridDim.x)) return;
  if (threadIdx.x == 0) {
    double t1 = 0.0, t2 = 0.0;
    for (unsigned b = 0; b < gridDim.x; ++b) {
      t1 += part[2 * b];
      t2 += part[2 * b + 1];
    }
    const double m1 = t1 / (double)n;
    double var = t2 / (double)n - m1 * m1;
    var = var < 0.0 ? 0.0 : var;
    out[0] = c + m1;
    out[1] = sqrt(var);
    // NaN advantages -> NaN stats -> non-finite loss -> DivergenceError (reference test)
    if (!isfinite(t1) || !isfinite(t2)) out[0] = out[1] = NAN;
    // raw sums for a cross-rank combination (ul_ppo_plan_adv_sums)
    const double nn = (double)n;
    out[2] = t1 + nn * c;
    out[3] = t2 + 2.0 * c * t1 + nn * c * c;
    out[4] = nn;
  }
}

// (mean, population std) from all-reduced [sum A, sum A^2, n]
__global__ void adv_finalize_kernel(const double* __restrict__ sums, double* out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const double n = sums[2], m = sums[0] / n;
  double var = sums[1] / n - m * m;
  var = var < 0.0 ? 0.0 : var;
  out[0] = m;
  out[1] = sqrt(var);
  if (!isfinite(sums[0]) || !isfinite(sums[1])) out[0] = out[1] = NAN;
}

// per-step loss finalisation after the (optional) all-reduce of the partials
__global__ void ppo_loss_finalize_kernel(const float* __restrict__ loss, const float* __restrict__ log_std,
                                         int A, double n, double vcoef, double ecoef,
                                         int last_in_epoch, ul_opt_ctl* ctl, ul_ppo_stats* st) {
  pdl_trigger();
  pdl_wait();
  if (threadIdx.x != 0) return;
  const double pol = -(double)loss[0] / n;
  const double val = (double)loss[1] / n;
  const double kl = (double)loss[2] / n;
  double ent = 0.0;
  for (int j = 0; j < A; ++j) ent += (double)log_std[j] + 0.5 * (kLog2Pi + 1.0);
  const double total = pol + vcoef * val - ecoef * ent;
  if (!isfinite(total)) ctl->loss_bad = 1;
  if (!ctl->diverged && isfinite(total)) {
    st->policy_sum += pol;
    st->value_sum += val;
    st->entropy_sum += ent;
    st->kl_last = kl;
    if (last_in_epoch) st->kl_epoch_sum += kl;
    st->steps += 1;
  }
}

__global__ void gauss_logp_kernel(const float* __restrict__ mean, int64_t ldm,
                                  const float* __restrict__ log_std, const float* __restrict__ act,
                                  int64_t lda, int64_t n, int A, float* __restrict__ out) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    double lp = 0.0;
    for (int j = 0; j < A; ++j) {
      const double ls = (double)log_std[j];
      const double z = ((double)act[i * lda + j] - (double)mean[i * ldm + j]) / exp(ls);
      lp += -ls - 0.5 * kLog2Pi - 0.5 * z * z;
    }
    out[i] = (float)lp;
  }
}

}  // namespace

int launch_ppo_head(const PpoHeadArgs& a, cudaStream_t s) {
  const unsigned blocks = (unsigned)ceil_div(a.n_local > 0 ? a.n_local : 1, kHeadThr);
  return launch_pdl("ppo_head_kernel", ppo_head_kernel, dim3(blocks), dim3(kHeadThr), 0, s, a);
}

int ppo_head_partial_doubles(int64_t n_local, int A) {
  // (per-CTA partials of ppo_head_kernel or of the fused output stage's
  // 64-row blocks, whichever is more)
  return (int)(ceil_div(n_local > 0 ? n_local : 1, 64) * (3 + A));
}

int launch_adv_stats(const float* adv, int64_t n, double* part, unsigned int* ticket, double* out,
                     cudaStream_t s) {
  int blocks = (int)ceil_div(n, 256 * 8);
  blocks = blocks < 1 ? 1 : (blocks > kAdvStatBlocks ? kAdvStatBlocks : blocks);
  adv_stats_kernel<<<blocks, 256, 0, s>>>(adv, n, part, ticket, out);
  return check_launch("adv_stats_kernel");
}

int launch_adv_finalize(const double* sums, double* out, cudaStream_t s) {
  adv_finalize_kernel<<<1, 32, 0, s>>>(sums, out);
  return check_launch("adv_finalize_kernel");
}

int launch_ppo_loss_finalize(const float* loss, const float* log_std, int A, double n,
                             double vcoef, double ecoef, int last_in_epoch, ul_opt_ctl* ctl,
                             ul_ppo_stats* st, cudaStream_t s) {
  return launch_pdl("ppo_loss_finalize_kernel", ppo_loss_finalize_kernel, dim3(1), dim3(32), 0, s,
                    loss, log_std, A, n, vcoef, ecoef, last_in_epoch, ctl, st);
}

}  // namespace ul

// log N(action; mean, exp(log_std)) summed over the action dims
// (R:tensornet/distributions.py:11-18); f64 arithmetic, f32 out.
extern "C" int ul_gaussian_logp(const float* mean, int64_t ld_mean, const float* log_std,
                                const float* action, int64_t ld_act, int64_t n, int A, float* out,
                                void* stream) {
  UL_CHECK_ARG(n >= 0 && A >= 1 && ld_mean >= A && ld_act >= A, "gaussian_logp: bad shape");
  if (n == 0) return UL_OK;
  int64_t blocks = ul::ceil_div(n, 256);
  blocks = blocks > 8 * ul::kNumSMs ? 8 * ul::kNumSMs : blocks;
  ul::gauss_logp_kernel<<<(unsigned)blocks, 256, 0, ul::as_stream(stream)>>>(
      mean, ld_mean, log_std, action, ld_act, n, A, out);
  return ul::check_launch("gauss_logp_kernel");
}
