// Tail of the joint clip / Adam prepare step (K13), shared by the prepare
// kernel (optim.cu) and the gradient reduction that folds it (mlp.cu
// reduce_all_kernel): fixed-order fold of per-block (sum g^2, non-finite)
// partials, the loss bookkeeping of R:algos/ppo.py:170-189, the joint norm
// and clip factor of R:tensornet/adam.py:30-40, and the per-segment update
// decision / step counters / divergence latch (R:tensornet/adam.py:43-80).
#pragma once
#include "internal.cuh"

namespace ul {
namespace {

constexpr double kLog2PiO = 1.8378770664093453;

// Runs in ONE CTA (blockDim 256).  Every global value it depends on is loaded
// up front with the loads in flight together -- the controller / stats
// records sit behind pointers the compiler must assume alias, so written as
// a chain of read-modify-writes the tail was ~10 us of serial load latency.
// (partials: sum g^2 of segment s from block b at part[b * ldp + s], its
// non-finite flag at bad[b * ldp + s])
static __device__ __noinline__ void prepare_tail(int nseg, const double* part, const int* bad_part,
                                          int ldp, ul_opt_ctl* ctl, const LossFinalize& lf,
                                          int has_lf, int nb, double* scratch) {
  __shared__ double red[UL_MAX_SEG];
  __shared__ int red_bad[UL_MAX_SEG];
  __shared__ double lstd[UL_MAX_ACT];
  // all segments' partials in one sweep (fixed per-thread order, then the
  // fixed-order block sum: deterministic)
  double acc[UL_MAX_SEG] = {0.0, 0.0, 0.0, 0.0};
  int bad[UL_MAX_SEG] = {0, 0, 0, 0};
  for (int b = threadIdx.x; b < nb; b += blockDim.x) {
#pragma unroll
    for (int s = 0; s < UL_MAX_SEG; ++s)
      if (s < nseg) {
        acc[s] += part[(int64_t)b * ldp + s];
        bad[s] |= bad_part[(int64_t)b * ldp + s];
      }
  }
  if (has_lf && (int)threadIdx.x < lf.A) lstd[threadIdx.x] = (double)lf.log_std[threadIdx.x];
#pragma unroll
  for (int s = 0; s < UL_MAX_SEG; ++s) {
    if (s >= nseg) break;
    const double tot = block_sum(acc[s], scratch);
    const int any_bad = __syncthreads_or(bad[s]);
    if (threadIdx.x == 0) {
      red[s] = tot;
      red_bad[s] = any_bad;
    }
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  // ---- loads (independent, issued together)
  const int loss_bad = ctl->loss_bad, was_diverged = ctl->diverged, steps = ctl->steps;
  const double max_norm = ctl->max_norm;
  int64_t t[UL_MAX_SEG];
#pragma unroll
  for (int s = 0; s < UL_MAX_SEG; ++s) t[s] = s < nseg ? ctl->t[s] : 0;
  float loss[3] = {0.f, 0.f, 0.f};
  ul_ppo_stats st{};
  if (has_lf) {
    loss[0] = lf.loss[0];
    loss[1] = lf.loss[1];
    loss[2] = lf.loss[2];
    st = *lf.st;
  }
  // ---- R:algos/ppo.py loss bookkeeping of the step (see heads.cu)
  int earlier_bad = loss_bad;
  if (has_lf) {
    const double pol = -(double)loss[0] / lf.n;
    const double val = (double)loss[1] / lf.n;
    const double kl = (double)loss[2] / lf.n;
    double ent = 0.0;
    for (int j = 0; j < lf.A; ++j) ent += lstd[j] + 0.5 * (kLog2PiO + 1.0);
    const double total = pol + lf.vcoef * val - lf.ecoef * ent;
    if (!isfinite(total)) earlier_bad = 1;
    if (!was_diverged && isfinite(total)) {
      st.policy_sum += pol;
      st.value_sum += val;
      st.entropy_sum += ent;
      st.kl_last = kl;
      if (lf.last_in_epoch) st.kl_epoch_sum += kl;
      st.steps += 1;
      *lf.st = st;
    }
  }
  // ---- joint norm, per-segment update decision (reference order: loss
  // check, then segment 0 finiteness, then segment 1, ...), divergence latch
  double joint = 0.0;
  for (int s = 0; s < nseg; ++s) {
    const double sum = red[s];
    const int sbad = red_bad[s];
    ctl->sumsq[s] = sum;
    ctl->seg_bad[s] = sbad;
    joint += sum;
    earlier_bad |= sbad;
    const int upd = !was_diverged && !earlier_bad;
    ctl->seg_update[s] = upd;
    if (upd) ctl->t[s] = t[s] + 1;
  }
  const double norm = sqrt(joint);
  ctl->norm = norm;
  // reference: factor applied only when max_norm > 0 and total > max_norm (NaN -> no clip)
  ctl->factor = (max_norm > 0.0 && norm > max_norm) ? max_norm / (norm + 1e-12) : 1.0;
  if (earlier_bad && !was_diverged) {
    ctl->diverged = 1;
    ctl->fail_step = steps;
  }
  ctl->loss_bad = 0;
  ctl->steps = steps + 1;
}

}  // namespace
}  // namespace ul
