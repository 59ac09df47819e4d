// Standalone kernels behind the per-call drop-in API of the SAC update and
// the Gaussian heads (the fused update itself is the plan in sac.cu):
//   ul_gaussian_dist      R:tensornet/distributions.py:29-63  (float64, like the reference)
//   ul_sample_squashed    R:tensornet/distributions.py:73-84  (float32 arithmetic)
//   ul_sac_soft_target    R:algos/sac.py:111-125              (y in float64)
//   ul_sac_mse_head       R:algos/sac.py:128-136              (loss + dout)
//   ul_sac_pick_head      R:algos/sac.py:194-205              (loss, argmin masks)
//   ul_sac_actor_head     R:algos/sac.py:207-217              (dmean, dlog_std)
//   ul_sum_f64            mean(logp + H) of alpha_loss_and_grad, :224-229
// Reductions use per-block partials folded in fixed order by the last block
// (deterministic); each call owns a small device workspace passed in by the
// caller (`work`, ul_api_work_doubles(n) doubles + one uint ticket at the end).
#include "internal.cuh"

namespace ul {
namespace {

constexpr double kLog2PiA = 1.8378770664093453;
constexpr int kT = 256;

// mode 0 plain sample (x = eps), 1 plain evaluation (x = action), 2 squashed
// sample (x = eps), 3 squashed evaluation (x = action), 4 squashed log-prob
// of given (u = x, a = a_in)
__global__ void dist_kernel(const double* __restrict__ mean, int64_t ldm,
                            const double* __restrict__ log_std, const double* __restrict__ x,
                            int64_t ldx, const double* __restrict__ a_in, int64_t n, int A,
                            int mode, double* __restrict__ sample, double* __restrict__ u_out,
                            double* __restrict__ logp) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    double lp = 0.0, corr = 0.0;
    for (int j = 0; j < A; ++j) {
      const double ls = log_std[j], sd = exp(ls), m = mean[i * ldm + j], v = x[i * ldx + j];
      double s, u;
      if (mode == 0) {         // plain sample
        u = m + sd * v;
        s = u;
      } else if (mode == 1) {  // plain evaluation at the action
        u = v;
        s = v;
      } else if (mode == 2) {  // squashed sample
        u = m + sd * v;
        s = tanh(u);
      } else if (mode == 3) {  // squashed evaluation: clip, atanh
        s = fmin(fmax(v, -1.0 + 1e-6), 1.0 - 1e-6);
        u = atanh(s);
      } else {                 // log-prob of a given (u, a) pair
        u = v;
        s = a_in[i * ldx + j];
      }
      const double z = (u - m) / sd;
      lp += -ls - 0.5 * kLog2PiA - 0.5 * z * z;
      if (mode >= 2) corr += log1p(-(s * s) + 1e-6);
      if (sample) sample[i * A + j] = s;
      if (u_out) u_out[i * A + j] = u;
    }
    logp[i] = lp - corr;
  }
}

// float32 arithmetic of sample_squashed on float32 mean / log_std / eps
__global__ void squashed_f32_kernel(const float* __restrict__ mean, int64_t ldm,
                                    const float* __restrict__ log_std,
                                    const float* __restrict__ eps, int64_t lde, int64_t n, int A,
                                    float* __restrict__ a_out, float* __restrict__ u_out,
                                    float* __restrict__ logp) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const float l2p = (float)kLog2PiA;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    float base = 0.f, corr = 0.f;
    for (int j = 0; j < A; ++j) {
      const float ls = log_std[j], sd = expf(ls), m = mean[i * ldm + j];
      const float u = __fadd_rn(m, __fmul_rn(sd, eps[i * lde + j]));
      const float a = tanhf(u);
      const float z = __fdiv_rn(__fsub_rn(u, m), sd);
      base += -ls - 0.5f * l2p - 0.5f * z * z;
      corr += log1pf(-(a * a) + 1e-6f);
      a_out[i * A + j] = a;
      u_out[i * A + j] = u;
    }
    logp[i] = base - corr;
  }
}

__global__ void soft_target_kernel(const double* __restrict__ r, const double* __restrict__ term,
                                   const double* __restrict__ nused, const float* __restrict__ q1,
                                   const float* __restrict__ q2, const float* __restrict__ logp,
                                   double log_alpha, double gamma, int64_t n,
                                   double* __restrict__ y) {
  const double alpha = exp(log_alpha);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const double soft = fmin((double)q1[i], (double)q2[i]) - alpha * (double)logp[i];
    y[i] = r[i] + pow(gamma, nused[i]) * (1.0 - term[i]) * soft;
  }
}

// loss = mean((q - y)^2); dq = 2 (q - y) / n
__global__ void __launch_bounds__(kT) mse_kernel(const float* __restrict__ q,
                                                 const double* __restrict__ y, int64_t n,
                                                 float* __restrict__ dq, double* part,
                                                 unsigned int* ticket, double* loss) {
  __shared__ double scratch[32];
  double acc = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const double e = (double)q[i] - y[i];
    acc += e * e;
    dq[i] = (float)(2.0 * e / (double)n);  // (the reference casts dout to f32)
  }
  const double b = block_sum(acc, scratch);
  if (threadIdx.x == 0) part[blockIdx.x] = b;
  if (!last_block_ticket(ticket, gridDim.x)) return;
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (unsigned k = 0; k < gridDim.x; ++k) s += part[k];
    *loss = s / (double)n;
  }
}

// loss = mean(alpha logp - min(q1, q2)); d1 = [q1 <= q2], d2 = 1 - d1
__global__ void __launch_bounds__(kT) pick_kernel(const float* __restrict__ q1,
                                                  const float* __restrict__ q2,
                                                  const float* __restrict__ logp, int64_t n,
                                                  double log_alpha, float* __restrict__ d1,
                                                  float* __restrict__ d2, double* part,
                                                  unsigned int* ticket, double* loss) {
  __shared__ double scratch[32];
  const double alpha = exp(log_alpha);
  double acc = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const float a = q1[i], b = q2[i];
    const bool pick = a <= b;
    d1[i] = pick ? 1.f : 0.f;
    d2[i] = pick ? 0.f : 1.f;
    acc += alpha * (double)logp[i] - (double)fminf(a, b);
  }
  const double b = block_sum(acc, scratch);
  if (threadIdx.x == 0) part[blockIdx.x] = b;
  if (!last_block_ticket(ticket, gridDim.x)) return;
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (unsigned k = 0; k < gridDim.x; ++k) s += part[k];
    *loss = s / (double)n;
  }
}

// dmean = (alpha dlogp/du - dQ/da (1 - a^2)) / n with dQ/da = dq1 + dq2 (the
// two critics' masked input gradients); dlog_std column sums ADDED into dls
// (actor_grads.log_std += dlog_std)
__global__ void __launch_bounds__(kT) actor_grad_kernel(
    const float* __restrict__ a, const float* __restrict__ eps, const float* __restrict__ dq1,
    const float* __restrict__ dq2, int64_t ldq, const float* __restrict__ log_std, int64_t n,
    int A, double log_alpha, float* __restrict__ dmean, double* part, unsigned int* ticket,
    float* __restrict__ dls) {
  __shared__ double scratch[32];
  const double alpha = exp(log_alpha), inv_n = 1.0 / (double)n;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int j = 0; j < A; ++j) {
    const double sd = exp((double)log_std[j]);
    double acc = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
      const double av = (double)a[i * A + j];
      const double oma = 1.0 - av * av;
      const double dlogp_du = 2.0 * av * oma / (oma + 1e-6);
      const double dq = (double)dq1[i * ldq + j] + (double)dq2[i * ldq + j];
      const double du_dls = sd * (double)eps[i * A + j];
      dmean[i * A + j] = (float)((alpha * dlogp_du - dq * oma) * inv_n);
      acc += (alpha * (-1.0 + dlogp_du * du_dls) - dq * oma * du_dls) * inv_n;
    }
    const double b = block_sum(acc, scratch);
    if (threadIdx.x == 0) part[(int64_t)blockIdx.x * A + j] = b;
  }
  if (!last_block_ticket(ticket, gridDim.x)) return;
  for (int j = threadIdx.x; j < A; j += blockDim.x) {
    double s = 0.0;
    for (unsigned k = 0; k < gridDim.x; ++k) s += part[(int64_t)k * A + j];
    dls[j] = dls[j] + (float)s;
  }
}

__global__ void __launch_bounds__(kT) sum_kernel(const float* __restrict__ x, int64_t n,
                                                 double shift, double* part,
                                                 unsigned int* ticket, double* out) {
  __shared__ double scratch[32];
  double acc = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    acc += (double)x[i] + shift;
  const double b = block_sum(acc, scratch);
  if (threadIdx.x == 0) part[blockIdx.x] = b;
  if (!last_block_ticket(ticket, gridDim.x)) return;
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (unsigned k = 0; k < gridDim.x; ++k) s += part[k];
    *out = s;
  }
}

constexpr int kApiBlocks = 256;  // reduction grid (partials + ticket fit the workspace)

unsigned blocks_for(int64_t n) {
  const int64_t b = ceil_div(n > 0 ? n : 1, kT);
  return (unsigned)(b < kApiBlocks ? b : kApiBlocks);
}

}  // namespace
}  // namespace ul

// workspace: kApiBlocks * UL_MAX_ACT partial doubles + the ticket (zeroed once)
extern "C" int64_t ul_api_work_doubles(void) { return (int64_t)ul::kApiBlocks * UL_MAX_ACT + 8; }

extern "C" int ul_gaussian_dist(const double* mean, int64_t ldm, const double* log_std,
                                const double* x, int64_t ldx, const double* a_in, int64_t n,
                                int A, int mode, double* sample, double* u_out, double* logp,
                                void* stream) {
  UL_CHECK_ARG(n >= 0 && A >= 1 && ldm >= A && ldx >= A && mode >= 0 && mode <= 4 &&
                   (mode != 4 || a_in),
               "gaussian_dist: bad shape / mode");
  if (n == 0) return UL_OK;
  ul::dist_kernel<<<ul::blocks_for(n), ul::kT, 0, ul::as_stream(stream)>>>(
      mean, ldm, log_std, x, ldx, a_in, n, A, mode, sample, u_out, logp);
  return ul::check_launch("dist_kernel");
}

extern "C" int ul_sample_squashed(const float* mean, int64_t ldm, const float* log_std,
                                  const float* eps, int64_t lde, int64_t n, int A, float* a,
                                  float* u, float* logp, void* stream) {
  UL_CHECK_ARG(n >= 0 && A >= 1 && ldm >= A && lde >= A, "sample_squashed: bad shape");
  if (n == 0) return UL_OK;
  ul::squashed_f32_kernel<<<ul::blocks_for(n), ul::kT, 0, ul::as_stream(stream)>>>(
      mean, ldm, log_std, eps, lde, n, A, a, u, logp);
  return ul::check_launch("squashed_f32_kernel");
}

extern "C" int ul_sac_soft_target(const double* r, const double* term, const double* nused,
                                  const float* q1t, const float* q2t, const float* logp,
                                  double log_alpha, double gamma, int64_t n, double* y,
                                  void* stream) {
  UL_CHECK_ARG(n >= 0, "soft_target: bad shape");
  if (n == 0) return UL_OK;
  ul::soft_target_kernel<<<ul::blocks_for(n), ul::kT, 0, ul::as_stream(stream)>>>(
      r, term, nused, q1t, q2t, logp, log_alpha, gamma, n, y);
  return ul::check_launch("soft_target_kernel");
}

extern "C" int ul_sac_mse_head(const float* q, const double* y, int64_t n, float* dq,
                               double* loss, double* work, void* stream) {
  UL_CHECK_ARG(n >= 1 && work, "mse_head: bad shape");
  const unsigned nb = ul::blocks_for(n);
  ul::mse_kernel<<<nb, ul::kT, 0, ul::as_stream(stream)>>>(
      q, y, n, dq, work, (unsigned int*)(work + ul_api_work_doubles() - 1), loss);
  return ul::check_launch("mse_kernel");
}

extern "C" int ul_sac_pick_head(const float* q1, const float* q2, const float* logp, int64_t n,
                                double log_alpha, float* d1, float* d2, double* loss,
                                double* work, void* stream) {
  UL_CHECK_ARG(n >= 1 && work, "pick_head: bad shape");
  ul::pick_kernel<<<ul::blocks_for(n), ul::kT, 0, ul::as_stream(stream)>>>(
      q1, q2, logp, n, log_alpha, d1, d2, work,
      (unsigned int*)(work + ul_api_work_doubles() - 1), loss);
  return ul::check_launch("pick_kernel");
}

extern "C" int ul_sac_actor_head(const float* a, const float* eps, const float* dq1,
                                 const float* dq2, int64_t ldq, const float* log_std, int64_t n,
                                 int A, double log_alpha, float* dmean, float* dlog_std,
                                 double* work, void* stream) {
  UL_CHECK_ARG(n >= 1 && A >= 1 && A <= UL_MAX_ACT && ldq >= A && work,
               "actor_head: bad shape");
  ul::actor_grad_kernel<<<ul::blocks_for(n), ul::kT, 0, ul::as_stream(stream)>>>(
      a, eps, dq1, dq2, ldq, log_std, n, A, log_alpha, dmean, work,
      (unsigned int*)(work + ul_api_work_doubles() - 1), dlog_std);
  return ul::check_launch("actor_grad_kernel");
}

extern "C" int ul_sum_f64(const float* x, int64_t n, double shift, double* out, double* work,
                          void* stream) {
  UL_CHECK_ARG(n >= 1 && work, "sum: bad shape");
  ul::sum_kernel<<<ul::blocks_for(n), ul::kT, 0, ul::as_stream(stream)>>>(
      x, n, shift, work, (unsigned int*)(work + ul_api_work_doubles() - 1), out);
  return ul::check_launch("sum_kernel");
}
