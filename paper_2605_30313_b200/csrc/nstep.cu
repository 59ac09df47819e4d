// FlashSAC collector-side transforms on the device:
// ReturnStdNormalizer.normalize (R:algos/estimators.py:153-163), NStepPacker.push
// (:166-207) and the replay insert of the packed rows (RowCodec layout,
// R:replaypath/storage.py:17-46) -- one environment step of N envs per call.
//
// State (device): per-env discounted returns (f64) + running Welford stats of
// the returns (count, mean, m2; f64) for the normaliser; per env a circular
// pending window of <= n items (obs, action, accumulated reward f64, k).
// Per call:
//   K1 nstep_norm_kernel  (1 block)  returns update, batch moments merged into
//                                    the running stats (Chan, fixed order),
//                                    rewards / (std + eps) clipped (f64)
//   K2 nstep_pack_kernel  (env/thread) pending rewards += gamma^k r, append,
//                                    decide the rows this env emits
//   K3 nstep_scan_kernel  (1 block)  exclusive scan of the per-env counts (the
//                                    reference's env-major emission order)
//   K4 nstep_emit_kernel  (warp/env) codec rows straight into the HBM ring
// The normaliser merges the step's returns as a batch (Chan) where the
// reference folds them one by one: the same statistics up to f64 rounding.
#include "internal.cuh"

namespace ul {
namespace {

struct NstepState {
  int n_envs, n, d, a;
  double gamma;
  // normaliser (norm_on = 0: rewards pass through)
  int norm_on;
  double ngamma, g_max, eps;
  double* returns;  // [N]
  double* stats;    // [count, mean, m2, std]
  double* rnorm;    // [N] this step's (normalised) rewards
  // pending windows
  float* p_obs;  // [N, n, d]
  float* p_act;  // [N, n, a]
  double* p_r;   // [N, n]
  int* p_k;      // [N, n]
  int* p_start;  // [N]
  int* p_len;    // [N]
  // this step's emission plan
  int* e_first;  // [N] slot of the first emitted item
  int* e_cnt;    // [N]
  int* e_done;   // [N] 1: episode end (all pending emitted with the env's terminated)
  int64_t* e_off;  // [N + 1] exclusive scan, e_off[N] = total
};

__global__ void __launch_bounds__(1024) nstep_norm_kernel(NstepState S, const float* __restrict__ r,
                                                          const uint8_t* __restrict__ term,
                                                          const uint8_t* __restrict__ trunc) {
  __shared__ double red[32];
  __shared__ double s_mean;
  const int N = S.n_envs;
  double sum = 0.0;
  for (int e = threadIdx.x; e < N; e += blockDim.x) {
    const bool done = term[e] || trunc[e];
    const double g = S.returns[e] * S.ngamma * (done ? 0.0 : 1.0) + (double)r[e];
    S.returns[e] = g;
    sum += g;
  }
  // batch mean, then centred sum of squares (fixed-order block reductions)
  double t = block_sum(sum, red);
  if (threadIdx.x == 0) s_mean = t / N;
  __syncthreads();
  const double bm = s_mean;
  double sq = 0.0;
  for (int e = threadIdx.x; e < N; e += blockDim.x) {
    const double dv = S.returns[e] - bm;
    sq += dv * dv;
  }
  t = block_sum(sq, red);
  if (threadIdx.x == 0) {
    // Chan merge of (N, bm, t) into the running (count, mean, m2)
    const double c = S.stats[0], mu = S.stats[1], m2 = S.stats[2];
    const double tot = c + N;
    const double delta = bm - mu;
    S.stats[0] = tot;
    S.stats[1] = mu + delta * (N / tot);
    S.stats[2] = m2 + t + delta * delta * (c * N / tot);
    S.stats[3] = tot < 2.0 ? 1.0 : sqrt(S.stats[2] / tot);
  }
  __syncthreads();
  const double sd = S.stats[3], bound = (1.0 - S.ngamma) * S.g_max;
  for (int e = threadIdx.x; e < N; e += blockDim.x)
    S.rnorm[e] = fmin(fmax((double)r[e] / (sd + S.eps), -bound), bound);
}

__global__ void nstep_pack_kernel(NstepState S, const float* __restrict__ obs,
                                  const float* __restrict__ act, const float* __restrict__ r,
                                  const uint8_t* __restrict__ term,
                                  const uint8_t* __restrict__ trunc) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= S.n_envs) return;
  const int n = S.n;
  const double re = S.norm_on ? S.rnorm[e] : (double)r[e];
  int st = S.p_start[e], len = S.p_len[e];
  // pending rewards += gamma^k r_e, k += 1
  for (int j = 0; j < len; ++j) {
    const int q = e * n + (st + j) % n;
    S.p_r[q] += pow(S.gamma, (double)S.p_k[q]) * re;
    S.p_k[q] += 1;
  }
  // append (obs, act, r, 1)
  const int slot = (st + len) % n;
  const int q = e * n + slot;
  for (int c = 0; c < S.d; ++c) S.p_obs[(int64_t)q * S.d + c] = obs[(int64_t)e * S.d + c];
  for (int c = 0; c < S.a; ++c) S.p_act[(int64_t)q * S.a + c] = act[(int64_t)e * S.a + c];
  S.p_r[q] = re;
  S.p_k[q] = 1;
  len += 1;
  const bool done = term[e] || trunc[e];
  if (done) {  // every pending item, with the env's terminated flag
    S.e_first[e] = st;
    S.e_cnt[e] = len;
    S.e_done[e] = 1;
    st = (st + len) % n;
    len = 0;
  } else if (S.p_k[e * n + st] == n) {  // the oldest window is full
    S.e_first[e] = st;
    S.e_cnt[e] = 1;
    S.e_done[e] = 0;
    st = (st + 1) % n;
    len -= 1;
  } else {
    S.e_first[e] = st;
    S.e_cnt[e] = 0;
    S.e_done[e] = 0;
  }
  S.p_start[e] = st;
  S.p_len[e] = len;
}

// exclusive scan of e_cnt (one block, fixed order)
__global__ void __launch_bounds__(1024) nstep_scan_kernel(NstepState S) {
  __shared__ int64_t part[1024];
  const int N = S.n_envs;
  const int per = (N + blockDim.x - 1) / blockDim.x;
  const int lo = threadIdx.x * per, hi = min(N, lo + per);
  int64_t s = 0;
  for (int e = lo; e < hi; ++e) s += S.e_cnt[e];
  part[threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t acc = 0;
    for (int i = 0; i < (int)blockDim.x; ++i) {
      const int64_t v = part[i];
      part[i] = acc;
      acc += v;
    }
    S.e_off[N] = acc;
  }
  __syncthreads();
  int64_t acc = part[threadIdx.x];
  for (int e = lo; e < hi; ++e) {
    S.e_off[e] = acc;
    acc += S.e_cnt[e];
  }
}

// codec row = obs (d) | action (a) | reward | next_obs (d) | terminated | n_used
__global__ void nstep_emit_kernel(NstepState S, const float* __restrict__ next_obs,
                                  const uint8_t* __restrict__ term, float* __restrict__ ring,
                                  int64_t cap, int64_t ldr, int64_t head) {
  const int lane = threadIdx.x & 31;
  const int e = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (e >= S.n_envs) return;
  const int cnt = S.e_cnt[e];
  const int d = S.d, a = S.a, n = S.n;
  for (int j = 0; j < cnt; ++j) {
    const int q = e * n + (S.e_first[e] + j) % n;
    float* row = ring + ((head + S.e_off[e] + j) % cap) * ldr;
    for (int c = lane; c < d; c += 32) {
      row[c] = S.p_obs[(int64_t)q * d + c];
      row[d + a + 1 + c] = next_obs[(int64_t)e * d + c];
    }
    for (int c = lane; c < a; c += 32) row[d + c] = S.p_act[(int64_t)q * a + c];
    if (lane == 0) {
      row[d + a] = (float)S.p_r[q];
      row[2 * d + a + 1] = (S.e_done[e] && term[e]) ? 1.f : 0.f;
      row[2 * d + a + 2] = (float)S.p_k[q];
    }
  }
}

int64_t nstep_state_bytes(int N, int n, int d, int a) {
  const int64_t Nn = (int64_t)N * n;
  return 8 * (int64_t)N * 2 + 8 * 4 + 4 * Nn * (d + a) + 8 * Nn + 4 * Nn + 4 * (int64_t)N * 5 +
         8 * ((int64_t)N + 1) + 1024;
}

NstepState carve_state(void* base, int N, int n, int d, int a) {
  NstepState S{};
  char* p = static_cast<char*>(base);
  auto take = [&](int64_t bytes) {
    char* r = p;
    p += (bytes + 15) / 16 * 16;
    return r;
  };
  const int64_t Nn = (int64_t)N * n;
  S.returns = (double*)take(8 * (int64_t)N);
  S.stats = (double*)take(8 * 4);
  S.rnorm = (double*)take(8 * (int64_t)N);
  S.p_r = (double*)take(8 * Nn);
  S.e_off = (int64_t*)take(8 * ((int64_t)N + 1));
  S.p_obs = (float*)take(4 * Nn * d);
  S.p_act = (float*)take(4 * Nn * a);
  S.p_k = (int*)take(4 * Nn);
  S.p_start = (int*)take(4 * (int64_t)N);
  S.p_len = (int*)take(4 * (int64_t)N);
  S.e_first = (int*)take(4 * (int64_t)N);
  S.e_cnt = (int*)take(4 * (int64_t)N);
  S.e_done = (int*)take(4 * (int64_t)N);
  return S;
}

}  // namespace
}  // namespace ul

// Device state bytes for N envs, window n, obs d, action a (zero-initialise).
extern "C" int64_t ul_nstep_state_bytes(int n_envs, int n, int obs_dim, int act_dim) {
  if (n_envs < 1 || n < 1 || obs_dim < 1 || act_dim < 1) return -1;
  return ul::nstep_state_bytes(n_envs, n, obs_dim, act_dim) + 256;
}

// One environment step: (optional) reward normalisation, n-step packing and
// the insert of the emitted codec rows into ring[(head + i) % cap] (pitch ldr
// floats).  Inputs are device arrays: obs/next_obs [N, d], act [N, a], r [N]
// f32, term/trunc [N] u8.  *count_out (device int64) receives the number of
// rows written (the env-major order of R:algos/estimators.py:195-207).
// norm_gamma <= 0 disables the normaliser.
extern "C" int ul_nstep_push(void* state, int n_envs, int n, int obs_dim, int act_dim,
                             double gamma, double norm_gamma, double g_max, double eps,
                             const float* obs, const float* act, const float* r,
                             const float* next_obs, const uint8_t* term, const uint8_t* trunc,
                             float* ring, int64_t cap, int64_t ldr, int64_t head,
                             int64_t* count_out, void* stream) {
  UL_CHECK_ARG(state && n_envs >= 1 && n >= 1 && obs_dim >= 1 && act_dim >= 1,
               "nstep: bad state / shape");
  UL_CHECK_ARG(ldr >= 2 * obs_dim + act_dim + 3 && cap >= 1, "nstep: ring pitch / capacity");
  cudaStream_t s = ul::as_stream(stream);
  ul::NstepState S = ul::carve_state(state, n_envs, n, obs_dim, act_dim);
  S.n_envs = n_envs;
  S.n = n;
  S.d = obs_dim;
  S.a = act_dim;
  S.gamma = gamma;
  S.norm_on = norm_gamma > 0.0 ? 1 : 0;
  S.ngamma = norm_gamma;
  S.g_max = g_max;
  S.eps = eps;
  if (S.norm_on) {
    ul::nstep_norm_kernel<<<1, 1024, 0, s>>>(S, r, term, trunc);
    UL_TRY(ul::check_launch("nstep_norm_kernel"));
  }
  ul::nstep_pack_kernel<<<(unsigned)ul::ceil_div(n_envs, 128), 128, 0, s>>>(S, obs, act, r, term,
                                                                             trunc);
  UL_TRY(ul::check_launch("nstep_pack_kernel"));
  ul::nstep_scan_kernel<<<1, 1024, 0, s>>>(S);
  UL_TRY(ul::check_launch("nstep_scan_kernel"));
  ul::nstep_emit_kernel<<<(unsigned)ul::ceil_div((int64_t)n_envs * 32, 256), 256, 0, s>>>(
      S, next_obs, term, ring, cap, ldr, head);
  UL_TRY(ul::check_launch("nstep_emit_kernel"));
  if (count_out)
    UL_CUDA(cudaMemcpyAsync(count_out, S.e_off + n_envs, sizeof(int64_t), cudaMemcpyDefault, s));
  return UL_OK;
}

// normaliser statistics (count, mean, m2, std) -> out[4] (device or host via UVA)
extern "C" int ul_nstep_norm_stats(void* state, int n_envs, int n, int obs_dim, int act_dim,
                                   double* out, void* stream) {
  ul::NstepState S = ul::carve_state(state, n_envs, n, obs_dim, act_dim);
  UL_CUDA(cudaMemcpyAsync(out, S.stats, 4 * sizeof(double), cudaMemcpyDefault,
                          ul::as_stream(stream)));
  return UL_OK;
}
