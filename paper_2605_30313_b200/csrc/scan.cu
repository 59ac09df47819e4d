// K1 GAE and K2 V-trace reverse scans over [T, N_env] (t-major, env-contiguous).
//
// Replaces R:algos/estimators.py:15-63 (gae, _next_values) and :66-122 (vtrace).
// Both recursions are first-order affine maps in the reverse time direction,
//     X_t = d_t + g_t * X_{t+1},   X_T = 0,
// (GAE: X = A, g = gamma*lam*(1-done); V-trace: X = vs - V, g = gamma*(1-done)*c),
// so the time axis is split into C chunks.  Block = 32 env lanes x C chunk warps
// x (8/C) env groups:
// every load is a coalesced 128 B row segment.  Pass 1 composes each chunk's
// affine map (P, Q); the C maps are folded through shared memory to give each
// chunk its incoming carry; pass 2 re-sweeps the chunk (L1/L2-hot) and writes.
// With large N (one wave is already full) C = 1 and pass 1 disappears.
// Arithmetic is float64 like the reference (R:algos/estimators.py:45-49);
// storage is float32 values/rewards + uint8 flags (22 B/elem for GAE).
#include <initializer_list>

#include "common.cuh"

namespace ul {
namespace {

constexpr int kWarps = 8;  // warps per block = chunks x env groups

struct GaeArgs {
  const float* r;
  const float* v;
  const uint8_t* term;
  const uint8_t* trunc;
  const float* tv;  // nullable
  const float* boot;
  int64_t T, N;
  double gamma, lam;
  float* adv;
  float* ret;
};

// next-state value per R:algos/estimators.py:15-26
__device__ __forceinline__ double next_value(const float* v, const float* boot, const float* tv,
                                             bool trunc, int64_t t, int64_t T, int64_t N,
                                             int64_t n) {
  if (tv != nullptr && trunc) return (double)tv[t * N + n];
  return t + 1 < T ? (double)v[(t + 1) * N + n] : (double)boot[n];
}

__global__ void gae_kernel(GaeArgs a) {
  __shared__ double sP[kWarps][32];
  __shared__ double sQ[kWarps][32];
  const int lane = threadIdx.x, chunk = threadIdx.y, C = blockDim.y;
  const int grp = threadIdx.z, G = blockDim.z;
  const int64_t n = ((int64_t)blockIdx.x * G + grp) * 32 + lane;
  const bool active = n < a.N;
  const int64_t L = (a.T + C - 1) / C;
  const int64_t t0 = chunk * L;
  const int64_t t1 = t0 + L < a.T ? t0 + L : a.T;
  const double gl = a.gamma * a.lam;

  double carry = 0.0;
  if (C > 1) {
    double P = 0.0, Q = 1.0;
    if (active) {
      for (int64_t t = t1 - 1; t >= t0; --t) {
        const int64_t o = t * a.N + n;
        const bool te = a.term[o] != 0, tr = a.trunc[o] != 0;
        const double nv = next_value(a.v, a.boot, a.tv, tr, t, a.T, a.N, n);
        const double d = (double)a.r[o] + (te ? 0.0 : a.gamma * nv) - (double)a.v[o];
        const double g = (te || tr) ? 0.0 : gl;
        P = d + g * P;
        Q = g * Q;
      }
    }
    sP[grp * C + chunk][lane] = P;
    sQ[grp * C + chunk][lane] = Q;
    __syncthreads();
    for (int j = C - 1; j > chunk; --j) carry = sP[grp * C + j][lane] + sQ[grp * C + j][lane] * carry;
  }
  if (!active) return;
  for (int64_t t = t1 - 1; t >= t0; --t) {
    const int64_t o = t * a.N + n;
    const bool te = a.term[o] != 0, tr = a.trunc[o] != 0;
    const double nv = next_value(a.v, a.boot, a.tv, tr, t, a.T, a.N, n);
    const double vt = (double)a.v[o];
    const double d = (double)a.r[o] + (te ? 0.0 : a.gamma * nv) - vt;
    carry = d + ((te || tr) ? 0.0 : gl) * carry;
    a.adv[o] = (float)carry;
    a.ret[o] = (float)(carry + vt);
  }
}

struct VtArgs {
  const float* bl;
  const float* tl;
  const float* r;
  const float* v;
  const uint8_t* term;
  const uint8_t* trunc;  // nullable -> all false
  const float* tv;       // nullable
  const float* boot;
  int64_t T, N;
  double gamma, rho_bar, c_bar;
  float* vs;
  float* pg;
};

__global__ void vtrace_kernel(VtArgs a) {
  __shared__ double sP[kWarps][32];
  __shared__ double sQ[kWarps][32];
  const int lane = threadIdx.x, chunk = threadIdx.y, C = blockDim.y;
  const int grp = threadIdx.z, G = blockDim.z;
  const int64_t n = ((int64_t)blockIdx.x * G + grp) * 32 + lane;
  const bool active = n < a.N;
  const int64_t L = (a.T + C - 1) / C;
  const int64_t t0 = chunk * L;
  const int64_t t1 = t0 + L < a.T ? t0 + L : a.T;

  // carry X_{t+1} = vs_{t+1} - V_{t+1}
  double carry = 0.0;
  if (C > 1) {
    double P = 0.0, Q = 1.0;
    if (active) {
      for (int64_t t = t1 - 1; t >= t0; --t) {
        const int64_t o = t * a.N + n;
        const bool te = a.term[o] != 0, tr = a.trunc ? a.trunc[o] != 0 : false;
        const double ratio = exp((double)a.tl[o] - (double)a.bl[o]);
        const double rho = fmin(a.rho_bar, ratio), c = fmin(a.c_bar, ratio);
        const double nv = next_value(a.v, a.boot, a.tv, tr, t, a.T, a.N, n);
        const double d = rho * ((double)a.r[o] + (te ? 0.0 : a.gamma * nv) - (double)a.v[o]);
        const double g = (te || tr) ? 0.0 : a.gamma * c;
        P = d + g * P;
        Q = g * Q;
      }
    }
    sP[grp * C + chunk][lane] = P;
    sQ[grp * C + chunk][lane] = Q;
    __syncthreads();
    for (int j = C - 1; j > chunk; --j) carry = sP[grp * C + j][lane] + sQ[grp * C + j][lane] * carry;
  }
  if (!active) return;
  // vs_{t+1}: bootstrap at the horizon, otherwise X_{t+1} + V_{t+1}
  for (int64_t t = t1 - 1; t >= t0; --t) {
    const int64_t o = t * a.N + n;
    const bool te = a.term[o] != 0, tr = a.trunc ? a.trunc[o] != 0 : false;
    const bool done = te || tr;
    const double ratio = exp((double)a.tl[o] - (double)a.bl[o]);
    const double rho = fmin(a.rho_bar, ratio), c = fmin(a.c_bar, ratio);
    const double vt = (double)a.v[o];
    const double v_next_raw = t + 1 < a.T ? (double)a.v[o + a.N] : (double)a.boot[n];
    const double nv = (a.tv != nullptr && tr) ? (double)a.tv[o] : v_next_raw;
    const double vs_next = t + 1 < a.T ? carry + v_next_raw : (double)a.boot[n];
    const double base = (double)a.r[o] - vt;
    const double d = rho * (base + (te ? 0.0 : a.gamma * nv));
    carry = d + (done ? 0.0 : a.gamma * c) * carry;
    a.vs[o] = (float)(carry + vt);
    const double w = done ? nv : vs_next;
    a.pg[o] = (float)(rho * (base + (te ? 0.0 : a.gamma * w)));
  }
}

// Wide-N fast path (one wave of 148 SMs is already full): 4 envs per thread
// with 16-byte loads, V(s_{t+1}) carried in registers from the previous step
// (one value load per element), so a thread streams exactly the algorithmic
// 22 B (GAE) / 30 B (V-trace) per element.
__device__ __forceinline__ float4 ld4(const float* p) { return __ldg(reinterpret_cast<const float4*>(p)); }
__device__ __forceinline__ uchar4 ldb4(const uint8_t* p) {
  return __ldg(reinterpret_cast<const uchar4*>(p));
}
__device__ __forceinline__ float f4(const float4& v, int i) {
  return i == 0 ? v.x : (i == 1 ? v.y : (i == 2 ? v.z : v.w));
}
__device__ __forceinline__ uint8_t b4(const uchar4& v, int i) {
  return i == 0 ? v.x : (i == 1 ? v.y : (i == 2 ? v.z : v.w));
}

__global__ void __launch_bounds__(256) gae_vec4_kernel(GaeArgs a) {
  const int64_t n4 = a.N / 4;
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= n4) return;
  const int64_t n = q * 4;
  const double gl = a.gamma * a.lam;
  double carry[4] = {0.0, 0.0, 0.0, 0.0};
  float4 vnext = ld4(a.boot + n);  // V(s_T) = bootstrap
  for (int64_t t = a.T - 1; t >= 0; --t) {
    const int64_t o = t * a.N + n;
    const float4 r = ld4(a.r + o), v = ld4(a.v + o);
    const uchar4 te = ldb4(a.term + o), tr = ldb4(a.trunc + o);
    float4 tv = make_float4(0.f, 0.f, 0.f, 0.f);
    if (a.tv) tv = ld4(a.tv + o);
    float4 adv, ret;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const bool bte = b4(te, i) != 0, btr = b4(tr, i) != 0;
      const double nv = (a.tv && btr) ? (double)f4(tv, i) : (double)f4(vnext, i);
      const double vt = (double)f4(v, i);
      const double d = (double)f4(r, i) + (bte ? 0.0 : a.gamma * nv) - vt;
      carry[i] = d + ((bte || btr) ? 0.0 : gl) * carry[i];
      reinterpret_cast<float*>(&adv)[i] = (float)carry[i];
      reinterpret_cast<float*>(&ret)[i] = (float)(carry[i] + vt);
    }
    *reinterpret_cast<float4*>(a.adv + o) = adv;
    *reinterpret_cast<float4*>(a.ret + o) = ret;
    vnext = v;
  }
}

__global__ void __launch_bounds__(256) vtrace_vec4_kernel(VtArgs a) {
  const int64_t n4 = a.N / 4;
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= n4) return;
  const int64_t n = q * 4;
  double carry[4] = {0.0, 0.0, 0.0, 0.0};  // X_{t+1} = vs_{t+1} - V_{t+1}
  const float4 boot = ld4(a.boot + n);
  float4 vnext = boot;
  for (int64_t t = a.T - 1; t >= 0; --t) {
    const int64_t o = t * a.N + n;
    const float4 bl = ld4(a.bl + o), tl = ld4(a.tl + o), r = ld4(a.r + o), v = ld4(a.v + o);
    const uchar4 te = ldb4(a.term + o);
    uchar4 tr = make_uchar4(0, 0, 0, 0);
    if (a.trunc) tr = ldb4(a.trunc + o);
    float4 tv = make_float4(0.f, 0.f, 0.f, 0.f);
    if (a.tv) tv = ld4(a.tv + o);
    float4 vs, pg;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const bool bte = b4(te, i) != 0, btr = b4(tr, i) != 0, done = bte || btr;
      const double ratio = exp((double)f4(tl, i) - (double)f4(bl, i));
      const double rho = fmin(a.rho_bar, ratio), c = fmin(a.c_bar, ratio);
      const double vt = (double)f4(v, i);
      const double v_next_raw = (double)f4(vnext, i);
      const double nv = (a.tv && btr) ? (double)f4(tv, i) : v_next_raw;
      const double vs_next = t + 1 < a.T ? carry[i] + v_next_raw : (double)f4(boot, i);
      const double base = (double)f4(r, i) - vt;
      const double d = rho * (base + (bte ? 0.0 : a.gamma * nv));
      carry[i] = d + (done ? 0.0 : a.gamma * c) * carry[i];
      reinterpret_cast<float*>(&vs)[i] = (float)(carry[i] + vt);
      const double w = done ? nv : vs_next;
      reinterpret_cast<float*>(&pg)[i] = (float)(rho * (base + (bte ? 0.0 : a.gamma * w)));
    }
    *reinterpret_cast<float4*>(a.vs + o) = vs;
    *reinterpret_cast<float4*>(a.pg + o) = pg;
    vnext = v;
  }
}

bool vec4_ok(int64_t N, std::initializer_list<const void*> ptrs) {
  if (N % 4) return false;
  for (const void* p : ptrs)
    if (p && ((uintptr_t)p & 15)) return false;
  return true;
}

// Chunks along T so that the grid covers ~2 waves of 148 SMs even for small N.
int pick_chunks(int64_t T, int64_t N) {
  const int64_t env_warps = ceil_div(N, 32);
  int C = 1;
  while (C < kWarps && C * 2 <= T && env_warps * C < 2 * kNumSMs * 16) C *= 2;
  return C;
}

dim3 scan_block(int C) { return dim3(32, C, kWarps / C); }
dim3 scan_grid(int64_t N, int C) { return dim3((unsigned)ceil_div(N, 32 * (kWarps / C))); }

}  // namespace
}  // namespace ul

extern "C" int ul_gae_f32(const float* rewards, const float* values, const uint8_t* terminated,
                          const uint8_t* truncated, const float* truncation_values,
                          const float* bootstrap, int64_t T, int64_t N, double gamma, double lam,
                          float* adv, float* ret, void* stream) {
  UL_CHECK_ARG(T >= 0 && N >= 0, "gae: negative shape (%lld, %lld)", (long long)T, (long long)N);
  if (T == 0 || N == 0) return UL_OK;
  UL_CHECK_ARG(rewards && values && terminated && truncated && bootstrap && adv && ret,
               "gae: null pointer");
  ul::GaeArgs a{rewards, values, terminated, truncated, truncation_values, bootstrap,
                T, N, gamma, lam, adv, ret};
  const int C = ul::pick_chunks(T, N);
  if (C == 1 && ul::vec4_ok(N, {rewards, values, terminated, truncated, truncation_values,
                                bootstrap, adv, ret})) {
    ul::gae_vec4_kernel<<<(unsigned)ul::ceil_div(N / 4, 256), 256, 0, ul::as_stream(stream)>>>(a);
    return ul::check_launch("gae_vec4_kernel");
  }
  ul::gae_kernel<<<ul::scan_grid(N, C), ul::scan_block(C), 0, ul::as_stream(stream)>>>(a);
  return ul::check_launch("gae_kernel");
}

extern "C" int ul_vtrace_f32(const float* behavior_logp, const float* target_logp,
                             const float* rewards, const float* values,
                             const uint8_t* terminated, const uint8_t* truncated,
                             const float* truncation_values, const float* bootstrap, int64_t T,
                             int64_t N, double gamma, double rho_bar, double c_bar, float* vs,
                             float* pg_adv, void* stream) {
  UL_CHECK_ARG(T >= 0 && N >= 0, "vtrace: negative shape");
  if (T == 0 || N == 0) return UL_OK;
  UL_CHECK_ARG(behavior_logp && target_logp && rewards && values && terminated && bootstrap &&
                   vs && pg_adv,
               "vtrace: null pointer");
  ul::VtArgs a{behavior_logp, target_logp, rewards, values, terminated, truncated,
               truncation_values, bootstrap, T, N, gamma, rho_bar, c_bar, vs, pg_adv};
  const int C = ul::pick_chunks(T, N);
  if (C == 1 && ul::vec4_ok(N, {behavior_logp, target_logp, rewards, values, terminated,
                                truncated, truncation_values, bootstrap, vs, pg_adv})) {
    ul::vtrace_vec4_kernel<<<(unsigned)ul::ceil_div(N / 4, 256), 256, 0,
                             ul::as_stream(stream)>>>(a);
    return ul::check_launch("vtrace_vec4_kernel");
  }
  ul::vtrace_kernel<<<ul::scan_grid(N, C), ul::scan_block(C), 0, ul::as_stream(stream)>>>(a);
  return ul::check_launch("vtrace_kernel");
}
