// Fused PPO output stage: both networks' skinny output layers (forward and
// backward) around the K9 loss head, in one kernel per minibatch step.
//
// Replaces, per minibatch row, the chain
//   skinny_fwd(actor head) -> skinny_fwd(critic head) -> ppo_head
//   -> skinny_bwd(actor head) -> skinny_bwd(critic head)
// i.e. R:tensornet/mlp.py:165 (output layer forward) for the actor mean and
// the critic value, R:algos/ppo.py:70-129 (ppo_loss_and_grads: Gaussian
// log-prob, clipped surrogate, clipped value loss, dmean / dv, dlog_std) and
// R:tensornet/mlp.py:192-197 (output layer backward: dW, db, and the hidden
// gradient dh = (dout W) * elu'(h) of the layer below).  Every quantity is
// row-local except the parameter gradients, so one 64-row tile of the two
// last hidden activations h_a, h_c is read once (cp.async into shared
// memory) and everything else happens on chip:
//   mean = h_a W_a^T + b_a, v = h_c w_c + b_c              (fp32, 4 threads/row)
//   loss math of K9 in float64 on one thread per row       (reference dtype)
//   dh_a = (dmean W_a) * elu'(h_a), dh_c = dv w_c * elu'(h_c) -> HBM (bf16 rows)
//   block partials [dW_a | db_a | colsum(dh_a)], [dw_c | db_c | colsum(dh_c)]
//   block partials of [pol, val, kl, dlog_std] -> last-CTA fixed-order fold
// The parameter-gradient partials are reduced later (fixed order) together
// with the deferred dW reductions of the backward pass.
#include <cuda_bf16.h>

#include "learner.cuh"

namespace ul {
namespace {

constexpr double kLog2PiF = 1.8378770664093453;
constexpr int kFRows = 64, kFThr = 256, kFWarps = kFThr / 32;
constexpr int kFMaxK = 256;  // widest last hidden layer handled (one staged chunk)

template <typename T>
__device__ __forceinline__ float4 fld4(const T* p);
template <>
__device__ __forceinline__ float4 fld4<float>(const float* p) {
  return *reinterpret_cast<const float4*>(p);
}
template <>
__device__ __forceinline__ float4 fld4<__nv_bfloat16>(const __nv_bfloat16* p) {
  const uint2 u = *reinterpret_cast<const uint2*>(p);
  return make_float4(__uint_as_float(u.x << 16), __uint_as_float(u.x & 0xFFFF0000u),
                     __uint_as_float(u.y << 16), __uint_as_float(u.y & 0xFFFF0000u));
}
template <typename T>
__device__ __forceinline__ void fst4(T* p, float4 v);
template <>
__device__ __forceinline__ void fst4<float>(float* p, float4 v) {
  *reinterpret_cast<float4*>(p) = v;
}
template <>
__device__ __forceinline__ void fst4<__nv_bfloat16>(__nv_bfloat16* p, float4 v) {
  __nv_bfloat162 a = __floats2bfloat162_rn(v.x, v.y), b = __floats2bfloat162_rn(v.z, v.w);
  uint2 u;
  u.x = *reinterpret_cast<uint32_t*>(&a);
  u.y = *reinterpret_cast<uint32_t*>(&b);
  *reinterpret_cast<uint2*>(p) = u;
}

__device__ __forceinline__ void cpa16(void* sdst, const void* gsrc, bool valid) {
  const uint32_t s = (uint32_t)__cvta_generic_to_shared(sdst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gsrc),
               "r"(valid ? 16 : 0)
               : "memory");
}

// element pitch of a staged row of k columns: 16-byte rows + 16 B pad (banks)
template <typename T>
__host__ __device__ constexpr int fpitch(int k) {
  return ((k * (int)sizeof(T) + 15) / 16 * 16 + 16) / (int)sizeof(T);
}

__host__ __device__ inline int rup8(int k) { return (k + 7) / 8 * 8; }

template <typename TH>
__host__ __device__ inline size_t fused_smem(int Ka, int Kc, int NP) {
  const int ka = rup8(Ka), kc = rup8(Kc);
  return (size_t)kFRows * fpitch<TH>(ka) * sizeof(TH) + (size_t)kFRows * fpitch<TH>(kc) * sizeof(TH) +
         (size_t)NP * fpitch<float>(ka) * 4 + (size_t)fpitch<float>(kc) * 4 +
         (size_t)kFRows * (NP + 1) * 4 + (size_t)kFRows * 4 + (size_t)kFWarps * (ka + kc) * 4;
}

template <typename TH>
__device__ __forceinline__ void stage_rows(const TH* __restrict__ h, int64_t ldh, int64_t M,
                                           int64_t r0, int k, TH* sh, int P) {
  constexpr int kE = 16 / (int)sizeof(TH);
  const int per_row = (k + kE - 1) / kE;
  for (int e = threadIdx.x; e < kFRows * per_row; e += kFThr) {
    const int rr = e / per_row, u = e - rr * per_row;
    const int64_t gr = r0 + rr;
    const bool ok = gr < M;
    cpa16(sh + rr * P + u * kE, h + (ok ? gr : 0) * ldh + u * kE, ok);
  }
}

// W [N, K] (reference row-major, pitch K) -> sw rows of pitch PW, zero rows
// N..NP-1 and columns K..KP-1; all loads issued before the stores
__device__ __forceinline__ void stage_wt(const float* __restrict__ W, int K, int N, int NP, int KP,
                                         float* sw, int PW) {
  const int total = NP * KP;
  for (int base = threadIdx.x; base < total; base += kFThr * 8) {
    float v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = base + u * kFThr;
      const int j = e / KP, c = e - j * KP;
      v[u] = (e < total && c < K && j < N) ? __ldg(W + (int64_t)j * K + c) : 0.f;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = base + u * kFThr;
      const int j = e / KP, c = e - j * KP;
      if (e < total) sw[j * PW + c] = v[u];
    }
  }
}

template <typename TH, int NP>
__global__ void __launch_bounds__(kFThr, 3) ppo_fused_kernel(const __grid_constant__ PpoFusedArgs f) {
  extern __shared__ __align__(16) uint8_t smem[];
  constexpr int NJ = (NP + 3) / 4;  // action dims per lane (j = q + 4m)
  const PpoHeadArgs& a = f.h;
  const int Ka = f.Ka, Kc = f.Kc, A = a.A, nq = 3 + A;
  const int ka = rup8(Ka), kc = rup8(Kc);
  const int Pa = fpitch<TH>(ka), Pc = fpitch<TH>(kc);
  const int PWa = fpitch<float>(ka), PWc = fpitch<float>(kc);
  TH* sha = reinterpret_cast<TH*>(smem);
  TH* shc = sha + kFRows * Pa;
  float* swa = reinterpret_cast<float*>(shc + kFRows * Pc);
  float* swc = swa + NP * PWa;
  float* sg = swc + PWc;                // [64][NP + 1] dmean
  float* sgv = sg + kFRows * (NP + 1);  // [64] dv
  float* sca = sgv + kFRows;            // [8 warps][ka] per-warp column sums of dh_a
  float* scc = sca + kFWarps * ka;      // [8 warps][kc] of dh_c
  __shared__ double s_ls[UL_MAX_ACT], s_isd[UL_MAX_ACT];
  __shared__ double red[kFWarps][3 + UL_MAX_ACT];
  __shared__ double s_lsum;
  __shared__ float s_b[UL_MAX_ACT + 1];

  const int t = threadIdx.x, lane = t & 31, w = t >> 5, r = t >> 2, q = t & 3;
  const int64_t r0 = (int64_t)blockIdx.x * kFRows;
  const int64_t M = a.n_local;
  const int64_t gr = r0 + r;
  const bool row_ok = gr < M;
  pdl_trigger();
  pdl_wait();
  // ---- one memory round trip: both h tiles (cp.async), W, biases, row data
  stage_rows<TH>(reinterpret_cast<const TH*>(f.ha), f.ldha, M, r0, ka, sha, Pa);
  stage_rows<TH>(reinterpret_cast<const TH*>(f.hc), f.ldhc, M, r0, kc, shc, Pc);
  asm volatile("cp.async.commit_group;" ::: "memory");
  stage_wt(f.Wa, Ka, A, NP, ka, swa, PWa);
  stage_wt(f.Wc, Kc, 1, 1, kc, swc, PWc);
  for (int j = t; j < A; j += kFThr) {
    const double ls = (double)a.log_std[j];
    s_ls[j] = ls;
    s_isd[j] = exp(-ls);
    s_b[j] = f.ba[j];
  }
  if (t == 0) s_b[UL_MAX_ACT] = f.bc[0];
  // this lane's action dims j = q + 4m and the row scalars
  float act[NJ];
#pragma unroll
  for (int m = 0; m < NJ; ++m) {
    const int j = q + 4 * m;
    act[m] = (row_ok && j < A) ? a.act[gr * a.ld_act + j] : 0.f;
  }
  double blogp = 0.0, advr = 0.0, ret = 0.0, oldv = 0.0;
  if (row_ok) {
    blogp = (double)a.blogp[gr];
    advr = (double)a.adv[gr];
    ret = (double)a.ret[gr];
    oldv = (double)a.oldv[gr];
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  __syncthreads();
  if (t == 0) {
    double s = 0.0;
    for (int j = 0; j < A; ++j) s += s_ls[j];
    s_lsum = s;
  }
  // ---- forward: mean (A outputs) and v, 4 threads per row (column groups
  // c = 4q + 16i), the row's partial sums meet through two lane shuffles
  float accA[NP], accC = 0.f;
#pragma unroll
  for (int j = 0; j < NP; ++j) accA[j] = 0.f;
  {
    const TH* hr = sha + r * Pa;
    for (int c = 4 * q; c < ka; c += 16) {
      const float4 hv = fld4<TH>(hr + c);  // columns >= Ka: W is zero there
#pragma unroll
      for (int j = 0; j < NP; ++j) {
        const float4 wv = *reinterpret_cast<const float4*>(swa + j * PWa + c);
        accA[j] = fmaf(hv.x, wv.x, fmaf(hv.y, wv.y, fmaf(hv.z, wv.z, fmaf(hv.w, wv.w, accA[j]))));
      }
    }
    const TH* hc = shc + r * Pc;
    for (int c = 4 * q; c < kc; c += 16) {
      const float4 hv = fld4<TH>(hc + c);
      const float4 wv = *reinterpret_cast<const float4*>(swc + c);
      accC = fmaf(hv.x, wv.x, fmaf(hv.y, wv.y, fmaf(hv.z, wv.z, fmaf(hv.w, wv.w, accC))));
    }
  }
#pragma unroll
  for (int j = 0; j < NP; ++j) {
    accA[j] += __shfl_xor_sync(0xffffffffu, accA[j], 1);
    accA[j] += __shfl_xor_sync(0xffffffffu, accA[j], 2);
  }
  accC += __shfl_xor_sync(0xffffffffu, accC, 1);
  accC += __shfl_xor_sync(0xffffffffu, accC, 2);
  __syncthreads();  // s_lsum
  // ---- K9 loss head in float64 (as ppo_head_kernel): the row's four lanes
  // split the action dims, then each evaluates the row scalars
  double zpart = 0.0, z[NJ];
#pragma unroll
  for (int m = 0; m < NJ; ++m) {
    const int j = q + 4 * m;
    float am = 0.f;
#pragma unroll
    for (int jj = 0; jj < NP; ++jj)
      if (jj == j) am = accA[jj];  // (register select, no local memory)
    z[m] = 0.0;
    if (j < A) {
      const double mean = (double)(am + s_b[j]);
      z[m] = ((double)act[m] - mean) * s_isd[j];
      zpart += z[m] * z[m];
    }
  }
  zpart += __shfl_xor_sync(0xffffffffu, zpart, 1);
  zpart += __shfl_xor_sync(0xffffffffu, zpart, 2);
  double pol = 0.0, val = 0.0, kl = 0.0, dlogp = 0.0, dv = 0.0;
  if (row_ok) {
    const double adv_mean = a.adv_stats ? a.adv_stats[0] : 0.0;
    const double adv_den = a.adv_stats ? a.adv_stats[1] + 1e-8 : 1.0;
    const double logp = -s_lsum - A * (0.5 * kLog2PiF) - 0.5 * zpart;
    const double adv = (advr - adv_mean) / adv_den;
    const double ratio = exp(logp - blogp);
    const double s1 = ratio * adv;
    const double rc = fmin(fmax(ratio, 1.0 - a.clip), 1.0 + a.clip);
    const double s2 = rc * adv;
    pol = fmin(s1, s2);
    dlogp = (s1 <= s2) ? -adv * ratio / a.n_global : 0.0;
    kl = blogp - logp;
    const double v = (double)(accC + s_b[UL_MAX_ACT]);
    if (a.clipped_v) {
      const double vc = oldv + fmin(fmax(v - oldv, -a.clip), a.clip);
      const double lu = (v - ret) * (v - ret), lc = (vc - ret) * (vc - ret);
      val = fmax(lu, lc);
      dv = lu >= lc ? 2.0 * (v - ret) / a.n_global : 0.0;
    } else {
      val = (v - ret) * (v - ret);
      dv = 2.0 * (v - ret) / a.n_global;
    }
  }
  double dls[NJ];
#pragma unroll
  for (int m = 0; m < NJ; ++m) {
    const int j = q + 4 * m;
    dls[m] = 0.0;
    if (j < A) {
      sg[r * (NP + 1) + j] = (float)(dlogp * z[m] * s_isd[j]);
      dls[m] = dlogp * (z[m] * z[m] - 1.0);
    }
  }
  if (q == 0) sgv[r] = (float)(dv * a.vcoef);
  // row terms -> per-warp sums: the scalars once per row (lane q == 0), the
  // dlog_std terms over the warp's 8 rows (lanes with equal q), then lanes 0..3
  {
    const double one = q == 0 ? 1.0 : 0.0;
    double v = warp_sum(pol * one);
    if (lane == 0) red[w][0] = v;
    v = warp_sum(val * one);
    if (lane == 0) red[w][1] = v;
    v = warp_sum(kl * one);
    if (lane == 0) red[w][2] = v;
#pragma unroll
    for (int m = 0; m < NJ; ++m) {
      double d = dls[m];
      d += __shfl_xor_sync(0xffffffffu, d, 4);
      d += __shfl_xor_sync(0xffffffffu, d, 8);
      d += __shfl_xor_sync(0xffffffffu, d, 16);
      const int j = q + 4 * m;
      if (lane < 4 && j < A) red[w][3 + j] = d;
    }
  }
  __syncthreads();  // sg / sgv ready
  // ---- hidden gradients of the layers below (the next GEMM's rows) and their
  // column sums over the warp's 8 rows (lanes with equal q: xor 4, 8, 16)
  {
    float g[NP];
#pragma unroll
    for (int j = 0; j < NP; ++j) g[j] = sg[r * (NP + 1) + j];
    const float gv = sgv[r];
    TH* da = reinterpret_cast<TH*>(f.dha) + gr * f.lddha;
    TH* dc = reinterpret_cast<TH*>(f.dhc) + gr * f.lddhc;
    for (int c = 4 * q; c < ka; c += 16) {
      float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int j = 0; j < NP; ++j) {
        const float4 wv = *reinterpret_cast<const float4*>(swa + j * PWa + c);
        s.x = fmaf(g[j], wv.x, s.x);
        s.y = fmaf(g[j], wv.y, s.y);
        s.z = fmaf(g[j], wv.z, s.z);
        s.w = fmaf(g[j], wv.w, s.w);
      }
      const float4 hv = fld4<TH>(sha + r * Pa + c);
      s.x *= elu_grad_from_act(hv.x);
      s.y *= elu_grad_from_act(hv.y);
      s.z *= elu_grad_from_act(hv.z);
      s.w *= elu_grad_from_act(hv.w);
      if (!row_ok) s = make_float4(0.f, 0.f, 0.f, 0.f);
      if (row_ok) {
        if (c + 4 <= Ka) {
          fst4<TH>(da + c, s);
        } else {
          const float sv[4] = {s.x, s.y, s.z, s.w};
          for (int i = 0; c + i < Ka; ++i) da[c + i] = (TH)sv[i];
        }
      }
      if (f.csa) {
#pragma unroll
        for (int o = 4; o <= 16; o <<= 1) {
          s.x += __shfl_xor_sync(0xffffffffu, s.x, o);
          s.y += __shfl_xor_sync(0xffffffffu, s.y, o);
          s.z += __shfl_xor_sync(0xffffffffu, s.z, o);
          s.w += __shfl_xor_sync(0xffffffffu, s.w, o);
        }
        if (lane < 4) *reinterpret_cast<float4*>(sca + w * ka + c) = s;
      }
    }
    for (int c = 4 * q; c < kc; c += 16) {
      const float4 wv = *reinterpret_cast<const float4*>(swc + c);
      const float4 hv = fld4<TH>(shc + r * Pc + c);
      float4 s = make_float4(gv * wv.x * elu_grad_from_act(hv.x), gv * wv.y * elu_grad_from_act(hv.y),
                             gv * wv.z * elu_grad_from_act(hv.z), gv * wv.w * elu_grad_from_act(hv.w));
      if (!row_ok) s = make_float4(0.f, 0.f, 0.f, 0.f);
      if (row_ok) {
        if (c + 4 <= Kc) {
          fst4<TH>(dc + c, s);
        } else {
          const float sv[4] = {s.x, s.y, s.z, s.w};
          for (int i = 0; c + i < Kc; ++i) dc[c + i] = (TH)sv[i];
        }
      }
      if (f.csc) {
#pragma unroll
        for (int o = 4; o <= 16; o <<= 1) {
          s.x += __shfl_xor_sync(0xffffffffu, s.x, o);
          s.y += __shfl_xor_sync(0xffffffffu, s.y, o);
          s.z += __shfl_xor_sync(0xffffffffu, s.z, o);
          s.w += __shfl_xor_sync(0xffffffffu, s.w, o);
        }
        if (lane < 4) *reinterpret_cast<float4*>(scc + w * kc + c) = s;
      }
    }
  }
  __syncthreads();  // sca / scc complete
  // ---- block partials of the parameter gradients (fixed order over rows)
  float* pa = f.parta + (int64_t)blockIdx.x * f.plena;
  float* pc = f.partc + (int64_t)blockIdx.x * f.plenc;
  {
    const int g4 = ka / 4;
    for (int pr = t; pr < g4 * A; pr += kFThr) {
      const int j = pr / g4, c = 4 * (pr - j * g4);
      float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 8
      for (int rr = 0; rr < kFRows; ++rr) {
        const float d = sg[rr * (NP + 1) + j];
        const float4 hv = fld4<TH>(sha + rr * Pa + c);
        s.x = fmaf(d, hv.x, s.x);
        s.y = fmaf(d, hv.y, s.y);
        s.z = fmaf(d, hv.z, s.z);
        s.w = fmaf(d, hv.w, s.w);
      }
      const float sv[4] = {s.x, s.y, s.z, s.w};
      for (int i = 0; i < 4 && c + i < Ka; ++i) pa[(int64_t)j * Ka + c + i] = sv[i];
    }
    const int g4c = kc / 4;
    for (int c4 = t; c4 < g4c; c4 += kFThr) {
      const int c = 4 * c4;
      float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 8
      for (int rr = 0; rr < kFRows; ++rr) {
        const float d = sgv[rr];
        const float4 hv = fld4<TH>(shc + rr * Pc + c);
        s.x = fmaf(d, hv.x, s.x);
        s.y = fmaf(d, hv.y, s.y);
        s.z = fmaf(d, hv.z, s.z);
        s.w = fmaf(d, hv.w, s.w);
      }
      const float sv[4] = {s.x, s.y, s.z, s.w};
      for (int i = 0; i < 4 && c + i < Kc; ++i) pc[c + i] = sv[i];
    }
    // bias partials
    if (t < A) {
      float s = 0.f;
      for (int rr = 0; rr < kFRows; ++rr) s += sg[rr * (NP + 1) + t];
      pa[(int64_t)A * Ka + t] = s;
    } else if (t == 64) {
      float s = 0.f;
      for (int rr = 0; rr < kFRows; ++rr) s += sgv[rr];
      pc[Kc] = s;
    }
    // column sums of the hidden gradients over the 8 warps (fixed order)
    if (f.csa)
      for (int c = t; c < Ka; c += kFThr) {
        float s = 0.f;
#pragma unroll
        for (int k = 0; k < kFWarps; ++k) s += sca[k * ka + c];
        pa[(int64_t)A * Ka + A + c] = s;
      }
    if (f.csc)
      for (int c = t; c < Kc; c += kFThr) {
        float s = 0.f;
#pragma unroll
        for (int k = 0; k < kFWarps; ++k) s += scc[k * kc + c];
        pc[Kc + 1 + c] = s;
      }
  }
  // ---- loss / dlog_std partials, last CTA folds them in fixed order
  double* part = a.part + (int64_t)blockIdx.x * nq;
  for (int qq = t; qq < nq; qq += kFThr) {
    double s = 0.0;
    for (int k = 0; k < kFWarps; ++k) s += red[k][qq];
    part[qq] = s;
  }
  if (!last_block_ticket(a.ticket, gridDim.x)) return;
  const unsigned nb = gridDim.x;
  for (int q0 = 0; q0 < nq; q0 += kFThr / 8) {
    const int qq = q0 + (t >> 3), l = t & 7;
    double s = 0.0;
    if (qq < nq) {
      for (unsigned b0 = l; b0 < nb; b0 += 64) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const unsigned b = b0 + 8 * u;
          v[u] = b < nb ? a.part[(int64_t)b * nq + qq] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) s += v[u];
      }
    }
    s += __shfl_xor_sync(0xffffffffu, s, 1);
    s += __shfl_xor_sync(0xffffffffu, s, 2);
    s += __shfl_xor_sync(0xffffffffu, s, 4);
    if (qq < nq && l == 0) {
      if (qq < 3) a.loss_out[qq] = (float)s;
      else a.dlogstd_out[qq - 3] = (float)(s + a.ent_coef_add);
    }
  }
}


inline int pad_np(int N) {
  const int sizes[] = {1, 2, 4, 8, 12, 16, 24, 32};
  for (int v : sizes)
    if (N <= v) return v;
  return 0;
}

template <typename TH, int NP>
int launch_np(const PpoFusedArgs& f, cudaStream_t s) {
  const size_t sm = fused_smem<TH>(f.Ka, f.Kc, NP);
  static bool attr = false;
  if (!attr) {
    UL_CUDA(cudaFuncSetAttribute(ppo_fused_kernel<TH, NP>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    attr = true;
  }
  const unsigned blocks = (unsigned)ceil_div(f.h.n_local > 0 ? f.h.n_local : 1, kFRows);
  return launch_pdl("ppo_fused_kernel", ppo_fused_kernel<TH, NP>, dim3(blocks), dim3(kFThr), sm, s,
                    f);
}

template <typename TH>
int launch_t(const PpoFusedArgs& f, cudaStream_t s) {
  switch (pad_np(f.h.A)) {
    case 1: return launch_np<TH, 1>(f, s);
    case 2: return launch_np<TH, 2>(f, s);
    case 4: return launch_np<TH, 4>(f, s);
    case 8: return launch_np<TH, 8>(f, s);
    case 12: return launch_np<TH, 12>(f, s);
    case 16: return launch_np<TH, 16>(f, s);
    case 24: return launch_np<TH, 24>(f, s);
    default: return launch_np<TH, 32>(f, s);
  }
}

}  // namespace

bool ppo_fused_ok(int A, int Ka, int Kc) {
  return A >= 1 && A <= 32 && Ka >= 1 && Ka <= kFMaxK && Kc >= 1 && Kc <= kFMaxK &&
         fused_smem<float>(Ka, Kc, pad_np(A)) <= 200 * 1024;
}

int launch_ppo_fused(const PpoFusedArgs& f, int dtype, ReduceJob* ja, ReduceJob* jc,
                     cudaStream_t s) {
  UL_CHECK_ARG(ppo_fused_ok(f.h.A, f.Ka, f.Kc), "ppo fused head: unsupported shape");
  UL_TRY(dtype == kBf16 ? launch_t<__nv_bfloat16>(f, s) : launch_t<float>(f, s));
  const int64_t nblk = ceil_div(f.h.n_local > 0 ? f.h.n_local : 1, kFRows);
  // fixed-order reductions of the block partials, folded into the caller's
  // next reduction launch: [dW | db | colsum(dh)] per network
  *ja = ReduceJob{};
  ja->src = f.parta;
  ja->nz = (int)nblk;
  ja->kind = 1;
  ja->len = f.plena;
  ja->n0 = (int64_t)f.h.A * f.Ka;
  ja->o0 = f.gwa;
  ja->n1 = f.h.A;
  ja->o1 = f.gba;
  ja->n2 = f.csa ? f.Ka : 0;
  ja->o2 = f.gcsa;
  *jc = ReduceJob{};
  jc->src = f.partc;
  jc->nz = (int)nblk;
  jc->kind = 1;
  jc->len = f.plenc;
  jc->n0 = f.Kc;
  jc->o0 = f.gwc;
  jc->n1 = 1;
  jc->o1 = f.gbc;
  jc->n2 = f.csc ? f.Kc : 0;
  jc->o2 = f.gcsc;
  return UL_OK;
}

}  // namespace ul
