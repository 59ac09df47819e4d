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


// ---------------------------------------------------------------------------
// Tensor-core variant (bf16 rows, A <= 32, K <= 256).  Two CTA roles per
// 64-row tile (grid.y = 2): every quantity of one network's output stage is
// row-local or a column sum over the tile, so the networks never exchange data.
//  actor (y = 0): the three small products on warp-level mma.sync m16n8k16
//    (bf16 in, fp32 accumulate) -- mean = h W^T, dh = dmean W (the dmean
//    fragments re-packed in registers as the A operand) and dW = dmean^T h
//    over the tile's rows (ldmatrix.trans feeds h as the column-major B
//    operand) -- around the Gaussian log-prob / clipped surrogate in float64;
//  critic (y = 1): v = h w + b, the clipped value loss, dh = dv w * elu'(h),
//    dw and colsum(dh) on SIMT lanes.
// 4 warps; actor warp w owns rows [16w, 16w + 16) for the row-local phases and
// output columns {8 n : n = w (mod 4)} for dW (no cross-warp dW reduction).
// W_a arrives as the Adam-refreshed bf16 staged copy (cp.async).  Split roles
// halve each CTA's serial chain and shared memory, so the whole grid (2 x 384
// CTAs at cfg2) is resident at once; tile staging loops carry no per-element
// integer division.
constexpr int kMRows = 64, kMThr = 128, kMWarps = 4;

__device__ __forceinline__ void mma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0,
                                         uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, "
      "{%8, %9}, {%0, %1, %2, %3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"((uint32_t)__cvta_generic_to_shared(p)));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t (&r)[4], const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"((uint32_t)__cvta_generic_to_shared(p)));
}
__device__ __forceinline__ uint32_t pk_bf16(float lo, float hi) {
  __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&h);
}
__device__ __forceinline__ float2 up_bf16(uint32_t u) {
  return make_float2(__uint_as_float(u << 16), __uint_as_float(u & 0xFFFF0000u));
}

__host__ __device__ inline int rup16(int k) { return (k + 15) / 16 * 16; }
__host__ __device__ inline size_t al16(size_t o) { return (o + 15) / 16 * 16; }

// dynamic smem layouts (bytes) of the two roles
struct ActorSmem {
  int ka, pa, pwa, pdm;
  size_t o_wa, o_dm, o_cs, o_dh, total;
  __host__ __device__ ActorSmem(int Ka, int NJT) {
    ka = rup16(Ka);
    pa = ka + 8;        // bf16 row pitch of the h_a tile (16 B aligned, conflict-free)
    pwa = ka + 8;       // W_a  [NJT*8][pwa] bf16 (B of the forward; .trans: B of dh)
    pdm = kMRows + 8;   // dmean^T [NJT*8][pdm] bf16 (A operand of dW)
    size_t o = (size_t)kMRows * pa * 2;
    o_wa = o;
    o += (size_t)NJT * 8 * pwa * 2;
    o_dm = o;
    o += (size_t)NJT * 8 * pdm * 2;
    o = al16(o);
    o_cs = o;           // colsum(dh_a) [ka], then db_a [warps][32]
    o += (size_t)ka * 4 + (size_t)kMWarps * 32 * 4;
    o = al16(o);
    o_dh = o;           // dh_a tile [kMRows][pa] bf16 (coalesced store + column sums)
    o += (size_t)kMRows * pa * 2;
    total = o;
  }
};
struct CriticSmem {
  int kc, pc;
  size_t o_wc, o_v, o_cr, total;
  __host__ __device__ CriticSmem(int Kc) {
    kc = rup8(Kc);
    pc = kc + 8;
    size_t o = al16((size_t)kMRows * pc * 2);
    o_wc = o;
    o += (size_t)kc * 4;
    o_v = o;            // v (forward) and dv, fp32
    o += (size_t)kMRows * 4 * 2;
    o_cr = o;           // [warps][kc] dw_c, then [warps][kc] colsum(dh_c)
    o += (size_t)2 * kMWarps * kc * 4;
    total = o;
  }
};

// cp.async of rows [0, R) of a bf16 row block (row rr = global row r0 + rr,
// valid while < nvalid; granules of 8 past k, and invalid rows, zero-filled)
// into rows of pitch P.  Thread t owns granule u = t % gt of rows t / gt,
// t / gt + kMThr / gt, ...  (gt = kpad / 8 <= 32).
__device__ __forceinline__ void stage_bf16_rows(const void* g, int64_t ld, int64_t r0,
                                                int64_t nvalid, int R, int k, int kpad,
                                                __nv_bfloat16* s, int P) {
  const int gdat = (k + 7) / 8, gt = kpad / 8;
  const int rstep = kMThr / gt;
  const int t = threadIdx.x;
  if (t >= rstep * gt) return;
  const int u = t % gt;
  const __nv_bfloat16* gb = reinterpret_cast<const __nv_bfloat16*>(g);
  for (int rr = t / gt; rr < R; rr += rstep) {
    const int64_t gr = r0 + rr;
    const bool ok = gr < nvalid && u < gdat;
    cpa16(s + rr * P + u * 8, gb + (ok ? gr * ld + u * 8 : 0), ok);
  }
}

template <int NJT>  // n-tiles of 8 action dims: A <= 8 * NJT (NJT = 2 or 4)
__device__ __forceinline__ void fused_actor(const PpoFusedArgs& f, uint8_t* smem) {
  constexpr int MT = NJT / 2;  // 16-row m tiles of action dims (dW) = k16 steps of dh
  const PpoHeadArgs& a = f.h;
  const int Ka = f.Ka, A = a.A, nq = 3 + A;
  const ActorSmem L(Ka, NJT);
  const int ka = L.ka;
  __nv_bfloat16* sha = reinterpret_cast<__nv_bfloat16*>(smem);
  __nv_bfloat16* swa = reinterpret_cast<__nv_bfloat16*>(smem + L.o_wa);
  __nv_bfloat16* sdm = reinterpret_cast<__nv_bfloat16*>(smem + L.o_dm);
  float* scs = reinterpret_cast<float*>(smem + L.o_cs);  // [ka] colsum(dh_a)
  float* sdb = scs + ka;                                 // [warps][32] db_a
  __nv_bfloat16* sdh = reinterpret_cast<__nv_bfloat16*>(smem + L.o_dh);
  __shared__ double s_ls[UL_MAX_ACT], s_isd[UL_MAX_ACT];
  __shared__ double red[kMWarps][3 + UL_MAX_ACT];
  __shared__ double s_lsum;
  __shared__ float s_b[UL_MAX_ACT];

  const int t = threadIdx.x, lane = t & 31, w = t >> 5, g = lane >> 2, q = lane & 3;
  const int64_t r0 = (int64_t)blockIdx.x * kMRows;
  const int64_t M = a.n_local;
  // ---- h_a tile and the staged bf16 W_a rows (cp.async, zero past A / Ka)
  stage_bf16_rows(f.ha, f.ldha, r0, M, kMRows, Ka, ka, sha, L.pa);
  stage_bf16_rows(f.wba, f.ldwb, 0, A, NJT * 8, Ka, ka, swa, L.pwa);
  asm volatile("cp.async.commit_group;" ::: "memory");
  for (int j = t; j < A; j += kMThr) {
    const double ls = (double)a.log_std[j];
    s_ls[j] = ls;
    s_isd[j] = exp(-ls);
    s_b[j] = f.ba[j];
  }
  // this lane's rows (R0 = 16w + g, R1 = R0 + 8) and action dims
  // j = 8 nt + 2q + {0, 1}: row scalars and actions, loads in flight now
  const int R[2] = {16 * w + g, 16 * w + g + 8};
  bool ok[2];
  float act[2][NJT][2];
  double blogp[2], advr[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int64_t gr = r0 + R[h];
    ok[h] = gr < M;
#pragma unroll
    for (int nt = 0; nt < NJT; ++nt)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int j = 8 * nt + 2 * q + e;
        act[h][nt][e] = (ok[h] && j < A) ? a.act[gr * a.ld_act + j] : 0.f;
      }
    blogp[h] = ok[h] ? (double)a.blogp[gr] : 0.0;
    advr[h] = ok[h] ? (double)a.adv[gr] : 0.0;
  }
  const double adv_mean = a.adv_stats ? a.adv_stats[0] : 0.0;
  const double adv_den = a.adv_stats ? a.adv_stats[1] + 1e-8 : 1.0;
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  __syncthreads();
  if (t == 0) {
    double s = 0.0;
    for (int j = 0; j < A; ++j) s += s_ls[j];
    s_lsum = s;
  }
  // ---- forward on the tensor cores: acc[nt] = h[16 rows] W^T (8 dims)
  float acc[NJT][4];
#pragma unroll
  for (int nt = 0; nt < NJT; ++nt)
#pragma unroll
    for (int e = 0; e < 4; ++e) acc[nt][e] = 0.f;
  for (int kk = 0; kk < ka; kk += 16) {
    uint32_t af[4];
    ldsm_x4(af, sha + (16 * w + (lane & 15)) * L.pa + kk + (lane >> 4) * 8);
#pragma unroll
    for (int nt = 0; nt < NJT; ++nt) {
      const __nv_bfloat16* bp = swa + (8 * nt + g) * L.pwa + kk + 2 * q;
      mma16816(acc[nt], af, *reinterpret_cast<const uint32_t*>(bp),
               *reinterpret_cast<const uint32_t*>(bp + 8));
    }
  }
  __syncthreads();  // s_lsum
  // ---- K9 policy head in float64 (rows R0, R1; the quad of lanes sharing g
  // splits the action dims), as ppo_head_kernel
  double pol = 0.0, kl = 0.0, dls[NJT][2];
#pragma unroll
  for (int nt = 0; nt < NJT; ++nt) dls[nt][0] = dls[nt][1] = 0.0;
  float dm[2][NJT][2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    double z[NJT][2];
    double zp = 0.0;
#pragma unroll
    for (int nt = 0; nt < NJT; ++nt)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int j = 8 * nt + 2 * q + e;
        z[nt][e] = 0.0;
        if (j < A) {
          const double mean = (double)(acc[nt][2 * h + e] + s_b[j]);
          z[nt][e] = ((double)act[h][nt][e] - mean) * s_isd[j];
          zp += z[nt][e] * z[nt][e];
        }
      }
    zp += __shfl_xor_sync(0xffffffffu, zp, 1);
    zp += __shfl_xor_sync(0xffffffffu, zp, 2);
    double dlogp = 0.0;
    if (ok[h]) {
      const double logp = -s_lsum - A * (0.5 * kLog2PiF) - 0.5 * zp;
      const double adv = (advr[h] - adv_mean) / adv_den;
      const double ratio = exp(logp - blogp[h]);
      const double s1 = ratio * adv;
      const double rc = fmin(fmax(ratio, 1.0 - a.clip), 1.0 + a.clip);
      const double s2 = rc * adv;
      if (q == 0) {
        pol += fmin(s1, s2);
        kl += blogp[h] - logp;
      }
      dlogp = (s1 <= s2) ? -adv * ratio / a.n_global : 0.0;
    }
#pragma unroll
    for (int nt = 0; nt < NJT; ++nt)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int j = 8 * nt + 2 * q + e;
        dm[h][nt][e] = 0.f;
        if (j < A) {
          dm[h][nt][e] = (float)(dlogp * z[nt][e] * s_isd[j]);
          dls[nt][e] += dlogp * (z[nt][e] * z[nt][e] - 1.0);
        }
      }
  }
  // dmean^T (bf16) for the dW product; db_a and dlog_std partials of the warp
#pragma unroll
  for (int nt = 0; nt < NJT; ++nt)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int j = 8 * nt + 2 * q + e;
      sdm[j * L.pdm + R[0]] = __float2bfloat16_rn(dm[0][nt][e]);
      sdm[j * L.pdm + R[1]] = __float2bfloat16_rn(dm[1][nt][e]);
      float sb = dm[0][nt][e] + dm[1][nt][e];
      double sl = dls[nt][e];
#pragma unroll
      for (int o = 4; o <= 16; o <<= 1) {
        sb += __shfl_xor_sync(0xffffffffu, sb, o);
        sl += __shfl_xor_sync(0xffffffffu, sl, o);
      }
      if (g == 0) {
        sdb[w * 32 + j] = sb;
        if (j < A) red[w][3 + j] = sl;
      }
    }
  {
    double v = warp_sum(pol);
    if (lane == 0) red[w][0] = v;
    v = warp_sum(kl);
    if (lane == 0) red[w][2] = v;
  }
  // ---- dh_a = (dmean W) * elu'(h_a) on the tensor cores; the dmean
  // fragments, rounded to bf16, are the A operand (k = action dims); results
  // to a shared-memory tile, then coalesced 16-byte stores + column sums
  {
    uint32_t af[MT][4];
#pragma unroll
    for (int m = 0; m < MT; ++m) {
      af[m][0] = pk_bf16(dm[0][2 * m][0], dm[0][2 * m][1]);
      af[m][1] = pk_bf16(dm[1][2 * m][0], dm[1][2 * m][1]);
      af[m][2] = pk_bf16(dm[0][2 * m + 1][0], dm[0][2 * m + 1][1]);
      af[m][3] = pk_bf16(dm[1][2 * m + 1][0], dm[1][2 * m + 1][1]);
    }
    for (int nc = 0; nc < ka / 8; ++nc) {
      float d[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int m = 0; m < MT; ++m) {
        // B (k = action dims, n = columns) = W_a rows transposed by ldmatrix
        uint32_t bf[4];
        ldsm_x4_t(bf, swa + (16 * m + (lane & 15)) * L.pwa + 8 * nc);
        mma16816(d, af[m], bf[0], bf[1]);
      }
      const int c = 8 * nc + 2 * q;
      const float2 h0 = up_bf16(*reinterpret_cast<const uint32_t*>(sha + R[0] * L.pa + c));
      const float2 h1 = up_bf16(*reinterpret_cast<const uint32_t*>(sha + R[1] * L.pa + c));
      d[0] = fmaf(d[0], fminf(h0.x, 0.f), d[0]);
      d[1] = fmaf(d[1], fminf(h0.y, 0.f), d[1]);
      d[2] = fmaf(d[2], fminf(h1.x, 0.f), d[2]);
      d[3] = fmaf(d[3], fminf(h1.y, 0.f), d[3]);
      // (invalid rows: dmean = 0 -> d = 0; columns >= Ka: zero W rows -> 0)
      *reinterpret_cast<uint32_t*>(sdh + R[0] * L.pa + c) = pk_bf16(d[0], d[1]);
      *reinterpret_cast<uint32_t*>(sdh + R[1] * L.pa + c) = pk_bf16(d[2], d[3]);
    }
  }
  __syncthreads();  // sdh, sdm, sdb complete
  {
    const int gk = ka / 8;  // 16-byte granules per row (<= 32)
    const int rstep = kMThr / gk;
    const bool vec = (Ka % 8) == 0 && (f.lddha % 8) == 0;
    if (t < rstep * gk) {
      const int u = t % gk, c = 8 * u;
      for (int rr = t / gk; rr < kMRows; rr += rstep) {
        const int64_t gr = r0 + rr;
        if (gr >= M || c >= Ka) continue;
        __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(f.dha) + gr * f.lddha + c;
        if (vec) {
          *reinterpret_cast<uint4*>(dst) = *reinterpret_cast<const uint4*>(sdh + rr * L.pa + c);
        } else {
          for (int k2 = 0; k2 < 8 && c + k2 < Ka; ++k2) dst[k2] = sdh[rr * L.pa + c + k2];
        }
      }
    }
    // colsum(dh_a) per column over the tile's rows, as the values were stored
    // (bf16): two columns per thread pass, fixed row order
    if (f.csa)
      for (int c2 = 2 * t; c2 < ka; c2 += 2 * kMThr) {
        float s0 = 0.f, s1 = 0.f;
#pragma unroll 8
        for (int rr = 0; rr < kMRows; ++rr) {
          const float2 v = up_bf16(*reinterpret_cast<const uint32_t*>(sdh + rr * L.pa + c2));
          s0 += v.x;
          s1 += v.y;
        }
        scs[c2] = s0;
        scs[c2 + 1] = s1;
      }
  }
  // ---- dW_a partial = dmean^T h over the block's rows (tensor cores): warp
  // w owns output columns 8 nt, nt = w, w + 4, ...
  float* pa = f.parta + (int64_t)blockIdx.x * f.plena;
  for (int nt = w; nt < ka / 8; nt += kMWarps) {
    float d[MT][4];
#pragma unroll
    for (int m = 0; m < MT; ++m)
#pragma unroll
      for (int e = 0; e < 4; ++e) d[m][e] = 0.f;
    for (int kr = 0; kr < kMRows; kr += 16) {
      uint32_t bf[4];
      ldsm_x4_t(bf, sha + (kr + (lane & 15)) * L.pa + 8 * nt);  // (x4: both halves identical)
#pragma unroll
      for (int m = 0; m < MT; ++m) {
        uint32_t af[4];
        const __nv_bfloat16* ap = sdm + (16 * m + g) * L.pdm + kr + 2 * q;
        af[0] = *reinterpret_cast<const uint32_t*>(ap);
        af[1] = *reinterpret_cast<const uint32_t*>(ap + 8 * L.pdm);
        af[2] = *reinterpret_cast<const uint32_t*>(ap + 8);
        af[3] = *reinterpret_cast<const uint32_t*>(ap + 8 * L.pdm + 8);
        mma16816(d[m], af, bf[0], bf[1]);
      }
    }
    const int c = 8 * nt + 2 * q;
#pragma unroll
    for (int m = 0; m < MT; ++m) {
      const int j0 = 16 * m + g, j1 = j0 + 8;
      if (c < Ka) {
        if (j0 < A) {
          pa[(int64_t)j0 * Ka + c] = d[m][0];
          pa[(int64_t)j0 * Ka + c + 1] = d[m][1];
        }
        if (j1 < A) {
          pa[(int64_t)j1 * Ka + c] = d[m][2];
          pa[(int64_t)j1 * Ka + c + 1] = d[m][3];
        }
      }
    }
  }
  __syncthreads();  // scs complete
  // ---- remaining partials in fixed order: db_a, colsum(dh_a)
  if (t < A) {
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < kMWarps; ++k) s += sdb[k * 32 + t];
    pa[(int64_t)A * Ka + t] = s;
  }
  if (f.csa)
    for (int c = t; c < Ka; c += kMThr) pa[(int64_t)A * Ka + A + c] = scs[c];
  // ---- policy-loss / kl / dlog_std partials (slot 1, the value loss, is the
  // critic role's); reduced with the pass's other partials
  float* lp = f.lossp + (int64_t)blockIdx.x * f.lossld;
  for (int qq = t; qq < f.lossld; qq += kMThr) {
    if (qq == 1) continue;
    double v = 0.0;
    if (qq < nq) {
      for (int k = 0; k < kMWarps; ++k) v += red[k][qq];
      if (blockIdx.x == 0 && qq >= 3) v += a.ent_coef_add;
    }
    lp[qq] = (float)v;
  }
}

__device__ __forceinline__ void fused_critic(const PpoFusedArgs& f, uint8_t* smem) {
  const PpoHeadArgs& a = f.h;
  const int Kc = f.Kc;
  const CriticSmem L(Kc);
  const int kc = L.kc;
  __nv_bfloat16* shc = reinterpret_cast<__nv_bfloat16*>(smem);
  float* swc = reinterpret_cast<float*>(smem + L.o_wc);
  float* sdv = reinterpret_cast<float*>(smem + L.o_v) + kMRows;
  float* scrit = reinterpret_cast<float*>(smem + L.o_cr);  // [warps][kc] dw_c, then colsum(dh_c)
  __shared__ double red[kMWarps];
  __shared__ float s_bc;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const int64_t r0 = (int64_t)blockIdx.x * kMRows;
  const int64_t M = a.n_local;
  stage_bf16_rows(f.hc, f.ldhc, r0, M, kMRows, Kc, kc, shc, L.pc);
  asm volatile("cp.async.commit_group;" ::: "memory");
  for (int c = t; c < kc; c += kMThr) swc[c] = c < Kc ? __ldg(f.Wc + c) : 0.f;
  if (t == 0) s_bc = f.bc[0];
  // two threads per row, halves of the columns; the even lane owns the row's loss
  const int row = t >> 1, half = t & 1;
  const int64_t gr = r0 + row;
  const bool ok = gr < M;
  const double ret = ok && !half ? (double)a.ret[gr] : 0.0;
  const double oldv = ok && !half ? (double)a.oldv[gr] : 0.0;
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  __syncthreads();
  // ---- critic forward, clipped value loss (R:algos/ppo.py:104-113)
  double vl = 0.0;
  {
    const int c0 = half * (kc / 2), c1 = half ? kc : kc / 2;
    float s = 0.f;
    const __nv_bfloat16* hr = shc + row * L.pc;
    for (int c = c0; c < c1; c += 2) {
      const float2 hv = up_bf16(*reinterpret_cast<const uint32_t*>(hr + c));
      s = fmaf(hv.x, swc[c], fmaf(hv.y, swc[c + 1], s));
    }
    s += __shfl_xor_sync(0xffffffffu, s, 1);
    if (!half) {
      double dv = 0.0;
      if (ok) {
        const double v = (double)(s + s_bc);
        if (a.clipped_v) {
          const double vc = oldv + fmin(fmax(v - oldv, -a.clip), a.clip);
          const double lu = (v - ret) * (v - ret), lc = (vc - ret) * (vc - ret);
          vl = fmax(lu, lc);
          dv = lu >= lc ? 2.0 * (v - ret) / a.n_global : 0.0;
        } else {
          vl = (v - ret) * (v - ret);
          dv = 2.0 * (v - ret) / a.n_global;
        }
      }
      sdv[row] = (float)(dv * a.vcoef);
    }
  }
  {
    const double v = warp_sum(vl);
    if (lane == 0) red[w] = v;
  }
  __syncthreads();  // sdv, red
  // ---- critic backward (SIMT): thread = (8-column group, rows rg, rg + R/..),
  // 16-byte row loads / stores; dw_c and colsum(dh_c) reduced over the row
  // groups (lane pairs, then warps in fixed order)
  {
    const int ncg = kc / 8;       // column groups (<= 32)
    const int nrg = kMThr / ncg;  // row groups
    const int cg = t % ncg, rg = t / ncg;
    float dw[8], cs[8], wcc[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      dw[e] = cs[e] = 0.f;
      wcc[e] = swc[8 * cg + e];
    }
    if (rg < nrg) {
      for (int rr = rg; rr < kMRows; rr += nrg) {
        const uint4 hv = *reinterpret_cast<const uint4*>(shc + rr * L.pc + 8 * cg);
        const float dvr = sdv[rr];
        const uint32_t hw[4] = {hv.x, hv.y, hv.z, hv.w};
        uint32_t ow[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 hh = up_bf16(hw[e]);
          const float d0 = dvr * wcc[2 * e] * (fminf(hh.x, 0.f) + 1.f);
          const float d1 = dvr * wcc[2 * e + 1] * (fminf(hh.y, 0.f) + 1.f);
          dw[2 * e] = fmaf(dvr, hh.x, dw[2 * e]);
          dw[2 * e + 1] = fmaf(dvr, hh.y, dw[2 * e + 1]);
          cs[2 * e] += d0;
          cs[2 * e + 1] += d1;
          ow[e] = pk_bf16(d0, d1);
        }
        const int c = 8 * cg;
        if (r0 + rr < M && c < Kc) {
          __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(f.dhc) + (r0 + rr) * f.lddhc + c;
          if (c + 8 <= Kc && ((f.lddhc & 7) == 0)) {
            *reinterpret_cast<uint4*>(dst) = make_uint4(ow[0], ow[1], ow[2], ow[3]);
          } else {
            const __nv_bfloat16* ob = reinterpret_cast<const __nv_bfloat16*>(ow);
            for (int e = 0; e < 8 && c + e < Kc; ++e) dst[e] = ob[e];
          }
        }
      }
    }
    // row groups of one warp: lanes l, l + ncg, ... share cg
    for (int o = ncg; o < 32; o <<= 1)
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        dw[e] += __shfl_xor_sync(0xffffffffu, dw[e], o);
        cs[e] += __shfl_xor_sync(0xffffffffu, cs[e], o);
      }
    if (lane < ncg)
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        scrit[w * kc + 8 * lane + e] = dw[e];
        scrit[kMWarps * kc + w * kc + 8 * lane + e] = cs[e];
      }
  }
  __syncthreads();  // scrit complete
  float* pc = f.partc + (int64_t)blockIdx.x * f.plenc;
  for (int c = t; c < Kc; c += kMThr) {
    float dw = 0.f, cs = 0.f;
#pragma unroll
    for (int k = 0; k < kMWarps; ++k) {
      dw += scrit[k * kc + c];
      cs += scrit[kMWarps * kc + k * kc + c];
    }
    pc[c] = dw;
    if (f.csc) pc[Kc + 1 + c] = cs;
  }
  if (t == 0) {
    float s = 0.f;
    for (int rr = 0; rr < kMRows; ++rr) s += sdv[rr];
    pc[Kc] = s;
    double v = 0.0;
    for (int k = 0; k < kMWarps; ++k) v += red[k];
    f.lossp[(int64_t)blockIdx.x * f.lossld + 1] = (float)v;
  }
}

template <int NJT>
__global__ void __launch_bounds__(kMThr, 5) ppo_fused_mma_kernel(const __grid_constant__ PpoFusedArgs f) {
  extern __shared__ __align__(16) uint8_t smem[];
  pdl_trigger();
  pdl_wait();
  if (blockIdx.y == 0) fused_actor<NJT>(f, smem);
  else fused_critic(f, smem);
}

inline size_t mma_smem(int Ka, int Kc, int NJT) {
  const size_t x = ActorSmem(Ka, NJT).total, y = CriticSmem(Kc).total;
  return x > y ? x : y;
}

template <int NJT>
int launch_mma(const PpoFusedArgs& f, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    UL_CUDA(cudaFuncSetAttribute(ppo_fused_mma_kernel<NJT>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    attr = true;
  }
  const unsigned blocks = (unsigned)ceil_div(f.h.n_local > 0 ? f.h.n_local : 1, kMRows);
  return launch_pdl("ppo_fused_mma_kernel", ppo_fused_mma_kernel<NJT>, dim3(blocks, 2), dim3(kMThr),
                    mma_smem(f.Ka, f.Kc, NJT), s, f);
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

int launch_ppo_fused(const PpoFusedArgs& fin, int dtype, ReduceJob* jobs, int* njobs,
                     cudaStream_t s) {
  PpoFusedArgs f = fin;
  ReduceJob* ja = jobs;
  ReduceJob* jc = jobs + 1;
  UL_CHECK_ARG(ppo_fused_ok(f.h.A, f.Ka, f.Kc), "ppo fused head: unsupported shape");
  static int mma_env = -1;
  if (mma_env < 0) {
    const char* e = getenv("UL_FUSED_MMA");
    mma_env = e ? atoi(e) != 0 : 1;
  }
  // tensor-core variant: bf16 rows, even K (bf16 pairs), smem within budget
  const int ncg = rup8(f.Kc) / 8;  // critic column groups: a power of two <= 32
  const bool mma = mma_env && dtype == kBf16 && (f.Ka % 2) == 0 && (f.Kc % 2) == 0 &&
                   (ncg & (ncg - 1)) == 0 && ncg <= 32 && f.wba != nullptr &&
                   mma_smem(f.Ka, f.Kc, f.h.A <= 16 ? 2 : 4) <= 200 * 1024;
  if (!mma) f.lossp = nullptr;  // (the SIMT variant folds its loss partials itself)
  UL_CHECK_ARG(!mma || f.lossp != nullptr, "ppo fused head: tensor-core variant needs lossp");
  if (mma) UL_TRY(f.h.A <= 16 ? launch_mma<2>(f, s) : launch_mma<4>(f, s));
  else UL_TRY(dtype == kBf16 ? launch_t<__nv_bfloat16>(f, s) : launch_t<float>(f, s));
  const int64_t nblk = ceil_div(f.h.n_local > 0 ? f.h.n_local : 1, mma ? kMRows : kFRows);
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
  *njobs = 2;
  if (f.lossp) {  // [pol, val, kl] -> loss_out, dlog_std -> the gradient slot
    ReduceJob* jl = jobs + 2;
    *jl = ReduceJob{};
    jl->src = f.lossp;
    jl->nz = (int)nblk;
    jl->kind = 1;
    jl->len = f.lossld;
    jl->n0 = 3;
    jl->o0 = f.h.loss_out;
    jl->n1 = f.h.A;
    jl->o1 = f.h.dlogstd_out;
    *njobs = 3;
  }
  return UL_OK;
}

}  // namespace ul
