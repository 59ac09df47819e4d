// K13 Adam + joint global-norm clip + finiteness, K12 Polyak.
//
// Replaces R:tensornet/adam.py:30-40 (clip_global_norm), :43-80 (adam_step) and
// R:algos/sac.py:100-108 (soft_update).  All state (lr, t, norm, divergence) is
// device resident in a ul_opt_ctl record so the whole PPO step sequence can be
// captured in one CUDA graph with no host round trip:
//   prepare : one persistent pass over every gradient segment -> per-block
//             (sum g^2, #non-finite) partials; the last block reduces them in a
//             fixed order (deterministic), computes the joint norm and clip
//             factor, decides per segment whether Adam runs (reference order:
//             loss check, then segment 0 finiteness, then segment 1, ...),
//             increments the per-segment step counters and latches `diverged`.
//   apply   : elementwise clip-scale + Adam update.  The f32 operation order of
//             the reference (m*=b1; m+=(1-b1)g; v*=b2; v+=(1-b2)g*g;
//             p -= lr*(m/bc1)/(sqrt(v/bc2)+eps)) is reproduced with
//             round-to-nearest intrinsics (no FMA contraction), so given equal
//             gradients the update is bit-identical to numpy.
// HBM bytes: prepare 4 B/param, apply 28 B/param (+4 if clipped grads are
// written back for the clip_global_norm API).
#include <cuda_bf16.h>

#include "internal.cuh"
#include "opt_tail.cuh"

namespace ul {
namespace {

constexpr int kPrepThreads = 256;

__global__ void __launch_bounds__(kPrepThreads) prepare_kernel(SegTable st, ul_opt_ctl* ctl,
                                                               LossFinalize lf, int has_lf) {
  __shared__ double scratch[32];
  const int nb = gridDim.x;
  pdl_trigger();
  pdl_wait();
  const int64_t stride = (int64_t)nb * blockDim.x;
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (st.nseg == 2) {
    // the PPO / SAC case: both segments' first 8 loads in flight together
    double acc[2] = {0.0, 0.0};
    int bad = 0;
    for (int64_t i0 = t0; i0 < st.n[0] || i0 < st.n[1]; i0 += 8 * stride) {
      float x[2][8];
#pragma unroll
      for (int s = 0; s < 2; ++s)
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int64_t i = i0 + u * stride;
          x[s][u] = i < st.n[s] ? __ldg(st.g[s] + i) : 0.f;
        }
#pragma unroll
      for (int s = 0; s < 2; ++s)
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          acc[s] += (double)x[s][u] * (double)x[s][u];
          bad |= (!isfinite(x[s][u])) << s;
        }
    }
    const double t0s = block_sum(acc[0], scratch);
    const double t1s = block_sum(acc[1], scratch + 16);
    const int any0 = __syncthreads_or(bad & 1), any1 = __syncthreads_or(bad & 2);
    if (threadIdx.x == 0) {
      ctl->part[blockIdx.x][0] = t0s;
      ctl->part[blockIdx.x][1] = t1s;
      ctl->part_bad[blockIdx.x][0] = any0;
      ctl->part_bad[blockIdx.x][1] = any1 ? 1 : 0;
    }
  } else {
    for (int s = 0; s < st.nseg; ++s) {
      const float* g = st.g[s];
      const int64_t n = st.n[s];
      double acc = 0.0;
      int bad = 0;
      // 8 loads in flight per thread (issued before the dependent adds)
      for (int64_t i0 = t0; i0 < n; i0 += 8 * stride) {
        float x[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int64_t i = i0 + u * stride;
          x[u] = i < n ? __ldg(g + i) : 0.f;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          acc += (double)x[u] * (double)x[u];
          bad |= !isfinite(x[u]);
        }
      }
      const double tot = block_sum(acc, scratch);
      const int any_bad = __syncthreads_or(bad);
      if (threadIdx.x == 0) {
        ctl->part[blockIdx.x][s] = tot;
        ctl->part_bad[blockIdx.x][s] = any_bad;
      }
    }
  }
  if (!last_block_ticket(&ctl->ticket, nb)) return;
  prepare_tail(st.nseg, &ctl->part[0][0], &ctl->part_bad[0][0], UL_MAX_SEG, ctl, lf, has_lf, nb,
               scratch);
}

struct AdamScalars {
  float b1, one_m_b1, b2, one_m_b2, bc1, bc2, lr, eps;
};

// numpy's f32 operation order, round-to-nearest, no FMA contraction
__device__ __forceinline__ void adam_elem(float gi, float& m, float& v, float& p,
                                          const AdamScalars& k) {
  m = __fadd_rn(__fmul_rn(m, k.b1), __fmul_rn(k.one_m_b1, gi));
  v = __fadd_rn(__fmul_rn(v, k.b2), __fmul_rn(__fmul_rn(k.one_m_b2, gi), gi));
  const float mh = __fdiv_rn(m, k.bc1);
  const float vh = __fdiv_rn(v, k.bc2);
  const float step = __fdiv_rn(__fmul_rn(k.lr, mh), __fadd_rn(__fsqrt_rn(vh), k.eps));
  p = __fsub_rn(p, step);
}

// write the updated parameter i of segment s into its staged operand slot
__device__ __forceinline__ void stage_param(const StageOut& so, int s, int64_t i, float p) {
  for (int l = 0; l < so.nl[s]; ++l) {
    const int64_t o = i - so.w_off[s][l];
    const int cols = so.cols[s][l];
    if (o >= 0 && o < (int64_t)so.rows[s][l] * cols) {
      int64_t d;
      if (so.ld[s][l] == cols) {  // unpadded staged rows (in % 8 == 0): same offset
        d = so.dst_off[s][l] + o;
      } else {
        const int r = (int)o / cols, c = (int)o - r * cols;
        d = so.dst_off[s][l] + (int64_t)r * so.ld[s][l] + c;
      }
      if (so.dtype == kBf16) reinterpret_cast<__nv_bfloat16*>(so.dst[s])[d] = __float2bfloat16_rn(p);
      else reinterpret_cast<float*>(so.dst[s])[d] = p;
      return;
    }
  }
}

// parameters i0 .. i0 + cnt - 1 (consecutive) of segment s: the layer search
// and the row / column split once per quad, then a running column
__device__ __forceinline__ void stage_quad(const StageOut& so, int s, int64_t i0, const float* pa,
                                           int cnt) {
  for (int l = 0; l < so.nl[s]; ++l) {
    const int cols = so.cols[s][l];
    const int size = so.rows[s][l] * cols;
    int o = (int)(i0 - so.w_off[s][l]);
    if (o + cnt <= 0 || o >= size) continue;
    int e = 0;
    if (o < 0) {
      e = -o;
      o = 0;
    }
    int r = o / cols, c = o - r * cols;
    const int64_t ld = so.ld[s][l];
    for (; e < cnt && o < size; ++e, ++o) {
      const int64_t d = so.dst_off[s][l] + (int64_t)r * ld + c;
      if (so.dtype == kBf16) reinterpret_cast<__nv_bfloat16*>(so.dst[s])[d] = __float2bfloat16_rn(pa[e]);
      else reinterpret_cast<float*>(so.dst[s])[d] = pa[e];
      if (++c == cols) {
        c = 0;
        ++r;
      }
    }
  }
}

// the controller values the apply pass reads (copied once per CTA)
struct ApplyCtl {
  int upd[UL_MAX_SEG];
  double t[UL_MAX_SEG], lr[UL_MAX_SEG];
  double factor, beta1, beta2, eps;
};

__device__ __forceinline__ void read_apply_ctl(const volatile ul_opt_ctl* c, int nseg, ApplyCtl* o) {
  for (int s = 0; s < nseg; ++s) {
    o->upd[s] = c->seg_update[s];
    o->t[s] = (double)c->t[s];
    o->lr[s] = c->lr[s];
  }
  o->factor = c->factor;
  o->beta1 = c->beta1;
  o->beta2 = c->beta2;
  o->eps = c->eps;
}

// clip scale + Adam over segment s, elements t0, t0 + stride, ... (float4
// lanes when aligned); refreshes the staged tensor-core weights
struct AdamVec {
  float4 g, m, v, p;
};

__device__ __forceinline__ AdamVec load_adam4(const SegTable& st, int s, int64_t i) {
  AdamVec a;
  a.g = reinterpret_cast<const float4*>(st.g[s])[i];
  a.m = reinterpret_cast<const float4*>(st.m[s])[i];
  a.v = reinterpret_cast<const float4*>(st.v[s])[i];
  a.p = reinterpret_cast<const float4*>(st.p[s])[i];
  return a;
}

__device__ __forceinline__ void adam4(const SegTable& st, int s, int64_t i, AdamVec a,
                                      const AdamScalars& k, float f, bool scale, int write_grads,
                                      const StageOut& so, int has_so) {
  float* ga = reinterpret_cast<float*>(&a.g);
  float* ma = reinterpret_cast<float*>(&a.m);
  float* va = reinterpret_cast<float*>(&a.v);
  float* pa = reinterpret_cast<float*>(&a.p);
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    if (scale) ga[e] = __fmul_rn(ga[e], f);
    adam_elem(ga[e], ma[e], va[e], pa[e], k);
  }
  if (write_grads && scale) reinterpret_cast<float4*>(st.g[s])[i] = a.g;
  reinterpret_cast<float4*>(st.m[s])[i] = a.m;
  reinterpret_cast<float4*>(st.v[s])[i] = a.v;
  reinterpret_cast<float4*>(st.p[s])[i] = a.p;
  if (has_so && so.dst[s]) stage_quad(so, s, 4 * i, pa, 4);
}

__device__ __forceinline__ AdamScalars adam_scalars(const ApplyCtl& c, int s) {
  AdamScalars k;
  const double t = c.t[s];
  k.b1 = (float)c.beta1;
  k.one_m_b1 = (float)(1.0 - c.beta1);
  k.b2 = (float)c.beta2;
  k.one_m_b2 = (float)(1.0 - c.beta2);
  k.bc1 = (float)(1.0 - pow(c.beta1, t));
  k.bc2 = (float)(1.0 - pow(c.beta2, t));
  k.lr = (float)c.lr[s];
  k.eps = (float)c.eps;
  return k;
}

// vector elements [v0, n4) step stride, scalar tail from 4 n4 + t0
__device__ void apply_seg(const SegTable& st, const ApplyCtl& c, const AdamScalars& k, int s,
                          int write_grads, int do_adam, const StageOut& so, int has_so, int64_t t0,
                          int64_t stride, int64_t v0 = -1) {
  const int upd = c.upd[s];
  // clip_global_norm scales even when a later Adam raises; Adam itself only on upd
  const float f = (float)c.factor;
  const bool scale = c.factor != 1.0;
  float* __restrict__ g = st.g[s];
  const int64_t n = st.n[s];
  if (!do_adam || !upd) {  // clip-only (clip_global_norm) or a skipped segment
    if (write_grads && scale)
      for (int64_t i = t0; i < n; i += stride) g[i] = __fmul_rn(g[i], f);
    return;
  }
  float *pm = st.m[s], *pv = st.v[s], *pp = st.p[s];
  const bool vec = (((uintptr_t)g | (uintptr_t)pm | (uintptr_t)pv | (uintptr_t)pp) & 15) == 0;
  const int64_t n4 = vec ? n / 4 : 0;
  for (int64_t i = v0 >= 0 ? v0 : t0; i < n4; i += stride)  // 16 B per array per thread
    adam4(st, s, i, load_adam4(st, s, i), k, f, scale, write_grads, so, has_so);
  for (int64_t i = 4 * n4 + t0; i < n; i += stride) {
    float gi = g[i];
    if (scale) gi = __fmul_rn(gi, f);
    if (write_grads && scale) g[i] = gi;
    float m = pm[i], v = pv[i], p = pp[i];
    adam_elem(gi, m, v, p, k);
    pm[i] = m;
    pv[i] = v;
    pp[i] = p;
    if (has_so && so.dst[s]) stage_param(so, s, i, p);
  }
}

__global__ void __launch_bounds__(256, 4) apply_kernel(SegTable st, const ul_opt_ctl* __restrict__ ctl, int write_grads,
                             int do_adam, StageOut so, int has_so) {
  __shared__ ApplyCtl c;
  __shared__ AdamScalars k;  // (bias corrections: two f64 pow per CTA, not per thread)
  pdl_trigger();
  const int s = blockIdx.y;
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  // The thread's first float4 of m, v, p is loaded BEFORE the dependency
  // wait: only an earlier Adam apply writes them, and that one completed
  // before this step's forward GEMMs ran (the kernels this launch may overlap
  // -- the gradient reduction / prepare -- never touch them).  g and the
  // controller come after the wait.
  bool pre = false;
  AdamVec a0{};
  if (s < st.nseg && do_adam) {
    const bool vec =
        (((uintptr_t)st.g[s] | (uintptr_t)st.m[s] | (uintptr_t)st.v[s] | (uintptr_t)st.p[s]) & 15) == 0;
    if (vec && t0 < st.n[s] / 4) {
      pre = true;
      a0.m = reinterpret_cast<const float4*>(st.m[s])[t0];
      a0.v = reinterpret_cast<const float4*>(st.v[s])[t0];
      a0.p = reinterpret_cast<const float4*>(st.p[s])[t0];
    }
  }
  pdl_wait();
  if (s >= st.nseg) return;
  if (threadIdx.x == 0) {
    read_apply_ctl(ctl, st.nseg, &c);
    if (do_adam) k = adam_scalars(c, s);
  }
  if (pre) a0.g = reinterpret_cast<const float4*>(st.g[s])[t0];
  __syncthreads();
  if (pre && c.upd[s]) {
    adam4(st, s, t0, a0, k, (float)c.factor, c.factor != 1.0, write_grads, so, has_so);
    apply_seg(st, c, k, s, write_grads, do_adam, so, has_so, t0, stride, t0 + stride);
  } else {
    apply_seg(st, c, k, s, write_grads, do_adam, so, has_so, t0, stride);
  }
}

__global__ void polyak_kernel(float* __restrict__ tgt, const float* __restrict__ src, int64_t n,
                              float keep, float tau) {
  // reference order: t *= (1-tau); t += tau*o   (two f32 roundings each)
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool vec = (((uintptr_t)tgt | (uintptr_t)src) & 15) == 0;
  const int64_t n4 = vec ? n / 4 : 0;
  float4* t4 = reinterpret_cast<float4*>(tgt);
  const float4* s4 = reinterpret_cast<const float4*>(src);
  for (int64_t i = t0; i < n4; i += 2 * stride) {  // two 16 B loads in flight per array
    const int64_t j = i + stride;
    const float4 a = t4[i], b = __ldg(s4 + i);
    float4 c, d;
    if (j < n4) {
      c = t4[j];
      d = __ldg(s4 + j);
    }
    t4[i] = make_float4(__fadd_rn(__fmul_rn(a.x, keep), __fmul_rn(tau, b.x)),
                        __fadd_rn(__fmul_rn(a.y, keep), __fmul_rn(tau, b.y)),
                        __fadd_rn(__fmul_rn(a.z, keep), __fmul_rn(tau, b.z)),
                        __fadd_rn(__fmul_rn(a.w, keep), __fmul_rn(tau, b.w)));
    if (j < n4)
      t4[j] = make_float4(__fadd_rn(__fmul_rn(c.x, keep), __fmul_rn(tau, d.x)),
                          __fadd_rn(__fmul_rn(c.y, keep), __fmul_rn(tau, d.y)),
                          __fadd_rn(__fmul_rn(c.z, keep), __fmul_rn(tau, d.z)),
                          __fadd_rn(__fmul_rn(c.w, keep), __fmul_rn(tau, d.w)));
  }
  for (int64_t i = 4 * n4 + t0; i < n; i += stride)
    tgt[i] = __fadd_rn(__fmul_rn(tgt[i], keep), __fmul_rn(tau, src[i]));
}

int fill_table(SegTable& st, int nseg, float* const* params, float* const* grads,
               float* const* m, float* const* v, const int64_t* sizes, bool need_state) {
  UL_CHECK_ARG(nseg >= 1 && nseg <= UL_MAX_SEG, "adam: nseg %d outside [1, %d]", nseg,
               UL_MAX_SEG);
  st.nseg = nseg;
  for (int s = 0; s < nseg; ++s) {
    UL_CHECK_ARG(sizes[s] >= 0, "adam: negative segment size");
    UL_CHECK_ARG(grads[s] != nullptr || sizes[s] == 0, "adam: null grad segment");
    st.g[s] = grads[s];
    st.n[s] = sizes[s];
    st.p[s] = need_state ? params[s] : nullptr;
    st.m[s] = need_state ? m[s] : nullptr;
    st.v[s] = need_state ? v[s] : nullptr;
    if (need_state)
      UL_CHECK_ARG(sizes[s] == 0 || (params[s] && m[s] && v[s]), "adam: null state segment");
  }
  for (int s = nseg; s < UL_MAX_SEG; ++s) {
    st.g[s] = st.p[s] = st.m[s] = st.v[s] = nullptr;
    st.n[s] = 0;
  }
  return UL_OK;
}

int64_t max_n(const SegTable& st) {
  int64_t mx = 1;
  for (int s = 0; s < st.nseg; ++s) mx = st.n[s] > mx ? st.n[s] : mx;
  return mx;
}

}  // namespace

int launch_prepare(const SegTable& st, ul_opt_ctl* ctl, cudaStream_t s, const LossFinalize* lf) {
  int64_t nmax = max_n(st);
  int blocks = (int)ceil_div(nmax, kPrepThreads * 8);
  blocks = blocks < 1 ? 1 : (blocks > UL_PREP_BLOCKS ? UL_PREP_BLOCKS : blocks);
  LossFinalize f{};
  if (lf) f = *lf;
  return launch_pdl("prepare_kernel", prepare_kernel, dim3(blocks), dim3(kPrepThreads), 0, s, st,
                    ctl, f, lf ? 1 : 0);
}

int launch_apply(const SegTable& st, ul_opt_ctl* ctl, int write_grads, int do_adam,
                 cudaStream_t s, const StageOut* so) {
  int64_t nmax = max_n(st);
  int bx = (int)ceil_div(nmax, 256 * 4);
  bx = bx < 1 ? 1 : (bx > 4 * kNumSMs ? 4 * kNumSMs : bx);
  StageOut o{};
  if (so) o = *so;
  return launch_pdl("apply_kernel", apply_kernel, dim3(bx, st.nseg), dim3(256), 0, s, st,
                    (const ul_opt_ctl*)ctl, write_grads, do_adam, o, so ? 1 : 0);
}

}  // namespace ul

extern "C" int ul_opt_ctl_init(ul_opt_ctl* host_ctl, int nseg, const double* lr, double beta1,
                               double beta2, double eps, double max_norm) {
  UL_CHECK_ARG(host_ctl != nullptr, "opt ctl: null");
  UL_CHECK_ARG(nseg >= 1 && nseg <= UL_MAX_SEG, "opt ctl: bad nseg");
  memset(host_ctl, 0, sizeof(ul_opt_ctl));
  for (int s = 0; s < nseg; ++s) host_ctl->lr[s] = lr[s];
  host_ctl->beta1 = beta1;
  host_ctl->beta2 = beta2;
  host_ctl->eps = eps;
  host_ctl->max_norm = max_norm;
  host_ctl->factor = 1.0;
  host_ctl->fail_step = -1;
  return UL_OK;
}

extern "C" int64_t ul_opt_ctl_bytes(void) { return (int64_t)sizeof(ul_opt_ctl); }

// Joint norm over `nseg` gradient segments; optional clip-scale of the grads in
// place (clip_global_norm semantics).  No Adam.  ctl->norm receives the pre-clip
// norm; ctl->max_norm is the clip threshold.
extern "C" int ul_clip_global_norm(float* const* grads, const int64_t* sizes, int nseg,
                                   ul_opt_ctl* ctl, void* stream) {
  ul::SegTable st;
  UL_TRY(ul::fill_table(st, nseg, nullptr, grads, nullptr, nullptr, sizes, false));
  cudaStream_t s = ul::as_stream(stream);
  UL_TRY(ul::launch_prepare(st, ctl, s));
  return ul::launch_apply(st, ctl, /*write_grads=*/1, /*do_adam=*/0, s);
}

// One Adam step over `nseg` (param, grad, m, v) segments sharing one clip
// group: prepare (norm / finiteness / step counters) then apply.
extern "C" int ul_adam_step(float* const* params, float* const* grads, float* const* m,
                            float* const* v, const int64_t* sizes, int nseg, ul_opt_ctl* ctl,
                            int write_clipped_grads, void* stream) {
  ul::SegTable st;
  UL_TRY(ul::fill_table(st, nseg, params, grads, m, v, sizes, true));
  cudaStream_t s = ul::as_stream(stream);
  UL_TRY(ul::launch_prepare(st, ctl, s));
  return ul::launch_apply(st, ctl, write_clipped_grads, /*do_adam=*/1, s);
}

extern "C" int ul_polyak(float* target, const float* online, int64_t n, double tau,
                         void* stream) {
  UL_CHECK_ARG(n >= 0, "polyak: negative size");
  if (n == 0) return UL_OK;
  int blocks = (int)ul::ceil_div(n, 256 * 4);
  blocks = blocks > 4 * ul::kNumSMs ? 4 * ul::kNumSMs : blocks;
  ul::polyak_kernel<<<blocks, 256, 0, ul::as_stream(stream)>>>(target, online, n,
                                                               (float)(1.0 - tau), (float)tau);
  return ul::check_launch("polyak_kernel");
}
