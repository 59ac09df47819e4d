// Fused forward of an MLP's hidden-layer chain on tcgen05 (bf16): every
// 128-row tile runs ALL hidden layers back to back inside one CTA, the
// activation tile staying in shared memory as the next layer's A operand.
//
//   h_0 = elu(x W_0^T + b_0), h_l = elu(h_{l-1} W_l^T + b_l)   (R:tensornet/mlp.py:153-172)
//
// The layer-by-layer path (gemm_tc.cu) writes h_l to HBM and the next
// launch reads it back; here h_l is written once (TMA store, the backward
// needs it) and consumed from shared memory, and the chain is one persistent
// launch for both networks (no per-layer fill / drain, no launch gaps).
//
//   warp 0      : TMA producer -- the x tile into the activation buffer,
//                 then every layer's W k-steps (N halves of <= 256 rows)
//                 through a 2-stage ring
//   warp 1      : TMEM allocator (512 columns) + tcgen05.mma issuer
//   warps 2..17 : epilogue -- tcgen05.ld, bias + ELU, bf16 rows written
//                 straight into the activation buffer in the UMMA K-major
//                 128-byte-swizzle layout (which is also the TMA SW128 box
//                 layout, so the same bytes leave by TMA store to HBM)
//
// Per tile: x -> [MMA l -> epilogue l]_l, the accumulator of layer l in TMEM
// columns [0, N_l) (N_l <= 512).  Eligible: bf16, hidden widths multiples of
// 64 and <= 512, input width <= 512, no LayerNorm (mlp.cu falls back).
//
// Status: OPT-IN (UL_FUSED_FWD=1).  Bit-identical to the layer-by-layer path
// (tests/test_gpu_fused_fwd.py) but slower at cfg2: 83.6 us per step for both
// networks against 59 us for the three grouped launches (ncu: tensor pipe
// 16.5 % active, L2 17 %, DRAM 9 %; 54 % of warp samples are the epilogue
// waiting on acc_full).  With a 512-wide layer the activation tile fills
// 128 KB of shared memory, so MMA, epilogue and the next tile's x load
// serialise inside each CTA and the W ring is only two stages deep; the
// layer-by-layer kernels overlap those across tiles (double-buffered TMEM).
#include "tc_common.cuh"

namespace ul {
namespace fm {

using namespace tc;

constexpr int kMaxL = 4;                // hidden layers per chain
constexpr int kNP = 2;                  // networks per launch
constexpr int kTileBytes = 128 * 128;   // one 128-row x 64-column bf16 K tile (16 KB)
constexpr int kStageBytes = 256 * 128;  // one W k-step of one N half (<= 256 rows)
constexpr int kStages = 2;
constexpr int kEpi = 16;
constexpr int kThreads = (2 + kEpi) * 32;

struct Chain {
  CUtensorMap x;         // input rows [M, K0] bf16, box {64, 128}, SW128
  CUtensorMap w[kMaxL];  // staged W_l [N_l, ld] bf16, box {64, min(N_l, 256)}, SW128
  CUtensorMap h[kMaxL];  // outputs h_l [M, N_l] bf16, box {64, 128}, SW128
  const float* bias[kMaxL];
  __nv_bfloat16* hp[kMaxL];  // h_l base (the ones column)
  int64_t ldh[kMaxL];
  int N[kMaxL], K[kMaxL];  // K[0] = input width, K[l] = N[l-1]
  int L, M, mt;
};

struct Params {
  Chain c[kNP];
  int np, tiles;
};

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(bar)) : "memory");
}

__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int c0,
                                             int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(map),
      "r"(su32(src)), "r"(c0), "r"(c1)
      : "memory");
}

__device__ __forceinline__ void epi_bar() {  // the 16 epilogue warps only
  asm volatile("bar.sync 1, %0;" ::"n"(kEpi * 32) : "memory");
}

__device__ __forceinline__ uint32_t idesc_bf16(int n) {
  // f32 accumulate, bf16 A/B, both K-major, N >> 3, M = 128 >> 4
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) |
         ((uint32_t)(128 >> 4) << 24);
}

__global__ void __launch_bounds__(kThreads, 1) fused_fwd_kernel(const __grid_constant__ Params P) {
  extern __shared__ __align__(1024) uint8_t smem[];
  if (threadIdx.x == 0 && (su32(smem) & 1023u)) __trap();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // [activation buffer: act_tiles x 16 KB][stage ring][barriers]
  int act_tiles = 1;
  for (int i = 0; i < P.np; ++i) {
    const Chain& C = P.c[i];
    act_tiles = max(act_tiles, (C.K[0] + 63) / 64);
    for (int l = 0; l < C.L; ++l) act_tiles = max(act_tiles, C.N[l] / 64);
  }
  uint8_t* act = smem;
  uint8_t* stage = smem + act_tiles * kTileBytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(stage + kStages * kStageBytes);
  uint64_t* empty = full + kStages;
  uint64_t* x_full = empty + kStages;
  uint64_t* act_free = x_full + 1;
  uint64_t* acc_full = act_free + 1;
  uint64_t* epi_done = acc_full + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(epi_done + 1);

  pdl_trigger();
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(x_full, 1);
    mbar_init(act_free, 1);
    mbar_init(acc_full, 1);
    mbar_init(epi_done, kEpi);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 0 && lane == 0) {
    for (int i = 0; i < P.np; ++i) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&P.c[i].x) : "memory");
      for (int l = 0; l < P.c[i].L; ++l) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(&P.c[i].w[l]) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&P.c[i].h[l]) : "memory");
      }
    }
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        su32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  pdl_wait();

  auto problem_of = [&](int t, int* pr, int* mtile) {
    if (P.np > 1 && t >= P.c[0].mt) {
      *pr = 1;
      *mtile = t - P.c[0].mt;
    } else {
      *pr = 0;
      *mtile = t;
    }
  };

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      int it = 0, tl = 0;
      for (int t = blockIdx.x; t < P.tiles; t += gridDim.x, ++tl) {
        int pr, mtile;
        problem_of(t, &pr, &mtile);
        const Chain& C = P.c[pr];
        const int m0 = mtile * 128;
        if (tl > 0) mbar_wait(act_free, (tl - 1) & 1);  // last tile's stores read the buffer
        const int kt0 = (C.K[0] + 63) / 64;
        mbar_expect_tx(x_full, kt0 * kTileBytes);
        for (int kt = 0; kt < kt0; ++kt) tma_load_2d(act + kt * kTileBytes, &C.x, x_full, kt * 64, m0);
        for (int l = 0; l < C.L; ++l) {
          const int nkt = (C.K[l] + 63) / 64, nh = (C.N[l] + 255) / 256;
          const int rows = C.N[l] < 256 ? C.N[l] : 256;
          for (int kt = 0; kt < nkt; ++kt)
            for (int h = 0; h < nh; ++h, ++it) {
              const int s = it % kStages;
              mbar_wait(&empty[s], ((it / kStages) & 1) ^ 1);
              mbar_expect_tx(&full[s], rows * 128);
              tma_load_2d(stage + s * kStageBytes, &C.w[l], &full[s], kt * 64, h * 256);
            }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------- MMA issuer
    if (lane == 0) {
      int it = 0, tl = 0, gl = 0;
      for (int t = blockIdx.x; t < P.tiles; t += gridDim.x, ++tl) {
        int pr, mtile;
        problem_of(t, &pr, &mtile);
        const Chain& C = P.c[pr];
        mbar_wait(x_full, tl & 1);
        for (int l = 0; l < C.L; ++l, ++gl) {
          // the previous layer's epilogue has drained TMEM and (l > 0) written
          // h_{l-1} into the activation buffer
          if (gl > 0) mbar_wait(epi_done, (gl - 1) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const int nkt = (C.K[l] + 63) / 64, nh = (C.N[l] + 255) / 256;
          for (int kt = 0; kt < nkt; ++kt)
            for (int h = 0; h < nh; ++h, ++it) {
              const int s = it % kStages;
              const int n = (C.N[l] - h * 256) < 256 ? (C.N[l] - h * 256) : 256;
              const uint32_t idesc = idesc_bf16(n);
              mbar_wait(&full[s], (it / kStages) & 1);
              asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
              const uint32_t a_base = su32(act + kt * kTileBytes);
              const uint32_t b_base = su32(stage + s * kStageBytes);
#pragma unroll
              for (int kk = 0; kk < 4; ++kk) {
                const uint64_t da = smem_desc(a_base + kk * 32, 16, 1024, 2);
                const uint64_t db = smem_desc(b_base + kk * 32, 16, 1024, 2);
                mma<__nv_bfloat16>(tmem + (uint32_t)(h * 256), da, db, idesc,
                                   (kt > 0 || kk > 0) ? 1u : 0u);
              }
              mma_commit(&empty[s]);
            }
          mma_commit(acc_full);
        }
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue
    const int ew = warp - 2, q = warp & 3, slice = ew >> 2;
    const int row = q * 32 + lane;
    const bool issuer = ew == 0 && lane == 0;
    const uint32_t tbase = tmem + ((uint32_t)(q * 32) << 16);
    int tl = 0, gl = 0;
    for (int t = blockIdx.x; t < P.tiles; t += gridDim.x, ++tl) {
      int pr, mtile;
      problem_of(t, &pr, &mtile);
      const Chain& C = P.c[pr];
      const int m0 = mtile * 128;
      for (int l = 0; l < C.L; ++l, ++gl) {
        mbar_wait(acc_full, gl & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        // the TMA stores of h_{l-1} must have read the buffer before it is
        // overwritten (the MMAs reading it are complete: acc_full)
        if (issuer) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        epi_bar();
        const int N = C.N[l], per = N / 4;
        const float* bias = C.bias[l];
        for (int c0 = slice * per; c0 < (slice + 1) * per; c0 += 16) {
          float v[16];
          tmem_ld16(tbase + (uint32_t)c0, v);
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] = elu_fast(v[i] + __ldg(bias + c0 + i));
          uint4 lo, hi;
          lo.x = pack_bf16(v[0], v[1]);
          lo.y = pack_bf16(v[2], v[3]);
          lo.z = pack_bf16(v[4], v[5]);
          lo.w = pack_bf16(v[6], v[7]);
          hi.x = pack_bf16(v[8], v[9]);
          hi.y = pack_bf16(v[10], v[11]);
          hi.z = pack_bf16(v[12], v[13]);
          hi.w = pack_bf16(v[14], v[15]);
          // K-major SW128: row r of 64-column tile kt at r * 128 B, its 16-byte
          // chunk j at (j ^ (r % 8)) -- the UMMA operand and TMA box layout
          uint8_t* tr = act + (c0 >> 6) * kTileBytes + row * 128;
          const int j0 = (c0 & 63) >> 3;
          *reinterpret_cast<uint4*>(tr + ((j0 ^ (row & 7)) << 4)) = lo;
          *reinterpret_cast<uint4*>(tr + (((j0 + 1) ^ (row & 7)) << 4)) = hi;
        }
        // visible to the async proxy (the next layer's MMAs, the TMA store);
        // TMEM reads complete before the MMA issuer overwrites the accumulator
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        epi_bar();
        if (issuer) {
          for (int kt = 0; kt < N / 64; ++kt) tma_store_2d(&C.h[l], act + kt * kTileBytes, kt * 64, m0);
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
        if (slice == 0 && m0 + row < C.M)  // the activation's ones column (dW bias trick)
          C.hp[l][(int64_t)(m0 + row) * C.ldh[l] + N] = __float2bfloat16_rn(1.f);
        if (lane == 0) mbar_arrive(epi_done);
      }
      if (issuer) {  // the next tile's x may land once the last stores read the buffer
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        mbar_arrive(act_free);
      }
    }
    if (issuer) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

}  // namespace fm

bool fused_fwd_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("UL_FUSED_FWD");
    on = e ? atoi(e) != 0 : 0;  // opt-in: see the header note
  }
  return on == 1;
}

// The hidden layers [0, nl - 1) of every network fit the fused chain?
bool fused_fwd_ok(const MlpNet* nets, int n, int dt) {
  if (!fused_fwd_enabled() || dt != kBf16 || n < 1 || n > fm::kNP) return false;
  for (int k = 0; k < n; ++k) {
    const NetView& v = *nets[k].v;
    const int L = v.n_layers - 1;
    if (L < 1 || L > fm::kMaxL || v.ln || !nets[k].wp) return false;
    if (v.dims[0] > 512 || ((uintptr_t)nets[k].x & 15) || (nets[k].ldx * 2) % 16) return false;
    for (int l = 1; l <= L; ++l)
      if (v.dims[l] % 64 || v.dims[l] > 512) return false;
  }
  return true;
}

int fused_forward(const MlpNet* nets, int n, int64_t M, cudaStream_t s) {
  if (M <= 0) return UL_OK;
  UL_CHECK_ARG(M < (int64_t(1) << 31), "fused forward: too many rows");
  fm::Params P{};
  P.np = n;
  int act_tiles = 1;
  for (int k = 0; k < n; ++k) {
    const MlpNet& N = nets[k];
    const NetView& v = *N.v;
    fm::Chain& C = P.c[k];
    C.L = v.n_layers - 1;
    C.M = (int)M;
    C.mt = (int)ceil_div(M, 128);
    C.K[0] = v.dims[0];
    act_tiles = act_tiles > (int)ceil_div(C.K[0], 64) ? act_tiles : (int)ceil_div(C.K[0], 64);
    UL_TRY(tc::make_map(&C.x, N.x, 2, v.dims[0], M, N.ldx, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B));
    for (int l = 0; l < C.L; ++l) {
      C.N[l] = v.dims[l + 1];
      if (l > 0) C.K[l] = v.dims[l];
      act_tiles = act_tiles > C.N[l] / 64 ? act_tiles : C.N[l] / 64;
      const int64_t ldw = (v.dims[l] + 7) / 8 * 8;  // staged bf16 rows (mlp.cu staged_w)
      const __nv_bfloat16* w =
          reinterpret_cast<const __nv_bfloat16*>(N.wp) + v.wb_off[l];
      UL_TRY(tc::make_map(&C.w[l], w, 2, v.dims[l], v.dims[l + 1], ldw, 64,
                          v.dims[l + 1] < 256 ? v.dims[l + 1] : 256, CU_TENSOR_MAP_SWIZZLE_128B));
      __nv_bfloat16* h = reinterpret_cast<__nv_bfloat16*>(
          const_cast<float*>(act_ptr(v, N.acts, M, l, kBf16)));
      C.hp[l] = h;
      C.ldh[l] = act_ld(v.dims[l + 1], kBf16);
      C.bias[l] = N.params + v.b_off[l];
      UL_TRY(tc::make_map(&C.h[l], h, 2, v.dims[l + 1], M, C.ldh[l], 64, 128,
                          CU_TENSOR_MAP_SWIZZLE_128B));
    }
    P.tiles += C.mt;
  }
  const size_t smem = (size_t)act_tiles * fm::kTileBytes + fm::kStages * fm::kStageBytes + 1024;
  static size_t attr = 0;
  if (smem > attr) {
    UL_CUDA(cudaFuncSetAttribute(fm::fused_fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem));
    attr = smem;
  }
  const int grid = P.tiles < kNumSMs ? P.tiles : kNumSMs;
  return launch_pdl("fused_fwd_kernel", fm::fused_fwd_kernel, dim3((unsigned)grid),
                    dim3(fm::kThreads), smem, s, P);
}

}  // namespace ul
