// K7/K8 tensor-core path: tcgen05 (5th-gen tensor core) + TMEM + TMA GEMM for sm_100a.
//
// C[M,N] = A(M,K) B(K,N) with fp32 accumulation in TMEM, two operand types:
//   * fp32 storage read as kind::tf32 (UMMA K = 8), no conversion pass;
//   * bf16 storage read as kind::f16 / bf16 (UMMA K = 16): the MLP's bf16
//     activation path, half the operand bytes of tf32 per FLOP.
// TMA streams 128-byte-swizzled [rows x 128 B] tiles into a STAGES-deep
// shared-memory ring, one elected thread issues tcgen05.mma (UMMA M=128,
// N=BN) into a double-buffered TMEM accumulator, and 16 epilogue warps drain
// TMEM with tcgen05.ld and apply the fused MLP epilogue (bias / ELU /
// ELU-gradient / split-K partial store), leaving through TMA stores.
// Operands may be K-major or MN-major (the MLP's dX and dW GEMMs read W and
// the activations transposed; UMMA's MN-major smem descriptors absorb that,
// nothing is transposed in HBM).
//   warp 0       : TMA producer               (one elected lane)
//   warp 1       : TMEM allocator + MMA issuer (one elected lane)
//   warps 2..17  : epilogue (TMEM lane quarter = warp % 4, BN/4 column slice)
// Output type: bf16 for the hidden-layer epilogues of the bf16 path (the next
// GEMM's operand), fp32 otherwise (split-K dW partials, output layers).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <cstdlib>

#include "internal.cuh"
#include "tc_common.cuh"

namespace ul {
namespace tc {


struct TcArgs {
  int M, N, K;
  int k_per_split;  // multiple of BK
  int mt, nt, zt;   // tile counts (M, N, K-split)
  void* C;          // output element type: see OutT
  int64_t ldc;
  const float* bias;
  int ones_col;          // >= 0: also write C[m, ones_col] = 1 (activation ones column)
  unsigned long long* trace;  // diagnostics (UL_TC_TRACE): CTA 0 event timestamps, or null
  float* csum;                // per-CTA output column sums [grid][ldcs], or null
  int ldcs;
  int bres_kt;                // B-resident launches: K tiles of B held in smem
  int tma_store;              // 1 (default): TMA bulk stores; 0: coalesced st.global (UL_TC_TMASTORE=0)
  // kEpiLnFull: LayerNorm gain / shift, per-row (mean, rstd) out, h ones column
  const float* ln_g;
  const float* ln_beta;
  float* ln_stats;
  void* ln_h;
  int ln_h_ones;
  int64_t ldh;
};

// trace slots: [0] entry, [1] setup done, [2..33] producer k-tile issue,
// [34..65] MMA full-barrier pass, [66..81] epilogue acc ready, [82..97]
// epilogue tile done, [98] exit
__device__ __forceinline__ void trace_at(unsigned long long* tr, int slot) {
  if (tr && blockIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    tr[slot] = t;
  }
}

constexpr int kEpiWarps = 16;  // four warps per TMEM lane quarter, each a BN/4 column slice
constexpr int kLnMaxRanks = kLnFullMaxN / 256;  // N-tile CTAs of one fused-LayerNorm cluster
constexpr int kPThreads = (2 + kEpiWarps) * 32;

// bf16 operands -> bf16 hidden activations / gradients; everything else fp32
template <typename TI, int EPI>
using OutT = typename std::conditional<sizeof(TI) == 2 && (EPI == kEpiBiasElu || EPI == kEpiEluGrad ||
                                                            EPI == kEpiBiasLn || EPI == kEpiLnFull),
                                       __nv_bfloat16, float>::type;

// [stage ring][16 epilogue staging boxes][barriers][bias x 2]; as many stages
// as fit the 227 KB of dynamic shared memory (at most 6)
template <int BN, bool PAIR, int OB /* output element bytes */, int EPI, bool BRES = false>
struct Smem {
  static constexpr int kABytes = BM * 128;
  static constexpr int kBBytes = (PAIR ? BN / 2 : BN) * 128;  // this CTA's share of B
  // B-resident: the ring streams A only; B's K tiles sit in smem for the
  // whole kernel (runtime-sized region after the ring)
  static constexpr int kStageBytes = kABytes + (BRES ? 0 : kBBytes);
  // each epilogue warp double-buffers a 32-row x 64-byte staging box (a
  // box's TMA store reads one while the next box fills the other)
  // (bf16 bias/ELU outputs: one box per warp, single-buffered -- its TMA
  // store has a whole tile to read it -- which buys the 4th stage)
  static constexpr int kNStg =
      (OB == 2 && (EPI == kEpiBias || EPI == kEpiBiasElu || EPI == kEpiBiasLn)) ? 1 : 2;
  static constexpr int kStagingBytes = kEpiWarps * kNStg * 32 * 64;
  // ELU-gradient epilogue: per-quarter column sums of the output (4 x 512 floats)
  static constexpr int kCsumBytes = EPI == kEpiEluGrad ? 4 * kCsumMaxN * 4 : 0;
  // fused LayerNorm: per-row (mean, M2) of the 4 column slices [4][128] and the
  // cluster's per-CTA partials, double-buffered [2][kLnMaxRanks][128] (float2)
  // and the gain / shift of the tile's columns, double-buffered [2][2][BN]
  static constexpr int kLnBytes = EPI == kEpiLnFull ? (4 + 2 * kLnMaxRanks) * 128 * 8 + 4 * BN * 4 : 0;
  static constexpr int kFixed = 512 /*barriers*/ + 2 * BN * 4 /*bias*/ + kCsumBytes +
                                kLnBytes;  // (base is 1 KB aligned)
  static constexpr int kBudget = 232448;
  static constexpr int kStagesFit = (kBudget - kStagingBytes - kFixed) / kStageBytes;
  // (B-resident: the ring depth is chosen per launch from what the resident
  // B tiles leave, up to kBresMaxStages; kStages = 3 sizes kBresMax)
  static constexpr int kStages = BRES ? 3 : (kStagesFit > 6 ? 6 : kStagesFit);
  static constexpr int kBresMaxStages = 8;
  static constexpr int kBytes = kStages * kStageBytes + kStagingBytes + kFixed;  // + B region
  static constexpr int kBresMax = kBudget - kBytes;
};

__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* map,
                                                 uint32_t bar_cluster, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(su32(dst)),
      "l"(map), "r"(bar_cluster), "r"(c0), "r"(c1)
      : "memory");
}

template <typename T>
__device__ __forceinline__ void mma_pair(uint32_t tmem_d, uint64_t da, uint64_t db,
                                         uint32_t idesc, uint32_t acc) {
  if constexpr (sizeof(T) == 4) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n"
        "}\n" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(idesc), "r"(acc));
  } else {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n"
        "}\n" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(idesc), "r"(acc));
  }
}

// commit the leader's MMAs to the same barrier offset in both CTAs of the pair
__device__ __forceinline__ void mma_commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(su32(bar)),
      "h"((uint16_t)3)
      : "memory");
}

// Persistent: the grid is sized to the co-resident CTAs (pairs); tiles are
// walked with a strided loop.  The smem ring runs continuously across tiles
// and the TMEM accumulator is double-buffered, so tile i's epilogue overlaps
// tile i+1's TMA + MMA main loop.
//
// PAIR (cta_group::2): the two CTAs of a cluster (one TPC) compute one
// 256 x BN tile with M=256 UMMAs issued by the leader CTA.  Each CTA loads its
// own 128 rows of A and HALF of the B tile (BN/2 rows of N), so a stage is
// 32 KB instead of 48 KB per SM -- the L2->SM operand traffic (the bound of
// these short-K GEMMs) drops by a third and one more stage fits in smem.  Both
// CTAs' TMA loads complete on the leader's full barrier; the leader's commits
// are multicast to both CTAs' empty / accumulator barriers; both epilogues
// drain their own TMEM lanes and release the accumulator on the leader.
// Up to kMaxProb independent problems (the actor's and the critic's layer,
// or every deferred dW GEMM of a backward pass) share one launch: tile groups
// [end[i-1], end[i]) belong to problem i.
struct TcMaps {
  CUtensorMap a, b, c, x;
};
constexpr int kMaxProb = 8;
struct TcBatch {
  TcMaps m[kMaxProb];
  TcArgs a[kMaxProb];
  int end[kMaxProb];  // prefix sums of the problems' tile-group counts
  int np, ngroups;
  int cs_pr;          // problem whose epilogue emits column sums, or -1
  int lnc;            // kEpiLnFull: CTAs per cluster = N tiles of every problem
  int bres_c;         // B-resident: (problem, N tile) combos; CTA i keeps combo i % bres_c
  int bres_nst;       // B-resident: A ring depth of this launch
  int bres_kt_max;    // B-resident: K tiles of the deepest problem (the smem layout)
  // chained layers (bias+ELU forward of stacked layers, one launch): problem
  // net * chain_L + l is layer l of net `net`; a CTA runs whole row chains
  // (every layer of one M tile), two chains interleaved layer by layer
  int chain_L, chain_nets, chain_mt, chain_S;  // chain_S: tiles per chain
};
constexpr int kMaxChainL = 4;

// BRES (B resident; single problem, no pair, no split-K, K <= a few tiles):
// each CTA owns one N tile (CTA index mod nt) and walks M tiles; B's K tiles
// are loaded once, so only A streams -- a third of the smem fill traffic of
// the 48 KB/stage ring for the forward and dX GEMMs (K = 128..256).
template <typename TI, bool A_MN, bool B_MN, int EPI, int BN, bool PAIR, bool BRES>
__global__ void __launch_bounds__(kPThreads, 1)
    tc_gemm_kernel(const __grid_constant__ TcBatch B) {
  const TcArgs& p0_ = B.a[0];
  const int ngroups = B.ngroups;
  using O = Op<TI>;
  using TO = OutT<TI, EPI>;
  using S = Smem<BN, PAIR, (int)sizeof(TO), EPI, BRES>;
  constexpr bool kOutBf16 = sizeof(TO) == 2;
  constexpr bool LN = EPI == kEpiLnFull;
  static_assert(!(LN && (PAIR || BRES)), "fused LayerNorm launches are single-CTA MMA clusters");
  constexpr int CS = PAIR ? 2 : 1;
  constexpr int BNL = BN / CS;  // B rows (N) this CTA loads
  constexpr int BK = O::BK;
  constexpr uint32_t kChunkBytes = (uint32_t)BK * 128;  // one MN-major TMA box
  // ring depth: compile-time, or per launch for B-resident launches (A-only
  // stages are small; more of them keep more operand bytes in flight)
  const int kStages = BRES ? B.bres_nst : S::kStages;
  constexpr uint32_t kCols = 2 * BN;  // two accumulator buffers
  constexpr uint32_t kBoxBytes = 32 * 64;  // one epilogue staging box
  static_assert(S::kStages >= 2, "shared memory too small for the pipeline");
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1 KB-aligned base by pointer arithmetic on the __shared__ array, so the
  // compiler keeps the shared state space (LDS/STS, not generic LD/ST)
  uint8_t* smem = smem_raw;  // 1 KB aligned (128 B-swizzled TMA tiles need it)
  if (threadIdx.x == 0 && (su32(smem_raw) & 1023u)) __trap();
  // (region sized for the deepest problem; a CTA fills its own problem's K tiles)
  const uint32_t bres_bytes = BRES ? (uint32_t)B.bres_kt_max * S::kBBytes : 0u;
  uint8_t* sbres = smem + kStages * S::kStageBytes;  // B-resident K tiles
  uint8_t* staging = sbres + bres_bytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(staging + S::kStagingBytes);
  uint64_t* empty = full + kStages;
  uint64_t* acc_full = empty + kStages;  // [2]
  uint64_t* acc_empty = acc_full + 2;    // [2]
  uint64_t* aux_bar = acc_empty + 2;     // [kEpiWarps]
  uint64_t* bres_bar = aux_bar + kEpiWarps;
  uint64_t* ln_bar = bres_bar + 2;  // [2] fused LayerNorm: the cluster's row partials landed
  uint64_t* ready = ln_bar + 2;     // [2 slots][kMaxChainL] chained layers: layer l - 1 stored
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(ready + 2 * kMaxChainL);  // (16 B aligned)

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned long long w_prod = 0, w_full = 0, w_acc = 0, w_epi = 0, w_issue = 0;  // (UL_TC_TRACE)
  const long long t_start = clock64();
  pdl_trigger();
  if (threadIdx.x == 0) trace_at(p0_.trace, 0);

  uint32_t crank = 0;
  if (PAIR || LN) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(crank));
  const bool leader = !PAIR || crank == 0;
  // (fused LayerNorm: a cluster of B.lnc CTAs walks the same M tiles, CTA
  // rank r computing N tile r of each)
  const int CSL = LN ? B.lnc : CS;
  const int cl = blockIdx.x / CSL, ncl = gridDim.x / CSL;
  // this CTA's tile sequence t = t_begin, t_begin + t_step, ... < t_end.
  // B-resident: CTA i keeps (problem, N tile) combo c = i % bres_c (its B
  // tile loaded once) and walks that problem's M tiles i / bres_c, + G, ...
  int t_begin = cl, t_step = ncl, t_end = ngroups, bres_pr = 0, bres_n = 0;
  // (CTA pairs: per cluster; each CTA of the pair keeps its half of the B tile)
  if (BRES) {
    const int C = B.bres_c, c = cl % C;
    int acc = 0;
    while (bres_pr < B.np - 1 && c >= acc + B.a[bres_pr].nt) acc += B.a[bres_pr++].nt;
    bres_n = c - acc;
    t_begin = cl / C;
    t_step = ncl / C;
    t_end = (B.a[bres_pr].mt + CS - 1) / CS;
  }
  // chained layers: this CTA's chains are cl, cl + ncl, ... (Q of them); its
  // tile sequence t = 0.. walks them in pairs, layer by layer: the pair's
  // layer-l tiles of chain A, then of chain B, then layer l + 1 ...
  constexpr bool kChainable = EPI == kEpiBiasElu && !PAIR && !BRES && !LN;
  const bool CH = kChainable && B.chain_L > 0;
  int chainQ = 0;
  if (CH) {
    const int nch = B.chain_nets * B.chain_mt;
    chainQ = cl < nch ? (nch - 1 - cl) / ncl + 1 : 0;
    t_begin = 0;
    t_step = 1;
    t_end = (chainQ / 2) * 2 * B.chain_S + (chainQ % 2) * B.chain_S;
  }

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);   // (leader) producer arrive + both CTAs' TMA bytes
      mbar_init(&empty[s], 1);  // one (multicast) MMA commit
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], CS * kEpiWarps);  // both CTAs' epilogue warps (leader)
    }
    for (int w = 0; w < kEpiWarps; ++w) mbar_init(&aux_bar[w], 1);
    mbar_init(bres_bar, 1);
    if (LN) {
      mbar_init(&ln_bar[0], 1);
      mbar_init(&ln_bar[1], 1);
    }
    if (CH)  // layer l of a chain waits for every epilogue warp of layer l - 1's tiles
      for (int sl = 0; sl < 2; ++sl)
        for (int l = 1; l < B.chain_L; ++l)
          mbar_init(&ready[sl * kMaxChainL + l], kEpiWarps * B.a[l - 1].nt);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 0 && lane == 0) {
    for (int i = 0; i < B.np; ++i) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&B.m[i].a) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(&B.m[i].b) : "memory");
    }
  }
  if (warp == 1) {
    if (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       su32(tmem_slot)),
                   "r"(kCols));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       su32(tmem_slot)),
                   "r"(kCols));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (PAIR || LN) cluster_sync_all();  // peer barriers initialised before any cross-CTA signal
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  pdl_wait();  // setup above overlapped the previous kernel's tail
  if (threadIdx.x == 0) trace_at(p0_.trace, 1);

  // group t -> (problem, M-tile group, N-tile, split); this CTA takes M-tile
  // group*CS + rank
  struct Tile {
    int pr, m0, n0, z, kt_n;
    int slot, layer, pair;  // chained layers only
  };
  auto tile_of = [&](int t) {
    Tile T;
    T.slot = T.layer = T.pair = 0;
    if (CH) {
      const int S = B.chain_S;
      const int pp = t / (2 * S);
      int r = t - pp * 2 * S;
      const bool single = 2 * pp + 1 >= chainQ;  // a last pair with one chain
      int l = 0, slot = 0, n = 0;
      for (; l < B.chain_L; ++l) {
        const int ntl = B.a[l].nt;
        const int w = single ? ntl : 2 * ntl;
        if (r < w) {
          slot = r / ntl;
          n = r - slot * ntl;
          break;
        }
        r -= w;
      }
      const int c = cl + (2 * pp + slot) * ncl;
      const int net = c / B.chain_mt, m = c - net * B.chain_mt;
      T.pr = net * B.chain_L + l;
      T.z = 0;
      T.n0 = n * BN;
      T.m0 = m * BM;
      const int K = B.a[T.pr].K;
      T.kt_n = K > 0 ? (K + BK - 1) / BK : 0;
      T.slot = slot;
      T.layer = l;
      T.pair = pp;
      return T;
    }
    if (BRES) {  // t = M tile of this CTA's (problem, N tile) combo
      const TcArgs& P = B.a[bres_pr];
      T.pr = bres_pr;
      T.z = 0;
      T.n0 = bres_n * BN;
      T.m0 = (t * CS + (int)crank) * BM;
      T.kt_n = P.K > 0 ? (P.K + BK - 1) / BK : 0;
      return T;
    }
    T.pr = 0;
    while (T.pr < B.np - 1 && t >= B.end[T.pr]) ++T.pr;
    const TcArgs& P = B.a[T.pr];
    const int tl = T.pr ? t - B.end[T.pr - 1] : t;
    const int mg = (P.mt + CS - 1) / CS;
    if (LN) {  // one M tile per group; the cluster rank picks the N tile
      T.z = 0;
      T.n0 = (int)crank * BN;
      T.m0 = tl * BM;
    } else {
      T.z = tl / (mg * P.nt);
      const int r = tl - T.z * mg * P.nt;
      T.n0 = (r / mg) * BN;
      T.m0 = ((r % mg) * CS + (int)crank) * BM;
    }
    const int kb = T.z * P.k_per_split;
    const int ke = min(P.K, kb + P.k_per_split);
    T.kt_n = ke > kb ? (ke - kb + BK - 1) / BK : 0;
    return T;
  };

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      int it = 0;
      if (BRES && t_begin < t_end) {
        // this CTA's N tile of B (a pair: its half, completing on the
        // leader's barrier), all K tiles, once
        const Tile T0 = tile_of(t_begin);
        const int nb = T0.n0 + (int)crank * BNL;
        const uint32_t bbar = su32(bres_bar) & 0xFEFFFFFFu;
        if (leader) mbar_expect_tx(bres_bar, (uint32_t)(CS * T0.kt_n) * S::kBBytes);
        for (int kt = 0; kt < T0.kt_n; ++kt) {
          uint8_t* sb = sbres + kt * S::kBBytes;
          if (B_MN) {
#pragma unroll
            for (int c = 0; c < BNL / O::kChunk; ++c) {
              if (PAIR)
                tma_load_2d_pair(sb + c * kChunkBytes, &B.m[T0.pr].b, bbar, nb + O::kChunk * c,
                                 kt * BK);
              else
                tma_load_2d(sb + c * kChunkBytes, &B.m[T0.pr].b, bres_bar, nb + O::kChunk * c,
                            kt * BK);
            }
          } else {
            if (PAIR) tma_load_2d_pair(sb, &B.m[T0.pr].b, bbar, kt * BK, nb);
            else tma_load_2d(sb, &B.m[T0.pr].b, bres_bar, kt * BK, nb);
          }
        }
      }
      for (int t = t_begin; t < t_end; t += t_step) {
        const Tile T = tile_of(t);
        const int m0 = T.m0, n0 = T.n0, kt_n = T.kt_n;
        const TcArgs& P = B.a[T.pr];
        const CUtensorMap* tA = &B.m[T.pr].a;
        const CUtensorMap* tB = &B.m[T.pr].b;
        const int nb0 = n0 + (int)crank * BNL;  // first B row (N) of this CTA's share
        // chained layers: this tile's A rows are the previous layer's output
        // rows of the same chain, stored by this CTA's epilogue
        if (CH && T.layer > 0) mbar_wait(&ready[T.slot * kMaxChainL + T.layer], T.pair & 1);
        for (int kt = 0; kt < kt_n; ++kt, ++it) {
          const int s = it % kStages;
          mbar_wait_acc(&empty[s], ((it / kStages) & 1) ^ 1, p0_.trace ? &w_prod : nullptr);
          uint8_t* sa = smem + s * S::kStageBytes;
          uint8_t* sb = sa + S::kABytes;
          const int k0 = T.z * P.k_per_split + kt * BK;
          if (it < 32) trace_at(p0_.trace, 2 + it);
          if (PAIR) {
            // both CTAs' bytes complete on the leader's barrier (peer bit cleared)
            const uint32_t fb = su32(&full[s]) & 0xFEFFFFFFu;
            if (leader) mbar_expect_tx(&full[s], 2 * S::kStageBytes);
            if (A_MN) {
#pragma unroll
              for (int c = 0; c < BM / O::kChunk; ++c)
                tma_load_2d_pair(sa + c * kChunkBytes, tA, fb, m0 + O::kChunk * c, k0);
            } else {
              tma_load_2d_pair(sa, tA, fb, k0, m0);
            }
            if (BRES) {
              // (B resident: the stage holds A only)
            } else if (B_MN) {
#pragma unroll
              for (int c = 0; c < BNL / O::kChunk; ++c)
                tma_load_2d_pair(sb + c * kChunkBytes, tB, fb, nb0 + O::kChunk * c, k0);
            } else {
              tma_load_2d_pair(sb, tB, fb, k0, nb0);
            }
          } else if (BRES) {
            mbar_expect_tx(&full[s], S::kStageBytes);  // A only
            tma_load_2d(sa, tA, &full[s], k0, m0);
          } else {
            mbar_expect_tx(&full[s], S::kStageBytes);
            if (A_MN) {
#pragma unroll
              for (int c = 0; c < BM / O::kChunk; ++c)
                tma_load_2d(sa + c * kChunkBytes, tA, &full[s], m0 + O::kChunk * c, k0);
            } else {
              tma_load_2d(sa, tA, &full[s], k0, m0);
            }
            if (B_MN) {
#pragma unroll
              for (int c = 0; c < BN / O::kChunk; ++c)
                tma_load_2d(sb + c * kChunkBytes, tB, &full[s], n0 + O::kChunk * c, k0);
            } else {
              tma_load_2d(sb, tB, &full[s], k0, n0);
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------- MMA issuer
    // instruction descriptor: f32 accum, A/B format, majors, N>>3, M>>4
    // (M = 256 for a CTA pair)
    const uint32_t idesc = (1u << 4) | (O::kFmt << 7) | (O::kFmt << 10) |
                           ((A_MN ? 1u : 0u) << 15) | ((B_MN ? 1u : 0u) << 16) |
                           ((uint32_t)(BN >> 3) << 17) | ((uint32_t)((CS * BM) >> 4) << 24);
    if (lane == 0 && leader) {
      int it = 0, local = 0;
      if (BRES && t_begin < t_end) mbar_wait(bres_bar, 0);
      for (int t = t_begin; t < t_end; t += t_step, ++local) {
        const Tile TT = tile_of(t);
        const int kt_n = TT.kt_n;
        // (chained layers: a layer narrower than BN issues N = its width)
        uint32_t idesc_t = idesc;
        if (CH) {
          const int w = min(BN, (B.a[TT.pr].N - TT.n0 + 15) / 16 * 16);
          idesc_t = (idesc & ~(0x3Fu << 17)) | ((uint32_t)(w >> 3) << 17);
        }
        const int b = local & 1;
        mbar_wait_acc(&acc_empty[b], ((local >> 1) & 1) ^ 1,  // epilogues drained this buffer
                      p0_.trace ? &w_acc : nullptr);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t acc = tmem + (uint32_t)(b * BN);
        for (int kt = 0; kt < kt_n; ++kt, ++it) {
          const int s = it % kStages;
          mbar_wait_acc(&full[s], (it / kStages) & 1, p0_.trace ? &w_full : nullptr);
          if (it < 32) trace_at(p0_.trace, 34 + it);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t a_base = su32(smem + s * S::kStageBytes);
          const uint32_t b_base =
              BRES ? su32(sbres + kt * S::kBBytes) : a_base + S::kABytes;
          const long long ti0 = p0_.trace ? clock64() : 0;
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            // K-major: 8-row x 128 B swizzle atoms (SBO 1024), one UMMA K step
            // = 32 B along the row.  MN-major: 128 B of M/N per smem row,
            // chunks of kChunk M/N elements kChunkBytes apart (LBO), one UMMA
            // K step = 8 (tf32) / 16 (bf16) rows.
            const uint64_t da = A_MN ? smem_desc(a_base + kk * O::kMnKStep, kChunkBytes,
                                                 O::kMnSbo, O::kMnLayout)
                                     : smem_desc(a_base + kk * 32, 16, 1024, 2);
            const uint64_t db = B_MN ? smem_desc(b_base + kk * O::kMnKStep, kChunkBytes,
                                                 O::kMnSbo, O::kMnLayout)
                                     : smem_desc(b_base + kk * 32, 16, 1024, 2);
            const uint32_t accum = (kt > 0 || kk > 0) ? 1u : 0u;
            if (PAIR) mma_pair<TI>(acc, da, db, idesc_t, accum);
            else mma<TI>(acc, da, db, idesc_t, accum);
          }
          // frees the stage (in both CTAs of a pair) once these MMAs read it
          if (PAIR) mma_commit_pair(&empty[s]);
          else mma_commit(&empty[s]);
          if (p0_.trace) w_issue += (unsigned long long)(clock64() - ti0);
        }
        if (PAIR) mma_commit_pair(&acc_full[b]);  // accumulator b complete (both CTAs)
        else mma_commit(&acc_full[b]);
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue
    // 16 warps: TMEM lane quarter = warp % 4 (hardware rule), column slice =
    // (warp - 2) / 4 of four BN/4-wide slices.  Each warp owns two 32-row x
    // 64-byte staging boxes (64 B swizzle; bf16: 32 columns, fp32: 16) used
    // alternately: the ELU-gradient operand arrives in a box by TMA, results
    // leave it by TMA store while the next box fills.  Values are computed
    // 16 columns at a time (one tcgen05.ld x16) so the ELU math never holds
    // more than 16 accumulators live (no register spills at 96 registers).
    constexpr int kBoxC = 64 / (int)sizeof(TO);  // columns per staging box
    const int ew = warp - 2;
    const int quarter = warp & 3;
    const int slice = ew >> 2;
    const int row = quarter * 32 + lane;
    constexpr int kSlice = BN / 4;
    constexpr int kBiasPer = kSlice / 32;  // bias values each lane stages per tile
    float* sbias = reinterpret_cast<float*>(tmem_slot + 4);
    // column sums of the ELU-gradient output (the bias gradient of the layer
    // below): csum_s[quarter][n]; each (quarter, n) has exactly one writer
    // warp -- the one with this quarter and n's slice -- so no atomics and a
    // fixed summation order.  Each warp zeroes the entries it owns.
    float* csum_s = sbias + 2 * BN;
    const int cs_pr = B.cs_pr;
    const bool csum_on = EPI == kEpiEluGrad && cs_pr >= 0;
    if (csum_on) {
      for (int n = lane; n < kCsumMaxN; n += 32)
        if ((n % BN) / kSlice == slice) csum_s[quarter * kCsumMaxN + n] = 0.f;
    }
    uint64_t* abar = aux_bar + ew;
    uint32_t aphase = 0;
    int local = 0;
    int cj = 0;  // this warp's box counter (staging buffer = cj & 1)
    // bias of the next tile, loaded one tile ahead so its global latency hides
    // behind the current tile's epilogue
    float bnext[kBiasPer], gnext[LN ? kBiasPer : 1], enext[LN ? kBiasPer : 1];
    // fused LayerNorm smem: gain / shift [2][BN] each, slice partials
    // [4][128] and the cluster's per-CTA partials [2][kLnMaxRanks][128]
    float* ln_sg = csum_s + S::kCsumBytes / 4;
    float* ln_se = ln_sg + 2 * BN;
    float2* ln_sl = reinterpret_cast<float2*>(ln_se + 2 * BN);
    float2* ln_buf = ln_sl + 4 * 128;
    auto load_bias = [&](int t) {
      if (t >= t_end) return;
      const Tile T = tile_of(t);
      const TcArgs& p = B.a[T.pr];
#pragma unroll
      for (int j = 0; j < kBiasPer; ++j) {
        const int n = T.n0 + slice * kSlice + j * 32 + lane;
        bnext[j] = n < p.N ? __ldg(p.bias + n) : 0.f;
        if constexpr (LN) {
          gnext[j] = n < p.N ? __ldg(p.ln_g + n) : 0.f;
          enext[j] = n < p.N ? __ldg(p.ln_beta + n) : 0.f;
        }
      }
    };
    if (EPI == kEpiBias || EPI == kEpiBiasElu || EPI == kEpiBiasLn || LN) load_bias(t_begin);
    // diagnostics: epilogue warp 0, tiles 0-1, boxes 0-3 -> trace slots 100..
#define UL_ETRACE(k) \
  if (ew == 0 && lane == 0 && local < 2 && cj < 4) trace_at(p0_.trace, 100 + cj * 6 + (k))
    for (int t = t_begin; t < t_end; t += t_step, ++local) {
      const Tile T = tile_of(t);
      const int m0 = T.m0, n0 = T.n0, z = T.z;
      const TcArgs& p = B.a[T.pr];
      const CUtensorMap* tC = &B.m[T.pr].c;
      const CUtensorMap* tX = &B.m[T.pr].x;
      const int b = local & 1;
      const bool have = T.kt_n > 0;
      if (EPI == kEpiBias || EPI == kEpiBiasElu || EPI == kEpiBiasLn || LN) {
#pragma unroll
        for (int j = 0; j < kBiasPer; ++j) {
          sbias[b * BN + slice * kSlice + j * 32 + lane] = bnext[j];
          if constexpr (LN) {
            ln_sg[b * BN + slice * kSlice + j * 32 + lane] = gnext[j];
            ln_se[b * BN + slice * kSlice + j * 32 + lane] = enext[j];
          }
        }
        __syncwarp();
        load_bias(t + t_step);
      }
      // ELU-gradient operand: when the slice fits the two staging boxes, load
      // both boxes now (after every earlier store has read its box), so the
      // TMA latency overlaps the accumulator wait and is paid once per tile
      constexpr int kNBox = kSlice / kBoxC;
      constexpr bool kAuxAhead = EPI == kEpiEluGrad && kNBox <= S::kNStg;
      if (kAuxAhead) {
        if (lane == 0) {
          asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
          mbar_expect_tx(abar, kNBox * kBoxBytes);
#pragma unroll
          for (int k = 0; k < kNBox; ++k)
            tma_load_3d(staging + (ew * S::kNStg + (cj + k) % S::kNStg) * kBoxBytes, tX, abar,
                        n0 + slice * kSlice + k * kBoxC, m0 + quarter * 32, 0);
        }
        __syncwarp();
      }
      if (have) mbar_wait_acc(&acc_full[b], (local >> 1) & 1, p0_.trace ? &w_epi : nullptr);
      if (ew == 0 && lane == 0 && local < 16) trace_at(p0_.trace, 66 + local);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const int m = m0 + row;
      const int crow = m0 + quarter * 32;  // row of this warp's 32-row box in C (split z)
      const uint32_t taddr = tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(b * BN);
      if constexpr (LN) {
        // ---- fused LayerNorm (kEpiLnFull).  Pass 1: a = acc + bias, rounded
        // to the stored bf16 (what the backward reads), -> C; this warp's
        // running (mean, M2) of its valid columns, 16-column chunks merged
        // with Chan's formula.
        float mu = 0.f, m2 = 0.f;
        float cnt = 0.f;
#pragma unroll 1
        for (int c0 = slice * kSlice; c0 < (slice + 1) * kSlice; c0 += kBoxC, ++cj) {
          uint8_t* stg = staging + (ew * S::kNStg + cj % S::kNStg) * kBoxBytes;
          if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
          __syncwarp();
          uint4* srow = reinterpret_cast<uint4*>(stg + lane * 64);
          const int sw = (lane >> 1) & 3;
#pragma unroll
          for (int h = 0; h < kBoxC / 16; ++h) {
            const int cc = c0 + 16 * h;
            float v[16];
            if (have) {
              tmem_ld16(taddr + (uint32_t)cc, v);
            } else {
#pragma unroll
              for (int i = 0; i < 16; ++i) v[i] = 0.f;
            }
            const float4* bv = reinterpret_cast<const float4*>(sbias + b * BN + cc);
            uint32_t pk[8];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const float4 q4 = bv[i];
              pk[2 * i] = pack_bf16(v[4 * i] + q4.x, v[4 * i + 1] + q4.y);
              pk[2 * i + 1] = pack_bf16(v[4 * i + 2] + q4.z, v[4 * i + 3] + q4.w);
            }
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              v[2 * e] = bf_lo(pk[e]);
              v[2 * e + 1] = bf_hi(pk[e]);
            }
            const int nv = min(16, max(0, p.N - (n0 + cc)));
            if (nv > 0) {
              float sm = 0.f, qd = 0.f, mc;
              const float fn = (float)nv;
              if (nv == 16) {  // (every chunk but a ragged row end)
#pragma unroll
                for (int i = 0; i < 16; ++i) sm += v[i];
                mc = sm * (1.f / 16.f);
#pragma unroll
                for (int i = 0; i < 16; ++i) qd = fmaf(v[i] - mc, v[i] - mc, qd);
              } else {
#pragma unroll
                for (int i = 0; i < 16; ++i) sm += i < nv ? v[i] : 0.f;
                mc = sm / fn;
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                  const float d = v[i] - mc;
                  qd += i < nv ? d * d : 0.f;
                }
              }
              const float tot = cnt + fn, delta = mc - mu;
              mu += delta * (fn / tot);
              m2 += qd + delta * delta * (cnt * fn / tot);
              cnt = tot;
            }
            srow[(2 * h) ^ sw] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
            srow[(2 * h + 1) ^ sw] = make_uint4(pk[4], pk[5], pk[6], pk[7]);
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0 && n0 + c0 < p.N && m0 + quarter * 32 < p.M) {
            asm volatile(
                "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(tC),
                "r"(su32(stg)), "r"(n0 + c0), "r"(crow), "r"(0)
                : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          }
        }
        // ---- row statistics: the 4 slices of this CTA (shared memory), then
        // the cluster's N tiles (each CTA's partial stored into every rank's
        // buffer by st.async, completing on that rank's ln_bar[b])
        ln_sl[slice * 128 + row] = make_float2(mu, m2);
        asm volatile("bar.sync 1, %0;" ::"n"(kEpiWarps * 32) : "memory");
        const int lnc = B.lnc;
        if (ew == 0 && lane == 0) {
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&ln_bar[b])),
                       "r"((uint32_t)(lnc * 128 * 8))
                       : "memory");
        }
        if (slice == 0) {
          float cm = 0.f, cq = 0.f, cn = 0.f;
#pragma unroll
          for (int sl = 0; sl < 4; ++sl) {
            const float fn = (float)min(kSlice, max(0, p.N - (n0 + sl * kSlice)));
            if (fn > 0.f) {
              const float2 pv = ln_sl[sl * 128 + row];
              const float tot = cn + fn, delta = pv.x - cm;
              cm += delta * (fn / tot);
              cq += pv.y + delta * delta * (cn * fn / tot);
              cn = tot;
            }
          }
          const uint32_t src = su32(&ln_buf[(b * kLnMaxRanks + (int)crank) * 128 + row]);
          const uint32_t bar = su32(&ln_bar[b]);
          for (int r = 0; r < lnc; ++r) {
            uint32_t ra, rb;
            asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(src), "r"(r));
            asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rb) : "r"(bar), "r"(r));
            asm volatile(
                "st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f32 [%0], {%1, %2}, [%3];" ::"r"(ra),
                "f"(cm), "f"(cq), "r"(rb)
                : "memory");
          }
        }
        mbar_wait(&ln_bar[b], (local >> 1) & 1);
        float mean = 0.f, m2t = 0.f, ntot = 0.f;
        for (int r = 0; r < lnc; ++r) {  // fixed rank order: deterministic
          const float fn = (float)min(BN, max(0, p.N - r * BN));
          if (fn > 0.f) {
            const float2 pv = ln_buf[(b * kLnMaxRanks + r) * 128 + row];
            const float tot = ntot + fn, delta = pv.x - mean;
            mean += delta * (fn / tot);
            m2t += pv.y + delta * delta * (ntot * fn / tot);
            ntot = tot;
          }
        }
        const float rstd = rsqrtf(m2t / (float)p.N + 1e-5f);
        if (crank == 0 && slice == 0 && m < p.M) {
          reinterpret_cast<float2*>(p.ln_stats)[m] = make_float2(mean, rstd);
          if (p.ln_h_ones >= 0)
            reinterpret_cast<__nv_bfloat16*>(p.ln_h)[(int64_t)m * p.ldh + p.ln_h_ones] =
                __float2bfloat16_rn(1.f);
        }
        // ---- pass 2: h = elu((a - mean) rstd g + beta) from the same rounded a -> h
#pragma unroll 1
        for (int c0 = slice * kSlice; c0 < (slice + 1) * kSlice; c0 += kBoxC, ++cj) {
          uint8_t* stg = staging + (ew * S::kNStg + cj % S::kNStg) * kBoxBytes;
          if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
          __syncwarp();
          uint4* srow = reinterpret_cast<uint4*>(stg + lane * 64);
          const int sw = (lane >> 1) & 3;
#pragma unroll
          for (int h = 0; h < kBoxC / 16; ++h) {
            const int cc = c0 + 16 * h;
            float v[16];
            if (have) {
              tmem_ld16(taddr + (uint32_t)cc, v);
            } else {
#pragma unroll
              for (int i = 0; i < 16; ++i) v[i] = 0.f;
            }
            const float4* bv = reinterpret_cast<const float4*>(sbias + b * BN + cc);
            const float4* gv = reinterpret_cast<const float4*>(ln_sg + b * BN + cc);
            const float4* ev = reinterpret_cast<const float4*>(ln_se + b * BN + cc);
            uint32_t pk[8];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const float4 q4 = bv[i], g4 = gv[i], e4 = ev[i];
              const uint32_t a01 = pack_bf16(v[4 * i] + q4.x, v[4 * i + 1] + q4.y);
              const uint32_t a23 = pack_bf16(v[4 * i + 2] + q4.z, v[4 * i + 3] + q4.w);
              // (x - mean) rstd g + beta = x (rstd g) + (beta - mean rstd g)
              const float r0 = rstd * g4.x, r1 = rstd * g4.y, r2 = rstd * g4.z, r3 = rstd * g4.w;
              pk[2 * i] = pack_bf16(elu_fast(fmaf(bf_lo(a01), r0, fmaf(-mean, r0, e4.x))),
                                    elu_fast(fmaf(bf_hi(a01), r1, fmaf(-mean, r1, e4.y))));
              pk[2 * i + 1] = pack_bf16(elu_fast(fmaf(bf_lo(a23), r2, fmaf(-mean, r2, e4.z))),
                                        elu_fast(fmaf(bf_hi(a23), r3, fmaf(-mean, r3, e4.w))));
            }
            srow[(2 * h) ^ sw] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
            srow[(2 * h + 1) ^ sw] = make_uint4(pk[4], pk[5], pk[6], pk[7]);
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0 && n0 + c0 < p.N && m0 + quarter * 32 < p.M) {
            asm volatile(
                "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(tX),
                "r"(su32(stg)), "r"(n0 + c0), "r"(crow), "r"(0)
                : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          }
        }
      } else {
      // (chained layers: a tile narrower than BN -- the 128-wide last hidden
      // layer -- leaves the slices past its width untouched)
      const int c_end = CH && n0 + (slice + 1) * kSlice > p.N
                            ? max(slice * kSlice, (p.N - n0 + kBoxC - 1) / kBoxC * kBoxC)
                            : (slice + 1) * kSlice;
#pragma unroll 1
      for (int c0 = slice * kSlice; c0 < c_end; c0 += kBoxC, ++cj) {
        uint8_t* stg = staging + (ew * S::kNStg + cj % S::kNStg) * kBoxBytes;
        // this staging box free again (the TMA store issued from it two boxes
        // ago has read it)
        if (!kAuxAhead && lane == 0) {
          if (S::kNStg == 2) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
          else asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        }
        __syncwarp();
        UL_ETRACE(0);
        if (EPI == kEpiEluGrad && !kAuxAhead) {
          if (lane == 0) {
            mbar_expect_tx(abar, kBoxBytes);
            tma_load_3d(stg, tX, abar, n0 + c0, m0 + quarter * 32, 0);
          }
        }
        // 32 rows x 64 B, 64 B swizzle: 16 B granule q of row r at q ^ ((r >> 1) & 3)
        uint4* srow = reinterpret_cast<uint4*>(stg + lane * 64);
        const int sw = (lane >> 1) & 3;
#pragma unroll
        for (int h = 0; h < kBoxC / 16; ++h) {
          const int cc = c0 + 16 * h;  // first column of these 16
          float v[16];
          if (have) {
            tmem_ld16(taddr + (uint32_t)cc, v);
          } else {
#pragma unroll
            for (int i = 0; i < 16; ++i) v[i] = 0.f;
          }
          if (h == 0) UL_ETRACE(1);
          if (EPI == kEpiBias || EPI == kEpiBiasElu || EPI == kEpiBiasLn) {
            const float4* bv = reinterpret_cast<const float4*>(sbias + b * BN + cc);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const float4 q = bv[i];
              v[4 * i] += q.x;
              v[4 * i + 1] += q.y;
              v[4 * i + 2] += q.z;
              v[4 * i + 3] += q.w;
            }
          }
          if (EPI == kEpiBiasElu) {
#pragma unroll
            for (int i = 0; i < 16; ++i) v[i] = elu_fast(v[i]);
          }
          if (EPI == kEpiEluGrad && h == 0 && (!kAuxAhead || c0 == slice * kSlice)) {
            mbar_wait(abar, aphase);  // (aux ahead: both boxes on one phase)
            aphase ^= 1;
          }
          if (h == 0) UL_ETRACE(2);
          if constexpr (!kOutBf16) {
            // 4 granules of 4 floats
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              float4* g = reinterpret_cast<float4*>(srow + (q ^ sw));
              if (EPI == kEpiEluGrad) {
                const float4 h4 = *g;
                v[4 * q] = fmaf(v[4 * q], fminf(h4.x, 0.f), v[4 * q]);
                v[4 * q + 1] = fmaf(v[4 * q + 1], fminf(h4.y, 0.f), v[4 * q + 1]);
                v[4 * q + 2] = fmaf(v[4 * q + 2], fminf(h4.z, 0.f), v[4 * q + 2]);
                v[4 * q + 3] = fmaf(v[4 * q + 3], fminf(h4.w, 0.f), v[4 * q + 3]);
              }
              *g = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
            }
          } else {
            // granules 2h, 2h + 1 of 8 bf16
#pragma unroll
            for (int j = 0; j < 2; ++j) {
              const int q = 2 * h + j;
              if (EPI == kEpiEluGrad) {
                const uint4 hq = srow[q ^ sw];
                const uint32_t hw[4] = {hq.x, hq.y, hq.z, hq.w};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                  // v * elu'(h) = v * (min(h, 0) + 1) = fma(v, min(h, 0), v)
                  v[8 * j + 2 * e] = fmaf(v[8 * j + 2 * e], fminf(bf_lo(hw[e]), 0.f), v[8 * j + 2 * e]);
                  v[8 * j + 2 * e + 1] =
                      fmaf(v[8 * j + 2 * e + 1], fminf(bf_hi(hw[e]), 0.f), v[8 * j + 2 * e + 1]);
                }
              }
              srow[q ^ sw] = make_uint4(pack_bf16(v[8 * j], v[8 * j + 1]),
                                        pack_bf16(v[8 * j + 2], v[8 * j + 3]),
                                        pack_bf16(v[8 * j + 4], v[8 * j + 5]),
                                        pack_bf16(v[8 * j + 6], v[8 * j + 7]));
            }
          }
        }
        UL_ETRACE(3);
        if (csum_on && T.pr == cs_pr) {
          // column sums of the box as stored (what the dW GEMM reads): lanes
          // l and l + 16 sum rows [0, 16) / [16, 32) of column group l & 15
          // straight from the swizzled staging box (rows >= M hold zeros)
          __syncwarp();
          const int cg = lane & 15, rh = (lane >> 4) * 16;
          float s0 = 0.f, s1 = 0.f;
#pragma unroll 4
          for (int r = rh; r < rh + 16; ++r) {
            const uint8_t* rp = stg + r * 64 + ((((cg * (kOutBf16 ? 4 : 4)) >> 4) ^ ((r >> 1) & 3)) << 4);
            if constexpr (kOutBf16) {  // column pair 2cg, 2cg + 1
              const uint32_t u = *reinterpret_cast<const uint32_t*>(rp + (cg & 3) * 4);
              s0 += bf_lo(u);
              s1 += bf_hi(u);
            } else {  // column cg
              s0 += *reinterpret_cast<const float*>(rp + (cg & 3) * 4);
            }
          }
          s0 += __shfl_xor_sync(0xffffffffu, s0, 16);
          s1 += __shfl_xor_sync(0xffffffffu, s1, 16);
          if (lane < 16) {
            const int n = n0 + c0 + (kOutBf16 ? 2 * cg : cg);
            if (n < kCsumMaxN) csum_s[quarter * kCsumMaxN + n] += s0;
            if (kOutBf16 && n + 1 < kCsumMaxN) csum_s[quarter * kCsumMaxN + n + 1] += s1;
          }
        }
        if (p.tma_store) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0 && n0 + c0 < p.N && m0 + quarter * 32 < p.M) {
            // 3-D map [splits][M][N]: a box never spills into the next split's rows
            asm volatile(
                "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                    tC),
                "r"(su32(stg)), "r"(n0 + c0), "r"(crow), "r"(z)
                : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          }
        } else {
          // coalesced 16-byte stores straight from the staging box: the warp
          // never waits on an async store engine shared with the operand loads
          __syncwarp();
          const int rows_ok = p.M - crow;  // rows of this warp's box inside M
          constexpr int kPer = 16 / (int)sizeof(TO);  // elements per granule
          TO* cb = reinterpret_cast<TO*>(p.C) + ((int64_t)z * p.M + crow) * p.ldc + n0 + c0;
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int r = i * 8 + (lane >> 2), g = lane & 3;
            if (r < rows_ok) {
              const uint4 val = reinterpret_cast<const uint4*>(stg + r * 64)[g ^ ((r >> 1) & 3)];
              TO* dst = cb + (int64_t)r * p.ldc + kPer * g;
              const int col = n0 + c0 + kPer * g;
              if (col + kPer <= p.N) {
                *reinterpret_cast<uint4*>(dst) = val;
              } else {
                const TO* e8 = reinterpret_cast<const TO*>(&val);
                for (int e = 0; e < kPer && col + e < p.N; ++e) dst[e] = e8[e];
              }
            }
          }
          __syncwarp();  // staging reads done before the box is reused
        }
        UL_ETRACE(4);
      }
      }  // (not LN)
#undef UL_ETRACE
      if (p.ones_col >= 0 && n0 == 0 && slice == 0 && m < p.M) {
        TO* cp = reinterpret_cast<TO*>(p.C);
        cp[(int64_t)m * p.ldc + p.ones_col] = (TO)1.f;
      }
      if (ew == 0 && lane == 0 && local < 16) trace_at(p0_.trace, 82 + local);
      // release accumulator buffer b to the (leader's) MMA warp
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) {
        if (PAIR && !leader) {
          uint32_t remote;
          asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(remote) : "r"(su32(&acc_empty[b])));
          asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote)
                       : "memory");
        } else {
          asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&acc_empty[b]))
                       : "memory");
        }
      }
      // chained layers: once this warp's stores of the tile have landed in
      // global memory (and its ones-column writes are ordered before the async
      // proxy), the next layer of the chain may TMA-load these rows
      if (CH && T.layer + 1 < B.chain_L) {
        asm volatile("fence.proxy.async.global;" ::: "memory");
        if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
        __syncwarp();
        if (lane == 0)
          asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(
                           su32(&ready[T.slot * kMaxChainL + T.layer + 1]))
                       : "memory");
      }
    }
    // the staging smem must outlive the stores' reads; their global writes
    // complete with the grid (kernel boundary / the dependent launch's
    // griddepcontrol.wait), so the CTA need not wait for them
    if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (EPI == kEpiEluGrad && B.cs_pr >= 0) {
    // this CTA's column-sum partial row (quarters in fixed order)
    const TcArgs& pcs = B.a[B.cs_pr];
    const float* csum_s = reinterpret_cast<const float*>(tmem_slot + 4) + 2 * BN;
    for (int n = threadIdx.x; n < pcs.ldcs; n += blockDim.x) {
      float v = 0.f;
      if (n < pcs.N && n < kCsumMaxN)
        v = ((csum_s[n] + csum_s[kCsumMaxN + n]) + csum_s[2 * kCsumMaxN + n]) +
            csum_s[3 * kCsumMaxN + n];
      pcs.csum[(int64_t)blockIdx.x * pcs.ldcs + n] = v;
    }
  }
  // no CTA may leave (or free TMEM) while its pair can still write into its
  // smem / TMEM or arrive on its barriers
  if (PAIR || LN) cluster_sync_all();
  if (threadIdx.x == 0) trace_at(p0_.trace, 98);
  if (p0_.trace) {  // role wait cycles summed over CTAs: 128 producer, 129 MMA full, 130 MMA
                    // acc-empty, 131 epilogue warp 2 acc-full, 132 CTA cycles, 133 CTAs
    if (warp == 0 && lane == 0) atomicAdd(p0_.trace + 128, w_prod);
    if (warp == 1 && lane == 0) {
      atomicAdd(p0_.trace + 129, w_full);
      atomicAdd(p0_.trace + 130, w_acc);
      atomicAdd(p0_.trace + 134, w_issue);  // MMA issue + commit time
    }
    if (warp == 2 && lane == 0) {
      atomicAdd(p0_.trace + 131, w_epi);
      atomicAdd(p0_.trace + 132, (unsigned long long)(clock64() - t_start));
      atomicAdd(p0_.trace + 133, 1ull);
    }
  }
  if (warp == 1) {
    if (PAIR)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kCols));
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kCols));
  }
}

// ------------------------------------------------------------------ host side
// UL_TC_TRACE=1: every launch records CTA 0's event times (ul_tc_trace reads them)
inline unsigned long long* trace_buffer() {
  static int on = -1;
  static unsigned long long* buf = nullptr;
  if (on < 0) {
    const char* e = getenv("UL_TC_TRACE");
    on = e && atoi(e) != 0;
    if (on && cudaMalloc(&buf, kTraceSlots * sizeof(unsigned long long)) != cudaSuccess) buf = nullptr;
    if (buf) cudaMemset(buf, 0, kTraceSlots * sizeof(unsigned long long));
  }
  return buf;
}

inline int tma_store_on() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("UL_TC_TMASTORE");
    on = e ? atoi(e) != 0 : 1;  // measured: TMA stores beat direct stores
  }
  return on;
}

// one problem's tensor maps + kernel arguments (Prob: M/N/K split already fixed)
struct Prob {
  const GemmDesc* d;
  int zs, kps, ones_col;
};

template <typename TI, bool A_MN, bool B_MN, int EPI, int BN, bool PAIR, bool BRES>
int make_problem(const Prob& q, TcMaps* m, TcArgs* a, int* ngroups) {
  using O = Op<TI>;
  using TO = OutT<TI, EPI>;
  constexpr int CS = PAIR ? 2 : 1;
  constexpr int eb = O::kBytes, ob = (int)sizeof(TO);
  const GemmDesc& d = *q.d;
  const CUtensorMapSwizzle mn_sw =
      eb == 4 ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B;
  const CUtensorMapSwizzle out_sw = CU_TENSOR_MAP_SWIZZLE_64B;  // 64-byte box rows
  const int boxc = 64 / ob;
  // A(m,k): K-major -> rows=M, inner=K ; MN-major -> rows=K, inner=M
  if (A_MN) UL_TRY(make_map(&m->a, d.A, eb, d.M, d.K, d.lda, O::kChunk, O::BK, mn_sw));
  else UL_TRY(make_map(&m->a, d.A, eb, d.K, d.M, d.lda, O::BK, BM, CU_TENSOR_MAP_SWIZZLE_128B));
  if (B_MN) UL_TRY(make_map(&m->b, d.B, eb, d.N, d.K, d.ldb, O::kChunk, O::BK, mn_sw));
  else  // one CTA's share of the B tile
    UL_TRY(make_map(&m->b, d.B, eb, d.K, d.N, d.ldb, O::BK, BN / CS, CU_TENSOR_MAP_SWIZZLE_128B));
  // C (and split-K partials [splits][M][ldc]) stored by 32-row x 64-byte TMA boxes
  UL_TRY(make_map(&m->c, d.C, ob, d.N, d.M, d.ldc, boxc, 32, out_sw, q.zs));
  if (EPI == kEpiEluGrad) UL_TRY(make_map(&m->x, d.aux, ob, d.N, d.M, d.ldaux, boxc, 32, out_sw, 1));
  else if (EPI == kEpiLnFull) UL_TRY(make_map(&m->x, d.ln_h, ob, d.N, d.M, d.ldh, boxc, 32, out_sw, 1));
  else m->x = m->c;
  const int mt = (int)ceil_div(d.M, BM), nt = (int)ceil_div(d.N, BN);
  *a = TcArgs{(int)d.M, (int)d.N, (int)d.K, q.kps, mt, nt, q.zs, d.C, d.ldc, d.bias,
              q.ones_col, trace_buffer(),
              EPI == kEpiEluGrad && d.N <= kCsumMaxN ? d.csum_part : nullptr,
              (int)ceil_div(d.N, 4) * 4, BRES ? (int)ceil_div(d.K, O::BK) : 0, tma_store_on()};
  *ngroups = (int)ceil_div(mt, CS) * nt * q.zs;
  if (EPI == kEpiLnFull) {  // a cluster of nt CTAs per M tile
    UL_CHECK_ARG(nt <= kLnMaxRanks && q.zs == 1 && d.ln_h && d.ln_g && d.ln_beta && d.ln_stats,
                 "gemm_tc: fused LayerNorm needs N <= %d, no split-K, h / g / beta / stats",
                 kLnMaxRanks * BN);
    a->ln_g = d.ln_g;
    a->ln_beta = d.ln_beta;
    a->ln_stats = d.ln_stats;
    a->ln_h = d.ln_h;
    a->ln_h_ones = d.ln_h_ones;
    a->ldh = d.ldh;
    *ngroups = mt;
  }
  return UL_OK;
}

// chained layers (chain_L > 0): q[net * chain_L + l] is layer l of net `net`
struct ChainSpec {
  int nets, L;
};

template <typename TI, bool A_MN, bool B_MN, int EPI, int BN, bool PAIR, bool BRES = false>
int launch(const Prob* q, int np, cudaStream_t s, const ChainSpec* chain = nullptr) {
  using TO = OutT<TI, EPI>;
  using SM = Smem<BN, PAIR, (int)sizeof(TO), EPI, BRES>;
  constexpr int CS = PAIR ? 2 : 1;
  UL_CHECK_ARG(np >= 1 && np <= kMaxProb, "gemm_tc: 1..%d problems per launch", kMaxProb);
  TcBatch B{};  // ~5 KB kernel parameter block (per call: launches may come from several threads)
  B.np = np;
  B.cs_pr = -1;
  int total = 0;
  for (int i = 0; i < np; ++i) {
    int ng = 0;
    UL_TRY((make_problem<TI, A_MN, B_MN, EPI, BN, PAIR, BRES>(q[i], &B.m[i], &B.a[i], &ng)));
    total += ng;
    B.end[i] = total;
    if (B.a[i].csum && B.cs_pr < 0) B.cs_pr = i;
    else B.a[i].csum = nullptr;  // one column-sum problem per launch
  }
  B.ngroups = total;
  // fused LayerNorm: every problem's N tiles form one cluster
  const int CSX = EPI == kEpiLnFull ? B.a[0].nt : CS;
  B.lnc = CSX;
  for (int i = 1; i < np; ++i)
    UL_CHECK_ARG(EPI != kEpiLnFull || B.a[i].nt == CSX, "gemm_tc: fused LayerNorm batch widths differ");
  auto kern = tc_gemm_kernel<TI, A_MN, B_MN, EPI, BN, PAIR, BRES>;
  // B-resident: one (problem, N tile) combo per CTA residue class; the B
  // region holds the deepest problem's K tiles
  int bres_kt = 0;
  B.bres_c = 0;
  for (int i = 0; i < np; ++i) {
    B.bres_c += B.a[i].nt;
    bres_kt = B.a[i].bres_kt > bres_kt ? B.a[i].bres_kt : bres_kt;
  }
  B.bres_kt_max = bres_kt;
  UL_CHECK_ARG(!BRES || B.bres_c * CS <= kNumSMs,
               "gemm_tc: B-resident launch with too many N tiles");
  B.bres_nst = SM::kStages;
  size_t bytes = SM::kBytes;
  if (BRES) {  // as many A stages as the resident B leaves room for (UL_TC_BRES_STAGES caps)
    static int cap_env = -1;
    if (cap_env < 0) {
      const char* e = getenv("UL_TC_BRES_STAGES");
      cap_env = e ? atoi(e) : SM::kBresMaxStages;
    }
    const size_t bres = (size_t)bres_kt * SM::kBBytes;
    const size_t other = SM::kBytes - (size_t)SM::kStages * SM::kStageBytes;
    int nst = (int)((SM::kBudget - other - bres) / SM::kStageBytes);
    nst = nst > cap_env ? cap_env : nst;
    nst = nst > SM::kBresMaxStages ? SM::kBresMaxStages : nst;
    UL_CHECK_ARG(nst >= 2, "gemm_tc: B-resident launch leaves no room for the A ring");
    B.bres_nst = nst;
    bytes = other + (size_t)nst * SM::kStageBytes + bres;
  }
  cudaLaunchConfig_t cfg{};
  cfg.blockDim = dim3(kPThreads);
  cfg.dynamicSmemBytes = bytes;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CSX;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  // persistent: as many clusters as can be co-resident (one CTA per SM; GPC
  // sizes may leave SMs idle for CS > 1, so ask the occupancy API rather than
  // queue a second wave behind the first)
  static int max_cl[kLnMaxRanks + 1] = {};  // per cluster size
  int& max_clusters = max_cl[CSX <= kLnMaxRanks ? CSX : 0];
  if (max_clusters == 0) {
    UL_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 BRES ? SM::kBudget : SM::kBytes));
    int n = kNumSMs / CSX;
    if (CSX > 1) {
      cfg.gridDim = dim3((unsigned)(n * CSX));
      int qn = 0;
      if (cudaOccupancyMaxActiveClusters(&qn, kern, &cfg) == cudaSuccess && qn > 0 && qn < n)
        n = qn;
      cudaGetLastError();
    }
    max_clusters = n;
  }
  // UL_TC_GRID_DX: cap the CTA count of the ELU-gradient (dX) launches, so
  // the two networks' dX chains (two streams) share the GPU instead of
  // queueing whole-GPU launches behind each other (experiment)
  static int grid_dx = -1;
  if (grid_dx < 0) {
    const char* e = getenv("UL_TC_GRID_DX");
    grid_dx = e ? atoi(e) : 0;
  }
  int cap = max_clusters;
  if (EPI == kEpiEluGrad && grid_dx > 0 && grid_dx / CS < cap) cap = grid_dx / CS;
  int grid = (total < cap ? total : cap) * CSX;
  if (chain) {  // whole row chains: one CTA per chain up to the co-resident CTAs
    UL_CHECK_ARG(EPI == kEpiBiasElu && !PAIR && !BRES && chain->L >= 1 && chain->L <= kMaxChainL &&
                     chain->nets >= 1 && chain->nets * chain->L == np,
                 "gemm_tc: bad chained-layer launch");
    B.chain_L = chain->L;
    B.chain_nets = chain->nets;
    B.chain_mt = B.a[0].mt;
    B.chain_S = 0;
    for (int l = 0; l < chain->L; ++l) B.chain_S += B.a[l].nt;
    for (int i = 0; i < np; ++i)
      UL_CHECK_ARG(B.a[i].mt == B.chain_mt && B.a[i].nt == B.a[i % chain->L].nt && B.a[i].zt == 1,
                   "gemm_tc: chained layers need equal M / widths per layer across nets");
    const int nch = chain->nets * B.chain_mt;
    grid = nch < cap ? nch : cap;
  }
  if (BRES) {  // every CTA (pair) keeps one (problem, N tile) combo
    int ncl_b = (cap < total ? cap : total) / B.bres_c * B.bres_c;
    if (ncl_b < B.bres_c) ncl_b = B.bres_c;
    grid = ncl_b * CSX;
  }
  cfg.gridDim = dim3((unsigned)grid);
  for (int i = 0; i < np; ++i)
    if (q[i].d->csum_nz) *q[i].d->csum_nz = i == B.cs_pr ? grid : 0;
  UL_CUDA(cudaLaunchKernelEx(&cfg, kern, B));
  return check_launch("tc_gemm_kernel");
}

// N tile: 256 for N > 128; UL_TC_BN_FWD / UL_TC_BN_DX = 128 cap the forward
// (bias epilogues) / ELU-gradient tiles (wave-quantisation experiments)
inline int bn_of(const GemmDesc& d) {
  static int cap_fwd = -1, cap_dx = -1;
  if (cap_fwd < 0) {
    const char* e = getenv("UL_TC_BN_FWD");
    cap_fwd = e ? atoi(e) : 256;
    const char* f = getenv("UL_TC_BN_DX");
    cap_dx = f ? atoi(f) : 256;
  }
  const int cap = d.epi == kEpiEluGrad ? cap_dx
                  : (d.epi == kEpiBias || d.epi == kEpiBiasElu || d.epi == kEpiBiasLn ||
                     d.epi == kEpiLnFull) ? cap_fwd
                                                                                         : 256;
  return d.N > 128 && cap >= 256 ? 256 : 128;
}

}  // namespace tc
// whether a dW batch (MN-major A and B, store epilogue) runs on CTA pairs
bool tc_dw_pairs() {
  const char* e = getenv("UL_TC_PAIR_DW");
  const char* e2 = getenv("UL_TC_PAIR");
  return (e ? atoi(e) != 0 : true) && !(e2 && atoi(e2) == 0);
}
namespace tc {

template <typename TI>
int dispatch(const Prob* q, int np, cudaStream_t s) {
  const GemmDesc& d = *q[0].d;
  int bn = 128;  // one tile width for the whole batch
  bool all_two_m = true;
  for (int i = 0; i < np; ++i) {
    bn = bn_of(*q[i].d) > bn ? bn_of(*q[i].d) : bn;
    all_two_m = all_two_m && ceil_div(q[i].d->M, BM) >= 2;
  }
  const bool amn = !d.a_kmajor, bmn = !d.b_kmajor;
  // CTA pairs (cta_group::2, M = 256 per UMMA) whenever there are two M
  // tiles; UL_TC_PAIR=0 disables them (experiments).
  static int pair_ok = -1;
  if (pair_ok == -1) {
    const char* e = getenv("UL_TC_PAIR");
    pair_ok = e ? atoi(e) : -2;
  }
  // default: pairs for tf32 (4-byte operands: the halved B traffic pays) and
  // for deep-K bf16 GEMMs (K >= 1024: the FlashSAC 1024-wide critics, 2.81 ->
  // 2.68 ms per cfg4 update); single CTAs for the shallow bf16 GEMMs (the cfg2
  // update, K <= 512, measured faster without)
  bool deep = true;
  for (int i = 0; i < np; ++i) deep = deep && q[i].d->K >= 1024;
  const bool want = pair_ok == -2 ? (sizeof(TI) == 4 || deep) : pair_ok != 0;
  // dW batches (both operands MN-major, K = the minibatch rows): CTA pairs
  // split B between the two SMs, cutting the per-SM operand stream of these
  // L2-bound GEMMs by a third; a single-M-tile problem's second CTA computes
  // on TMA zero fill (UL_TC_PAIR_DW=0 disables)
  static int pair_dw = -1;
  if (pair_dw < 0) {
    const char* e = getenv("UL_TC_PAIR_DW");
    pair_dw = e ? atoi(e) != 0 : 1;
  }
  const bool dw_batch = amn && bmn && d.epi == kEpiStore;
  // UL_TC_PAIR_DX / UL_TC_PAIR_FWD: pairs for the ELU-gradient dX GEMMs /
  // the bias(+ELU) forward GEMMs only (experiments)
  static int pair_dx = -1, pair_fwd = -1;
  if (pair_dx < 0) {
    const char* e = getenv("UL_TC_PAIR_DX");
    pair_dx = e ? atoi(e) != 0 : 0;
    const char* f = getenv("UL_TC_PAIR_FWD");
    pair_fwd = f ? atoi(f) != 0 : 0;
  }
  const bool pair = (want && all_two_m) || (dw_batch && pair_dw && pair_ok != 0) ||
                    (all_two_m && pair_dx && d.epi == kEpiEluGrad) ||
                    (all_two_m && pair_fwd && (d.epi == kEpiBiasElu || d.epi == kEpiBias ||
                                               d.epi == kEpiBiasLn));
  // B resident (A streamed alone) when one problem's whole N tile of B fits
  // the smem left over by the 3-stage A ring, and there is no split-K
  // (default: not for the ELU-gradient dX GEMMs -- the cfg2 update measured
  // 4.643 ms with streamed B against 4.679 ms B-resident; UL_TC_BRES=1 / 0
  // forces it on / off everywhere)
  static int bres_env = -2;
  if (bres_env == -2) {
    const char* e = getenv("UL_TC_BRES");
    bres_env = e ? (atoi(e) != 0 ? 1 : 0) : -1;
  }
  const bool bres_ok = bres_env >= 0 ? bres_env == 1 : d.epi != kEpiEluGrad;
  const int64_t bk = sizeof(TI) == 2 ? 64 : 32;
  // (several problems: every CTA keeps one problem's N tile; UL_TC_BRES_MULTI=0
  // restricts B residency to single-problem launches)
  static int bres_multi = -1;
  if (bres_multi < 0) {
    const char* e = getenv("UL_TC_BRES_MULTI");
    bres_multi = e ? atoi(e) != 0 : 1;
  }
  bool one_split = true;
  for (int i = 0; i < np; ++i) one_split = one_split && q[i].zs == 1;
  const bool bres_base = bres_ok && (np == 1 || bres_multi) && !amn && one_split &&
                         (sizeof(TI) == 2 || !pair);
  // B bytes per CTA / (problem, N tile) combos at tile width b
  auto bres_fits = [&](int b, int64_t max_bytes) {
    int64_t bytes = 0, combos = 0;
    for (int i = 0; i < np; ++i) {
      const int64_t x = ceil_div(q[i].d->K, bk) * (int64_t)b * 128;
      bytes = x > bytes ? x : bytes;
      combos += ceil_div(q[i].d->N, b);
    }
    return bres_base && bytes <= max_bytes && combos <= kNumSMs;
  };
  // A 256-wide B tile too deep for one CTA's shared memory: a CTA PAIR keeps
  // it resident, half in each SM (cta_group::2 MMAs read both halves), and
  // streams only A (opt-in UL_TC_PAIR_BRES=1; UL_TC_PAIR_BRES_DX=1 extends it
  // to the ELU-gradient dX GEMMs.  Measured on the cfg2 update: 4.33 / 4.48 ms
  // against 4.30 without -- the pair's cross-SM MMA costs more than the
  // halved B stream saves at K <= 512)
  static int pair_bres = -1, pair_bres_dx = -1;
  if (pair_bres < 0) {
    const char* e = getenv("UL_TC_PAIR_BRES");
    pair_bres = e ? atoi(e) != 0 : 0;
    const char* f = getenv("UL_TC_PAIR_BRES_DX");
    pair_bres_dx = f ? atoi(f) != 0 : 0;
  }
  auto bres_fits_pair = [&](int b, int64_t max_bytes) {
    if (!pair_bres || sizeof(TI) != 2 || !all_two_m || amn || !one_split) return false;
    if (!(np == 1 || bres_multi)) return false;
    if (d.epi == kEpiEluGrad ? !pair_bres_dx : !(bres_env != 0)) return false;
    int64_t bytes = 0, combos = 0;
    for (int i = 0; i < np; ++i) {
      const int64_t x = ceil_div(q[i].d->K, bk) * (int64_t)(b / 2) * 128;
      bytes = x > bytes ? x : bytes;
      combos += ceil_div(q[i].d->N, b);
    }
    return bytes <= max_bytes && 2 * combos <= kNumSMs;
  };
  // UL_TC_BRES128=1: a 256-wide B tile too deep for shared memory becomes
  // B-resident 128-wide tiles (measured: cfg2 update 4.41 -> 4.60 ms, cfg4
  // 2.78 -> 2.84 ms, cfg3 0.724 -> 0.713 ms -- off by default)
  static int bres128 = -1;
  if (bres128 < 0) {
    const char* e = getenv("UL_TC_BRES128");
    bres128 = e ? atoi(e) != 0 : 0;
  }
  // fused LayerNorm (bf16 only): single-CTA MMA, clusters along N
  if (d.epi == kEpiLnFull) {
    if constexpr (sizeof(TI) == 2) {
      if (!amn && !bmn) {
        if (bn == 256) return launch<TI, false, false, kEpiLnFull, 256, false>(q, np, s);
        return launch<TI, false, false, kEpiLnFull, 128, false>(q, np, s);
      }
    }
    set_error("gemm_tc: fused LayerNorm needs bf16 K-major operands");
    return UL_ERR_VALUE;
  }
#define UL_TC_BRES_MAX(EPI, BN) Smem<BN, false, (int)sizeof(OutT<TI, EPI>), EPI, true>::kBresMax
#define UL_TC_BRES_MAX_P(EPI, BN) Smem<BN, true, (int)sizeof(OutT<TI, EPI>), EPI, true>::kBresMax
#define UL_TC_BN(AMN, BMN, EPI, BN)                                                          \
  if (!AMN && bres_fits(BN, UL_TC_BRES_MAX(EPI, BN)))                                       \
    return launch<TI, AMN, BMN, EPI, BN, false, true>(q, np, s);                            \
  if (!AMN && bres_fits_pair(BN, UL_TC_BRES_MAX_P(EPI, BN)))                                \
    return launch<TI, AMN, BMN, EPI, BN, true, true>(q, np, s);                             \
  if (BN == 256 && !AMN && bres128 && bres_fits(128, UL_TC_BRES_MAX(EPI, 128)))             \
    return launch<TI, AMN, BMN, EPI, 128, false, true>(q, np, s);                           \
  if (pair) return launch<TI, AMN, BMN, EPI, BN, true>(q, np, s);                           \
  return launch<TI, AMN, BMN, EPI, BN, false>(q, np, s);
#define UL_TC_CASE(AMN, BMN, EPI)                 \
  if (amn == AMN && bmn == BMN && d.epi == EPI) { \
    if (bn == 256) {                              \
      UL_TC_BN(AMN, BMN, EPI, 256)                \
    }                                             \
    UL_TC_BN(AMN, BMN, EPI, 128)                  \
  }
  UL_TC_CASE(false, false, kEpiBias)
  UL_TC_CASE(false, false, kEpiBiasLn)
  UL_TC_CASE(false, false, kEpiBiasElu)
  UL_TC_CASE(false, false, kEpiStore)
  UL_TC_CASE(false, true, kEpiEluGrad)
  UL_TC_CASE(false, true, kEpiStore)
  UL_TC_CASE(true, true, kEpiStore)
#undef UL_TC_CASE
#undef UL_TC_BN
#undef UL_TC_BRES_MAX
#undef UL_TC_BRES_MAX_P
  set_error("gemm_tc: unsupported layout/epilogue combination");
  return UL_ERR_VALUE;
}

}  // namespace tc

int tc_bk(int dtype) { return dtype == kBf16 ? tc::Op<__nv_bfloat16>::BK : tc::Op<float>::BK; }

bool tc_eligible(const GemmDesc& d) {
  const int eb = d.dtype == kBf16 ? 2 : 4;
  const int ob = (d.dtype == kBf16 && (d.epi == kEpiBiasElu || d.epi == kEpiEluGrad ||
                                       d.epi == kEpiBiasLn || d.epi == kEpiLnFull)) ? 2 : 4;
  auto al = [](const void* p) { return ((uintptr_t)p & 15) == 0; };
  // bf16 runs every hidden GEMM on the tensor cores (TMA zero-fills partial
  // tiles); tf32 keeps tiny shapes on the SIMT kernel
  const bool big = d.dtype == kBf16 || (d.M >= 128 && d.N >= 64 && d.K >= 32);
  return big && d.M >= 1 && d.N >= 1 && d.K >= 1 && d.M < (1ll << 31) && d.N < (1ll << 31) &&
         d.K < (1ll << 31) && al(d.A) && al(d.B) && al(d.C) && (d.lda * eb % 16 == 0) &&
         (d.ldb * eb % 16 == 0) && (d.ldc * ob % 16 == 0) &&
         (d.epi != kEpiEluGrad || (al(d.aux) && d.ldaux * ob % 16 == 0)) &&
         !(d.a_kmajor == false && d.b_kmajor == true);
}

int tc_num_splits(int64_t K, int splits, int dtype) {
  const int bk = tc_bk(dtype);
  splits = splits < 1 ? 1 : splits;
  const int64_t kps = ceil_div(ceil_div(K, splits), bk) * bk;
  return (int)ceil_div(K > 0 ? K : 1, kps);
}

static tc::Prob prob_of(const GemmDesc& d, int ones_col) {
  const int bk = tc_bk(d.dtype);
  const int splits = d.splits < 1 ? 1 : d.splits;
  tc::Prob q;
  q.d = &d;
  q.kps = (int)(ceil_div(ceil_div(d.K, splits), bk) * bk);
  q.zs = (int)ceil_div(d.K > 0 ? d.K : 1, q.kps);
  q.ones_col = ones_col < 0 ? d.ones_col : ones_col;
  return q;
}

// Same contract as gemm_f32 (split partials [zs][M][ldc] at C when splits >
// 1); `ones_col` >= 0 additionally writes 1.0 into that column.
// ---------------------------------------------------------------- 3xTF32
// a = hi + lo with hi = rna_tf32(a) (exactly representable in tf32) and lo =
// a - hi (exact in fp32); a*b ~= hi_a hi_b + hi_a lo_b + lo_a hi_b, the
// dropped lo*lo term and lo's own tf32 rounding are ~2^-22 relative -- fp32
// parity.  The three products are ONE tf32 GEMM over a tripled K:
// A' = [A_hi | A_hi | A_lo], B' = [B_hi | B_lo | B_hi] along K (columns of a
// K-major operand, rows of an MN-major one; each block zero-padded to Kp), so
// every epilogue, split-K and layout of the tf32 kernel is reused unchanged.
namespace {
__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t u;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(u) : "f"(x));
  return __uint_as_float(u);
}

// K' = zs x [hi | hi-or-lo | ...] blocks: split-K chunk z of the original
// operand (K range [z Kp, (z+1) Kp)) becomes K' range [3 z Kp, 3 (z+1) Kp)
// holding its three parts, so a split-K GEMM keeps the same zs partials.
// Memory-bound: 4 K' elements (one float4) per thread, the block / chunk
// decomposition computed once per float4 (Kp % 32 == 0) in 32-bit math.
__device__ __forceinline__ float split_part(float v, int b, int lo_mask) {
  const float hi = tf32_rna(v);
  return ((lo_mask >> b) & 1) ? v - hi : hi;
}

// K-major operand [R][K] -> [R][K3]
__global__ void split3_cols_kernel(const float* __restrict__ src, int64_t lds, int R, int K,
                                   int Kp, int K3, int lo_mask, float* __restrict__ dst,
                                   int64_t ldd) {
  const int q4 = K3 / 4;  // float4 per row (K3 % 4 == 0)
  const int64_t total = (int64_t)R * q4;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += stride) {
    const int r = (int)(i / q4), j = 4 * (int)(i - (int64_t)r * q4);
    const int z = j / (3 * Kp), rem = j - z * 3 * Kp, b = rem / Kp;
    const int k0 = z * Kp + rem - b * Kp;
    const float* s = src + (int64_t)r * lds;
    float4 o;
    o.x = split_part(k0 < K ? s[k0] : 0.f, b, lo_mask);
    o.y = split_part(k0 + 1 < K ? s[k0 + 1] : 0.f, b, lo_mask);
    o.z = split_part(k0 + 2 < K ? s[k0 + 2] : 0.f, b, lo_mask);
    o.w = split_part(k0 + 3 < K ? s[k0 + 3] : 0.f, b, lo_mask);
    *reinterpret_cast<float4*>(dst + (int64_t)r * ldd + j) = o;
  }
}

// MN-major operand [K][C] -> [K3][C]: dst row j <- source row k (or zeros)
__global__ void split3_rows_kernel(const float* __restrict__ src, int64_t lds, int K, int C,
                                   int Kp, int K3, int lo_mask, float* __restrict__ dst,
                                   int64_t ldd) {
  const int c4 = (C + 3) / 4;
  for (int j = blockIdx.y; j < K3; j += gridDim.y) {
    const int z = j / (3 * Kp), rem = j - z * 3 * Kp, b = rem / Kp;
    const int k = z * Kp + rem - b * Kp;
    const float* s = src + (int64_t)k * lds;
    float* d = dst + (int64_t)j * ldd;
    for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < c4; q += gridDim.x * blockDim.x) {
      const int c = 4 * q;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (k < K) {
        if (c + 3 < C && ((lds & 3) == 0)) v = *reinterpret_cast<const float4*>(s + c);
        else {
          v.x = s[c];
          v.y = c + 1 < C ? s[c + 1] : 0.f;
          v.z = c + 2 < C ? s[c + 2] : 0.f;
          v.w = c + 3 < C ? s[c + 3] : 0.f;
        }
      }
      float4 o = make_float4(split_part(v.x, b, lo_mask), split_part(v.y, b, lo_mask),
                             split_part(v.z, b, lo_mask), split_part(v.w, b, lo_mask));
      if (c + 3 < C || ((ldd & 3) == 0 && c + 3 < ldd)) {
        *reinterpret_cast<float4*>(d + c) = o;
      } else {
        d[c] = o.x;
        if (c + 1 < C) d[c + 1] = o.y;
        if (c + 2 < C) d[c + 2] = o.z;
      }
    }
  }
}

float* g_x3 = nullptr;
size_t g_x3_cap = 0;
}  // namespace

// Grows by allocating a larger buffer; a replaced buffer is never freed,
// because CUDA graphs captured earlier keep its address baked in.
int x3_reserve(size_t floats) {
  if (floats <= g_x3_cap) return UL_OK;
  float* nb = nullptr;
  UL_CUDA(cudaMalloc(&nb, floats * sizeof(float)));
  g_x3 = nb;
  g_x3_cap = floats;
  return UL_OK;
}

int gemm_tc(const GemmDesc& d, int ones_col, cudaStream_t s);

static int gemm_tc_x3(const GemmDesc& d, int ones_col, cudaStream_t s) {
  const int64_t splits = d.splits < 1 ? 1 : d.splits;
  const int64_t Kp = ceil_div(ceil_div(d.K, splits), 32) * 32;  // per split, tf32 BK multiple
  const int64_t zs = ceil_div(d.K > 0 ? d.K : 1, Kp);
  const int64_t K3 = 3 * Kp * zs;
  // stored shapes (rows R x cols C) of the operands
  const int64_t Ra = d.a_kmajor ? d.M : d.K, Ca = d.a_kmajor ? d.K : d.M;
  const int64_t Rb = d.b_kmajor ? d.N : d.K, Cb = d.b_kmajor ? d.K : d.N;
  const int64_t lda2 = d.a_kmajor ? K3 : d.lda, ldb2 = d.b_kmajor ? K3 : d.ldb;
  const int64_t na = d.a_kmajor ? d.M * K3 : K3 * d.lda;
  const int64_t nb = d.b_kmajor ? d.N * K3 : K3 * d.ldb;
  const size_t need = (size_t)(ceil_div(na, 64) * 64 + nb);
  if (need > g_x3_cap) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(s, &cs);
    UL_CHECK_ARG(cs == cudaStreamCaptureStatusNone,
                 "3xTF32: split scratch (%zu floats) not reserved before graph capture", need);
    UL_TRY(x3_reserve(need));
  }
  float* a2 = g_x3;
  float* b2 = g_x3 + ceil_div(na, 64) * 64;
  auto split = [&](const float* srcp, int64_t lds, bool kmajor, int64_t R, int64_t C, int mask,
                   float* dst, int64_t ldd) -> int {
    if (kmajor) {  // [R][K] -> [R][K3]
      int64_t b = ceil_div(R * (K3 / 4), 256);
      b = b > 16 * kNumSMs ? 16 * kNumSMs : (b < 1 ? 1 : b);
      split3_cols_kernel<<<(unsigned)b, 256, 0, s>>>(srcp, lds, (int)R, (int)d.K, (int)Kp,
                                                     (int)K3, mask, dst, ldd);
      return check_launch("split3_cols_kernel");
    }
    // [K][C] -> [K3][C]
    const int64_t c4 = ceil_div(C, 4);
    const unsigned gx = (unsigned)ceil_div(c4, 128);
    int64_t gy = (16 * kNumSMs) / (int64_t)gx;
    gy = gy > K3 ? K3 : (gy < 1 ? 1 : gy);
    split3_rows_kernel<<<dim3(gx, (unsigned)gy), 128, 0, s>>>(srcp, lds, (int)d.K, (int)C,
                                                              (int)Kp, (int)K3, mask, dst, ldd);
    return check_launch("split3_rows_kernel");
  };
  UL_TRY(split(d.A, d.lda, d.a_kmajor, Ra, Ca, 0b100, a2, lda2));
  UL_TRY(split(d.B, d.ldb, d.b_kmajor, Rb, Cb, 0b010, b2, ldb2));
  GemmDesc e = d;
  e.x3 = false;
  e.A = a2;
  e.lda = lda2;
  e.B = b2;
  e.ldb = ldb2;
  e.K = K3;
  e.splits = (int)zs;
  return gemm_tc(e, ones_col, s);
}

int gemm_tc(const GemmDesc& d, int ones_col, cudaStream_t s) {
  if (d.M == 0 || d.N == 0) return UL_OK;
  if (d.x3) return gemm_tc_x3(d, ones_col, s);
  const tc::Prob q = prob_of(d, ones_col);
  if (d.dtype == kBf16) return tc::dispatch<__nv_bfloat16>(&q, 1, s);
  return tc::dispatch<float>(&q, 1, s);
}

// Independent GEMMs in as few persistent launches as their compatibility
// allows: problems sharing dtype, operand layouts and epilogue (at most one
// with column sums) run as one batch of up to tc::kMaxProb.  Used for the
// deferred dW GEMMs of a backward pass (every layer of both networks).
int gemm_tc_batch(const GemmDesc* d, int n, cudaStream_t s) {
  bool done[64] = {};
  UL_CHECK_ARG(n >= 0 && n <= 64, "gemm_tc_batch: at most 64 problems");
  for (int i = 0; i < n; ++i)
    if (d[i].x3) {  // one at a time through the split scratch
      for (int j = 0; j < n; ++j) UL_TRY(gemm_tc(d[j], -1, s));
      return UL_OK;
    }
  for (int i = 0; i < n; ++i) done[i] = d[i].M == 0 || d[i].N == 0;
  for (int i = 0; i < n; ++i) {
    if (done[i]) continue;
    tc::Prob q[tc::kMaxProb];
    int nq = 0;
    bool cs = false;
    for (int j = i; j < n && nq < tc::kMaxProb; ++j) {
      if (done[j]) continue;
      const GemmDesc& a = d[i];
      const GemmDesc& b = d[j];
      const bool csj = b.csum_part != nullptr;
      if (b.dtype != a.dtype || b.a_kmajor != a.a_kmajor || b.b_kmajor != a.b_kmajor ||
          b.epi != a.epi || (cs && csj))
        continue;
      cs = cs || csj;
      q[nq++] = prob_of(b, -1);
      done[j] = true;
    }
    if (d[i].dtype == kBf16) UL_TRY(tc::dispatch<__nv_bfloat16>(q, nq, s));
    else UL_TRY(tc::dispatch<float>(q, nq, s));
  }
  return UL_OK;
}

// Two independent GEMMs (e.g. the actor's and the critic's layer) in one
// persistent launch when they share dtype, layouts, epilogue, tile width and
// CTA pairing; otherwise two launches.  Each desc's ones_col applies.
// Stacked bias+ELU layers of up to 2 networks as ONE launch (chained layers):
// d[net * L + l] = layer l of net `net` (bf16, K-major operands, 256-wide N
// tiles, layer l's A = layer l - 1's C).  A CTA runs whole row chains -- every
// layer of one 128-row M tile, the next layer's tiles waiting only for this
// CTA's own stores of the layer below -- so the per-launch fill / drain and
// the grid-wide dependency wait between layers disappear.
int gemm_tc_chain(const GemmDesc* d, int nets, int L, cudaStream_t s) {
  UL_CHECK_ARG(nets >= 1 && nets <= 2 && L >= 1 && L <= tc::kMaxChainL, "chain: shape");
  tc::Prob q[tc::kMaxProb];
  for (int i = 0; i < nets * L; ++i) {
    UL_CHECK_ARG(d[i].dtype == kBf16 && d[i].a_kmajor && d[i].b_kmajor && d[i].epi == kEpiBiasElu &&
                     (d[i].splits <= 1) && !d[i].x3,
                 "chain: layers must be bf16 bias+ELU GEMMs with K-major operands");
    q[i] = prob_of(d[i], -1);
  }
  const tc::ChainSpec cs{nets, L};
  return tc::launch<__nv_bfloat16, false, false, kEpiBiasElu, 256, false>(q, nets * L, s, &cs);
}

static bool group_compatible(const GemmDesc& d0, const GemmDesc& d1) {
  return d0.dtype == d1.dtype && d0.a_kmajor == d1.a_kmajor && d0.b_kmajor == d1.b_kmajor &&
         d0.epi == d1.epi && tc::bn_of(d0) == tc::bn_of(d1) &&
         (ceil_div(d0.M, tc::BM) >= 2) == (ceil_div(d1.M, tc::BM) >= 2) &&
         !(d0.csum_part && d1.csum_part) &&
         (d0.epi != kEpiLnFull || ceil_div(d0.N, tc::bn_of(d0)) == ceil_div(d1.N, tc::bn_of(d1)));
}

// n (<= kMaxProb) independent GEMMs -- the same layer of several networks --
// in one persistent launch when all share dtype, layouts, epilogue, tile
// width and CTA pairing (and at most one carries a column-sum output);
// otherwise one launch each.  Each desc's ones_col applies.
int gemm_tc_group_n(const GemmDesc* d, int n, cudaStream_t s) {
  UL_CHECK_ARG(n >= 1 && n <= tc::kMaxProb, "gemm_tc_group_n: 1..8 problems");
  bool split = n == 1;
  int ncs = 0;
  for (int k = 0; k < n; ++k) {
    split = split || d[k].M == 0 || d[k].N == 0 || d[k].x3 ||  // (3xTF32: one split scratch)
            !group_compatible(d[0], d[k]);
    ncs += d[k].csum_part != nullptr;
  }
  if (split || ncs > 1) {
    for (int k = 0; k < n; ++k)
      if (d[k].M != 0 && d[k].N != 0) UL_TRY(gemm_tc(d[k], -1, s));
    return UL_OK;
  }
  tc::Prob q[tc::kMaxProb];
  for (int k = 0; k < n; ++k) q[k] = prob_of(d[k], -1);
  if (d[0].dtype == kBf16) return tc::dispatch<__nv_bfloat16>(q, n, s);
  return tc::dispatch<float>(q, n, s);
}

int gemm_tc_group(const GemmDesc& d0, const GemmDesc& d1, cudaStream_t s) {
  const GemmDesc d[2] = {d0, d1};
  return gemm_tc_group_n(d, 2, s);
}

}  // namespace ul

// Diagnostics: copy the trace buffer (kTraceSlots x u64: CTA-0 timestamps in ns,
// role wait-cycle sums at 128..133).
extern "C" int ul_tc_trace(unsigned long long* host_out) {
  unsigned long long* b = ul::tc::trace_buffer();
  UL_CHECK_ARG(b != nullptr, "tc trace: set UL_TC_TRACE=1 before the first GEMM");
  UL_CUDA(cudaMemcpy(host_out, b, ul::tc::kTraceSlots * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
  return UL_OK;
}

extern "C" int ul_tc_trace_reset(void) {
  unsigned long long* b = ul::tc::trace_buffer();
  UL_CHECK_ARG(b != nullptr, "tc trace: set UL_TC_TRACE=1 before the first GEMM");
  UL_CUDA(cudaMemset(b, 0, ul::tc::kTraceSlots * sizeof(unsigned long long)));
  return UL_OK;
}

// Test hook: one tcgen05 GEMM, same layout/epilogue codes as ul_gemm_f32.
// dtype 0: fp32 operands (kind::tf32), 1: bf16 operands (kind::f16); with
// dtype 1 the ELU / ELU-gradient epilogues read and write bf16.
extern "C" int ul_gemm_tc(int layout, int epi, int64_t M, int64_t N, int64_t K, const void* A,
                          int64_t lda, const void* B, int64_t ldb, void* C, int64_t ldc,
                          const float* bias, const void* aux, int64_t ldaux, int splits, int dtype,
                          void* stream) {
  ul::GemmDesc g{};
  g.M = M; g.N = N; g.K = K;
  g.A = (const float*)A; g.lda = lda; g.B = (const float*)B; g.ldb = ldb;
  g.C = (float*)C; g.ldc = ldc;
  g.bias = bias; g.aux = (const float*)aux; g.ldaux = ldaux;
  g.a_kmajor = layout & 1; g.b_kmajor = (layout >> 1) & 1; g.epi = epi; g.splits = splits;
  g.dtype = dtype;
  UL_CHECK_ARG(dtype == 0 || dtype == 1, "gemm_tc: dtype must be 0 (fp32/tf32) or 1 (bf16)");
  UL_CHECK_ARG(ul::tc_eligible(g), "gemm_tc: shape/alignment not eligible for tcgen05");
  return ul::gemm_tc(g, -1, ul::as_stream(stream));
}
