// Shared tcgen05 / TMA / mbarrier building blocks of the tensor-core kernels
// (gemm_tc.cu: the general GEMM; fused_mlp.cu: the fused forward chain).
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "internal.cuh"

namespace ul {
namespace tc {

constexpr int BM = 128;

// operand traits: one 128-byte swizzle row holds BK elements of K
template <typename T>
struct Op;
template <>
struct Op<float> {
  static constexpr int kBytes = 4, BK = 32, kChunk = 32;  // kChunk: MN elements per 128 B
  static constexpr uint32_t kFmt = 2;                      // TF32
  // MN-major: 32-byte swizzle atoms (the only legal MN-major tf32 layout)
  static constexpr uint32_t kMnLayout = 1, kMnSbo = 512, kMnKStep = 1024;
};
template <>
struct Op<__nv_bfloat16> {
  static constexpr int kBytes = 2, BK = 64, kChunk = 64;
  static constexpr uint32_t kFmt = 1;  // BF16 under kind::f16
  static constexpr uint32_t kMnLayout = 2, kMnSbo = 1024, kMnKStep = 2048;
};

__device__ __forceinline__ uint32_t su32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar)),
               "r"(bytes)
               : "memory");
}

// Bounded wait: a pipeline bug traps (error surfaces at the next sync) instead
// of hanging the GPU until the host-side timeout.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
#pragma unroll 1
  for (uint32_t spin = 0; spin < (1u << 26); ++spin) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
        "selp.u32 %0, 1, 0, P1;\n"
        "}\n"
        : "=r"(done)
        : "r"(su32(bar)), "r"(parity)
        : "memory");
    if (done) return;
  }
  __trap();
}

// diagnostics (UL_TC_TRACE): wait cycles accumulated per role, summed over
// CTAs into trace slots 128.. (see ul_tc_trace / tools/trace_gemm.py)
constexpr int kTraceSlots = 160;
__device__ __forceinline__ void mbar_wait_acc(uint64_t* bar, uint32_t parity,
                                              unsigned long long* acc) {
  if (acc == nullptr) {
    mbar_wait(bar, parity);
    return;
  }
  const long long t0 = clock64();
  mbar_wait(bar, parity);
  *acc += (unsigned long long)(clock64() - t0);
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(su32(dst)),
      "l"(map), "r"(su32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(su32(dst)),
      "l"(map), "r"(su32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

// UMMA shared-memory matrix descriptor, sm100 version bit.  Layout type 2 =
// SWIZZLE_128B (16-byte atoms), 1 = SWIZZLE_128B_BASE32B (32-byte atoms).
__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo,
                                              uint32_t layout) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)layout << 61;
  return d;
}

template <typename T>
__device__ __forceinline__ void mma(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc,
                                    uint32_t acc) {
  if constexpr (sizeof(T) == 4) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n"
        "}\n" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(idesc), "r"(acc));
  } else {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
        "}\n" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(idesc), "r"(acc));
  }
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   su32(bar))
               : "memory");
}

__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" :::
                   "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t addr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(addr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// ELU on the tensor-core path: exp via ex2.approx (abs. error ~1e-7 near 0,
// far inside the tf32/bf16 GEMM error; the fp32 parity path keeps expm1f)
__device__ __forceinline__ float ex2_ftz(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// 4 instructions: FMUL, MUFU.EX2, FSETP, predicated FADD (very negative z
// flushes to exp = 0; large positive z selects z)
__device__ __forceinline__ float elu_fast(float z) {
  const float e = ex2_ftz(z * 1.4426950408889634f);
  return z > 0.f ? z : e - 1.f;
}

// ELU of two values with one packed f16x2 MUFU.EX2 (half the SFU work of two
// f32 exps); exp(z) - 1 for z <= 0 lies in (-1, 0], where f16's 11-bit
// significand is finer than the bf16 the result is stored in.
__device__ __forceinline__ void elu_pair_f16(float& z0, float& z1) {
  const float t0 = fmaxf(z0, -16.f) * 1.4426950408889634f;  // log2(e); ex2(-23) ~ 1e-7
  const float t1 = fmaxf(z1, -16.f) * 1.4426950408889634f;
  uint32_t h;
  asm("{\n"
      ".reg .b32 t;\n"
      "cvt.rn.f16x2.f32 t, %2, %1;\n"
      "ex2.approx.f16x2 %0, t;\n"
      "}\n"
      : "=r"(h)
      : "f"(t0), "f"(t1));
  __half2 e2 = *reinterpret_cast<__half2*>(&h);
  const float2 ef = __half22float2(e2);
  z0 = z0 > 0.f ? z0 : ef.x - 1.f;
  z1 = z1 > 0.f ? z1 : ef.y - 1.f;
}

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}
__device__ __forceinline__ float bf_lo(uint32_t u) { return __uint_as_float(u << 16); }
__device__ __forceinline__ float bf_hi(uint32_t u) { return __uint_as_float(u & 0xFFFF0000u); }

// ------------------------------------------------------------------ host side
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                              const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                              const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

inline EncodeFn encode_fn() {
  static EncodeFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
  }
  return fn;
}

// 2-D (planes == 0) or 3-D tensor map over a row-major [planes][outer][inner]
// array with row pitch `ld` elements and plane pitch outer * ld; box
// {box_inner, box_outer(, 1)}; OOB -> zero.
inline int make_map(CUtensorMap* map, const void* base, int elem_bytes, int64_t inner, int64_t outer,
             int64_t ld, int box_inner, int box_outer, CUtensorMapSwizzle sw,
             int64_t planes = 0) {
  EncodeFn fn = encode_fn();
  if (!fn) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return UL_ERR_CUDA;
  }
  if (((uintptr_t)base & 15) || ((ld * elem_bytes) & 15)) {
    set_error("tensor map: base/pitch not 16-byte aligned");
    return UL_ERR_VALUE;
  }
  cuuint64_t dims[3] = {(cuuint64_t)inner, (cuuint64_t)outer, (cuuint64_t)planes};
  cuuint64_t strides[2] = {(cuuint64_t)(ld * elem_bytes), (cuuint64_t)(outer * ld * elem_bytes)};
  cuuint32_t box[3] = {(cuuint32_t)box_inner, (cuuint32_t)box_outer, 1u};
  cuuint32_t es[3] = {1u, 1u, 1u};
  CUresult r = fn(map,
                  elem_bytes == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                  : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16,
                  planes > 0 ? 3 : 2, const_cast<void*>(base), dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (%d)", (int)r);
    return UL_ERR_CUDA;
  }
  return UL_OK;
}


}  // namespace tc
}  // namespace ul
