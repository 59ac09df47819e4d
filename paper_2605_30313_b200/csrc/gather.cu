// K4 minibatch gather, K5 replay ring insert, K6 replay sample gather,
// plus the device minibatch permutation used in performance mode.
//
// Replaces the fancy-index copies of R:algos/ppo.py:161-176 (obs[idx], ...),
// ReplayStorage.insert R:replaypath/storage.py:76-104 and the sampled-row
// copy of _read_rows_locked :106-110 / DeviceReplayCache :245-249.
//
// One launch gathers several arrays that share an index vector ("descs"):
// the work of each desc is flattened to (row, 16/8/4-byte unit) items so a
// warp always streams contiguous bytes of a row, whatever the row width
// (obs 940 B, actions 48 B, scalars 4 B).  Algorithmic bytes: 2 x rows x
// row_bytes + 8 B/index.
#include <cuda_bf16.h>

#include "internal.cuh"

namespace ul {
namespace {

constexpr int kMaxDesc = 12;
// row groups in flight per warp (8 measured slower: fewer resident warps)
constexpr int kRowGroups = 4;

struct GatherTable {
  const char* src[kMaxDesc];
  char* dst[kMaxDesc];
  int64_t src_stride[kMaxDesc];  // bytes
  int64_t dst_stride[kMaxDesc];  // bytes
  int64_t units[kMaxDesc];       // units per row
  int unit[kMaxDesc];            // unit bytes (16, 8 or 4)
  int64_t ones[kMaxDesc];        // byte offset of a float set to 1.0 in each row, -1 none
  int cvt[kMaxDesc];             // 1: fp32 source rows -> bf16 destination rows
  int lpr_shift[kMaxDesc];       // log2(lanes per row)
  int blk0[kMaxDesc + 1];        // desc d owns blocks [blk0[d], blk0[d+1]) of the 1-D grid
  int ndesc;
};

template <int U>
struct Vec;
template <>
struct Vec<16> { using T = uint4; };
template <>
struct Vec<8> { using T = uint2; };
template <>
struct Vec<4> { using T = uint32_t; };

// float 1.0 into 4-byte lane e of a register vector (selects; a dynamic
// index would push the vector to local memory)
__device__ __forceinline__ void set_one(uint4& v, int e) {
  v.x = e == 0 ? 0x3f800000u : v.x;
  v.y = e == 1 ? 0x3f800000u : v.y;
  v.z = e == 2 ? 0x3f800000u : v.z;
  v.w = e == 3 ? 0x3f800000u : v.w;
}
__device__ __forceinline__ void set_one(uint2& v, int e) {
  v.x = e == 0 ? 0x3f800000u : v.x;
  v.y = e == 1 ? 0x3f800000u : v.y;
}
__device__ __forceinline__ void set_one(uint32_t& v, int) { v = 0x3f800000u; }

// One desc's rows.  A warp owns 32 / lpr rows at a time, lpr = a power of two
// >= units per row (<= 32) lanes per row: lanes stream contiguous 16/8/4-byte
// units of a row, no per-unit division, and R row groups are in flight per
// warp (all loads issued before any store).  CVT: 16-byte fp32 source units
// become 8-byte bf16 destination units.
template <int U, bool CVT>
__device__ __forceinline__ void copy_rows(const char* __restrict__ src, char* __restrict__ dst,
                                          int64_t sst, int64_t dstr, int upr, int lpr_shift,
                                          const int64_t* __restrict__ idx, int64_t n,
                                          int64_t modulo, int64_t lo, int64_t hi, int* err,
                                          int64_t ones, int blk, int nblk) {
  using T = typename Vec<U>::T;
  constexpr int R = kRowGroups;
  const int lane = threadIdx.x & 31;
  const int lpr = 1 << lpr_shift, rpw = 32 >> lpr_shift;
  const int sub = lane & (lpr - 1);
  const int64_t gw = ((int64_t)blk * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)nblk * blockDim.x) >> 5;
  const int64_t step = nw * rpw;  // rows between a warp's consecutive row groups
  const int ones_u = ones >= 0 ? (int)(ones / U) : -1;
  const int ones_e = ones >= 0 ? (int)((ones % U) / 4) : 0;
  // the next row group's indices are loaded one iteration ahead, so a row's
  // address is ready when its loads issue (index and row round trips overlap)
  int64_t nxt[R];
  {
    const int64_t b0 = gw * rpw + (lane >> lpr_shift);
#pragma unroll
    for (int k = 0; k < R; ++k) {
      const int64_t r = b0 + k * step;
      nxt[k] = r < n ? (idx ? __ldg(idx + r) : r) : 0;
    }
  }
  for (int64_t base = gw * rpw + (lane >> lpr_shift); base < n; base += step * R) {
    const char* sp[R];
    char* dp[R];
    int64_t cur[R];
#pragma unroll
    for (int k = 0; k < R; ++k) {
      cur[k] = nxt[k];
      const int64_t r = base + step * R + k * step;
      nxt[k] = r < n ? (idx ? __ldg(idx + r) : r) : 0;
    }
#pragma unroll
    for (int k = 0; k < R; ++k) {
      const int64_t r = base + k * step;
      sp[k] = nullptr;
      dp[k] = dst + r * dstr;
      if (r >= n) continue;
      int64_t s = cur[k];
      if (s < lo || s >= hi) {
        if (err && sub == 0) atomicOr(err, 1);
        continue;
      }
      if (modulo > 0) s = (modulo & (modulo - 1)) == 0 ? (s & (modulo - 1)) : s % modulo;
      sp[k] = src + s * sst;
    }
    // two units per lane per row in flight (rows up to 64 units = 1 KB of
    // 16-byte units), then any remainder
    for (int u0 = sub; u0 < upr; u0 += 2 * lpr) {
      const int u1 = u0 + lpr;
      T v[R][2];
#pragma unroll
      for (int k = 0; k < R; ++k) {
        if (sp[k]) {
          v[k][0] = __ldg(reinterpret_cast<const T*>(sp[k]) + u0);
          if (u1 < upr) v[k][1] = __ldg(reinterpret_cast<const T*>(sp[k]) + u1);
        }
      }
#pragma unroll
      for (int k = 0; k < R; ++k) {
        if (!sp[k]) continue;
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int u = e ? u1 : u0;
          if (u >= upr) continue;
          if constexpr (CVT && U == 4) {  // one fp32 -> one bf16 (4-byte-aligned source rows)
            float f = __uint_as_float(v[k][e]);
            if (u == ones_u) f = 1.f;
            reinterpret_cast<__nv_bfloat16*>(dp[k])[u] = __float2bfloat16_rn(f);
          } else if (CVT) {
            float4 f4 = *reinterpret_cast<float4*>(&v[k][e]);
            float f[4] = {f4.x, f4.y, f4.z, f4.w};
            if (u == ones_u) {  // (selects, no dynamically indexed local array)
              f[0] = ones_e == 0 ? 1.f : f[0];
              f[1] = ones_e == 1 ? 1.f : f[1];
              f[2] = ones_e == 2 ? 1.f : f[2];
              f[3] = ones_e == 3 ? 1.f : f[3];
            }
            __nv_bfloat162 a = __floats2bfloat162_rn(f[0], f[1]);
            __nv_bfloat162 b = __floats2bfloat162_rn(f[2], f[3]);
            uint2 o;
            o.x = *reinterpret_cast<uint32_t*>(&a);
            o.y = *reinterpret_cast<uint32_t*>(&b);
            reinterpret_cast<uint2*>(dp[k])[u] = o;
          } else {
            if (u == ones_u) set_one(v[k][e], ones_e);
            reinterpret_cast<T*>(dp[k])[u] = v[k][e];
          }
        }
      }
    }
  }
}

// CVT4: some desc converts 4-byte-aligned rows one float per lane (a separate
// instantiation, so the common launch keeps its register budget)
template <bool CVT4>
__global__ void __launch_bounds__(256) gather_kernel(GatherTable t,
                                                     const int64_t* __restrict__ idx, int64_t n,
                                                     int64_t modulo, int64_t lo, int64_t hi,
                                                     int* err) {
  pdl_trigger();
  pdl_wait();
  // this block's desc: blocks are apportioned to descs by their row work
  int d = 0;
  while (d + 1 < t.ndesc && (int)blockIdx.x >= t.blk0[d + 1]) ++d;
  const int blk = (int)blockIdx.x - t.blk0[d], nblk = t.blk0[d + 1] - t.blk0[d];
  const int upr = (int)t.units[d], sh = t.lpr_shift[d];
  if (t.cvt[d]) {
    if (!CVT4 || t.unit[d] == 16)
      copy_rows<16, true>(t.src[d], t.dst[d], t.src_stride[d], t.dst_stride[d], upr, sh, idx, n,
                          modulo, lo, hi, err, t.ones[d], blk, nblk);
    else
      copy_rows<4, true>(t.src[d], t.dst[d], t.src_stride[d], t.dst_stride[d], upr, sh, idx, n,
                         modulo, lo, hi, err, t.ones[d], blk, nblk);
    return;
  }
  switch (t.unit[d]) {
    case 16:
      copy_rows<16, false>(t.src[d], t.dst[d], t.src_stride[d], t.dst_stride[d], upr, sh, idx, n,
                           modulo, lo, hi, err, t.ones[d], blk, nblk);
      break;
    case 8:
      copy_rows<8, false>(t.src[d], t.dst[d], t.src_stride[d], t.dst_stride[d], upr, sh, idx, n,
                          modulo, lo, hi, err, t.ones[d], blk, nblk);
      break;
    default:
      copy_rows<4, false>(t.src[d], t.dst[d], t.src_stride[d], t.dst_stride[d], upr, sh, idx, n,
                          modulo, lo, hi, err, t.ones[d], blk, nblk);
  }
}

int64_t gather_cap_blocks() {
  static int64_t cap = -1;
  if (cap < 0) {
    const char* e = getenv("UL_GATHER_BLOCKS_PER_SM");
    cap = (int64_t)(e ? atoi(e) : 8) * kNumSMs;  // 8 measured best (minibatch 4.3 TB/s)
  }
  return cap;
}

int unit_for(uintptr_t a, uintptr_t b, int64_t s1, int64_t s2, int64_t rb) {
  for (int u = 16; u >= 4; u >>= 1)
    if (a % u == 0 && b % u == 0 && s1 % u == 0 && s2 % u == 0 && rb % u == 0) return u;
  return 0;
}

// ------------------------------------------------- device permutation (perf mode)
// Keyed Feistel bijection on [0, 2^(2h)) + cycle walking into [0, n).  Not the
// numpy Philox shuffle (that stream is sequential); used only when the caller
// opts into device-generated minibatch indices.
__device__ __forceinline__ uint32_t mix32(uint32_t x, uint32_t k) {
  x ^= k;
  x *= 0x9E3779B1u;
  x ^= x >> 15;
  x *= 0x85EBCA77u;
  x ^= x >> 13;
  return x;
}

__global__ void feistel_perm_kernel(int64_t n, int half_bits, uint64_t seed, int64_t* out) {
  const uint32_t mask = (1u << half_bits) - 1u;
  const uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    uint64_t x = (uint64_t)i;
    do {
      uint32_t L = (uint32_t)(x >> half_bits) & mask, R = (uint32_t)x & mask;
#pragma unroll
      for (int r = 0; r < 6; ++r) {
        const uint32_t F = mix32(R + (uint32_t)r * 0x632BE5ABu, (r & 1) ? k1 : k0) & mask;
        const uint32_t nl = R;
        R = L ^ F;
        L = nl;
      }
      x = ((uint64_t)L << half_bits) | R;
    } while (x >= (uint64_t)n);
    out[i] = (int64_t)x;
  }
}

struct PermKeys {
  uint64_t key[16];
};

// blockIdx.y = permutation e (its own key), out rows ld apart
__global__ void feistel_perms_kernel(int64_t n, int half_bits, PermKeys keys, int64_t* out,
                                     int64_t ld) {
  pdl_trigger();
  pdl_wait();
  const uint32_t mask = (1u << half_bits) - 1u;
  const uint64_t seed = keys.key[blockIdx.y];
  const uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
  int64_t* o = out + (int64_t)blockIdx.y * ld;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    uint64_t x = (uint64_t)i;
    do {
      uint32_t L = (uint32_t)(x >> half_bits) & mask, R = (uint32_t)x & mask;
#pragma unroll
      for (int r = 0; r < 6; ++r) {
        const uint32_t F = mix32(R + (uint32_t)r * 0x632BE5ABu, (r & 1) ? k1 : k0) & mask;
        const uint32_t nl = R;
        R = L ^ F;
        L = nl;
      }
      x = ((uint64_t)L << half_bits) | R;
    } while (x >= (uint64_t)n);
    o[i] = (int64_t)x;
  }
}

}  // namespace
}  // namespace ul

namespace ul {
// Gather rows of up to 12 arrays by one index vector (see ul_gather_rows);
// cvt (may be null): per desc, 1 = fp32 source rows written as bf16 (row_bytes
// counts source bytes, a multiple of 16; destination rows are half as wide).
int gather_rows(int ndesc, const void* const* src, void* const* dst, const int64_t* src_stride,
                const int64_t* dst_stride, const int64_t* row_bytes, const int64_t* ones_byte,
                const int* cvt, const int64_t* idx, int64_t n, int64_t modulo, int64_t lo,
                int64_t hi, int* err, cudaStream_t stream,
                int64_t cap_blocks) {
  UL_CHECK_ARG(ndesc >= 1 && ndesc <= kMaxDesc, "gather: ndesc %d outside [1,%d]", ndesc,
               kMaxDesc);
  UL_CHECK_ARG(n >= 0, "gather: negative row count");
  if (n == 0) return UL_OK;
  GatherTable t{};
  t.ndesc = ndesc;
  int nb_total = 0;
  for (int d = 0; d < ndesc; ++d) {
    const int c = cvt ? cvt[d] : 0;
    int u;
    if (c) {
      // 16-byte fp32 units -> 8-byte bf16 units when the rows allow it, else
      // one float -> one bf16 (4-byte-aligned rows, e.g. unpadded 940 B obs rows)
      if (((uintptr_t)src[d] & 15) == 0 && ((uintptr_t)dst[d] & 7) == 0 &&
          src_stride[d] % 16 == 0 && dst_stride[d] % 8 == 0 && row_bytes[d] % 16 == 0) {
        u = 16;
      } else {
        UL_CHECK_ARG(((uintptr_t)src[d] & 3) == 0 && ((uintptr_t)dst[d] & 1) == 0 &&
                         src_stride[d] % 4 == 0 && dst_stride[d] % 2 == 0 && row_bytes[d] % 4 == 0,
                     "gather: bf16 conversion needs 4-byte source rows (desc %d)", d);
        u = 4;
      }
    } else {
      u = unit_for((uintptr_t)src[d], (uintptr_t)dst[d], src_stride[d], dst_stride[d],
                   row_bytes[d]);
    }
    UL_CHECK_ARG(u > 0, "gather: desc %d not 4-byte aligned", d);
    t.src[d] = (const char*)src[d];
    t.dst[d] = (char*)dst[d];
    t.src_stride[d] = src_stride[d];
    t.dst_stride[d] = dst_stride[d];
    t.unit[d] = u;
    t.units[d] = row_bytes[d] / u;
    t.cvt[d] = c;
    t.ones[d] = ones_byte ? ones_byte[d] : -1;
    UL_CHECK_ARG(t.ones[d] < row_bytes[d], "gather: ones column outside the row");
    UL_CHECK_ARG(t.units[d] < (1 << 30), "gather: row too wide");
    int sh = 0;
    while (sh < 5 && (1 << sh) < t.units[d]) ++sh;
    t.lpr_shift[d] = sh;
    // warps needed for kRowGroups row groups in flight each -> 8-warp blocks
    const int64_t warps = ceil_div(n, (int64_t)(32 >> sh) * kRowGroups);
    int64_t nb = ceil_div(warps, 8);
    const int64_t cap = cap_blocks > 0 ? cap_blocks : gather_cap_blocks();
    nb = nb > cap ? cap : nb;
    t.blk0[d] = nb_total;
    nb_total += (int)nb;
  }
  t.blk0[ndesc] = nb_total;
  bool cvt4 = false;
  for (int d = 0; d < ndesc; ++d) cvt4 = cvt4 || (t.cvt[d] && t.unit[d] == 4);
  if (cvt4)
    return launch_pdl("gather_kernel", gather_kernel<true>, dim3((unsigned)nb_total), dim3(256), 0,
                      stream, t, idx, n, modulo, lo, hi, err);
  return launch_pdl("gather_kernel", gather_kernel<false>, dim3((unsigned)nb_total), dim3(256), 0,
                    stream, t, idx, n, modulo, lo, hi, err);
}
}  // namespace ul

// Gather rows of up to 12 arrays by one index vector.  desc arrays have ndesc
// entries: src/dst device pointers, strides and row widths in BYTES.  Rows are
// src + (idx[i] [% modulo]) * src_stride.  Indices outside [lo, hi) are
// skipped and raise *err (device flag).  idx == NULL gathers rows 0..n-1.
extern "C" int ul_gather_rows(int ndesc, const void* const* src, void* const* dst,
                              const int64_t* src_stride, const int64_t* dst_stride,
                              const int64_t* row_bytes, const int64_t* ones_byte,
                              const int64_t* idx, int64_t n,
                              int64_t modulo, int64_t lo, int64_t hi, int* err, void* stream) {
  return ul::gather_rows(ndesc, src, dst, src_stride, dst_stride, row_bytes, ones_byte, nullptr,
                         idx, n, modulo, lo, hi, err, ul::as_stream(stream));
}

namespace ul {
namespace {
// fp32 rows [rows, lds] (any 4-byte alignment, e.g. the 940-byte H2D landing
// rows) -> bf16 rows [rows, ldd]: thread = 8 output columns (one 16-byte
// store), 8 coalesced 4-byte loads; columns >= width are 0 except `ones`
// (1.0).  One pass over a whole segment field per H2D.
__global__ void __launch_bounds__(256) rows_to_bf16_kernel(const float* __restrict__ src,
                                                           int64_t lds, int width,
                                                           __nv_bfloat16* __restrict__ dst,
                                                           int64_t ldd, int64_t rows, int ones) {
  pdl_trigger();
  pdl_wait();
  const int q8 = (int)(ldd / 8);
  const int64_t total = rows * q8;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / q8;
    const int c0 = (int)(i - r * q8) * 8;
    const float* sr = src + r * lds;
    float v[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int c = c0 + e;
      v[e] = c < width ? __ldg(sr + c) : (c == ones ? 1.f : 0.f);
    }
    uint4 o;
    __nv_bfloat162 p0 = __floats2bfloat162_rn(v[0], v[1]), p1 = __floats2bfloat162_rn(v[2], v[3]);
    __nv_bfloat162 p2 = __floats2bfloat162_rn(v[4], v[5]), p3 = __floats2bfloat162_rn(v[6], v[7]);
    o.x = *reinterpret_cast<uint32_t*>(&p0);
    o.y = *reinterpret_cast<uint32_t*>(&p1);
    o.z = *reinterpret_cast<uint32_t*>(&p2);
    o.w = *reinterpret_cast<uint32_t*>(&p3);
    *reinterpret_cast<uint4*>(dst + r * ldd + c0) = o;
  }
}
}  // namespace
}  // namespace ul

// fp32 rows -> bf16 rows of ldd elements (ldd % 8 == 0, dst 16-byte aligned),
// columns past `width` zero except `ones_col` (1.0; -1 none)
extern "C" int ul_rows_to_bf16(const float* src, int64_t lds, int width, void* dst, int64_t ldd,
                               int64_t rows, int ones_col, void* stream) {
  UL_CHECK_ARG(rows >= 0 && width >= 0 && lds >= width && ldd >= width && ldd % 8 == 0 &&
                   ((uintptr_t)dst & 15) == 0 && ((uintptr_t)src & 3) == 0,
               "rows_to_bf16: bad shape / alignment");
  if (rows == 0) return UL_OK;
  const int64_t total = rows * (ldd / 8);
  int64_t blocks = ul::ceil_div(total, (int64_t)256);
  blocks = blocks > 16 * ul::kNumSMs ? 16 * ul::kNumSMs : blocks;
  return ul::launch_pdl("rows_to_bf16_kernel", ul::rows_to_bf16_kernel, dim3((unsigned)blocks),
                        dim3(256), 0, ul::as_stream(stream), src, lds, width,
                        reinterpret_cast<__nv_bfloat16*>(dst), ldd, rows, ones_col);
}

// ul_gather_rows with per-desc fp32 -> bf16 conversion (no index window)
extern "C" int ul_gather_rows_cvt(int ndesc, const void* const* src, void* const* dst,
                                  const int64_t* src_stride, const int64_t* dst_stride,
                                  const int64_t* row_bytes, const int64_t* ones_byte,
                                  const int* cvt, const int64_t* idx, int64_t n, void* stream) {
  return ul::gather_rows(ndesc, src, dst, src_stride, dst_stride, row_bytes, ones_byte, cvt, idx,
                         n, 0, 0, INT64_MAX, nullptr, ul::as_stream(stream));
}

// Replay ring insert (R:replaypath/storage.py:76-104): write n rows of `width`
// floats at absolute index head.. into ring[cap, width]; rows may live in
// pinned host memory (H2D) or device memory (D2D).  n >= cap keeps only the
// last cap rows, each at its own absolute slot.  1-2 async copies.
extern "C" int ul_ring_insert(float* ring, int64_t cap, int64_t width, int64_t head,
                              const float* rows, int64_t n, void* stream) {
  UL_CHECK_ARG(cap >= 1 && width >= 1 && head >= 0 && n >= 0, "ring insert: bad shape");
  if (n == 0) return UL_OK;
  cudaStream_t s = ul::as_stream(stream);
  int64_t first = head, count = n;
  const float* src = rows;
  if (n >= cap) {
    first = head + n - cap;
    count = cap;
    src = rows + (n - cap) * width;
  }
  const int64_t start = first % cap;
  const int64_t part1 = count < cap - start ? count : cap - start;
  const size_t rb = sizeof(float) * (size_t)width;
  UL_CUDA(cudaMemcpyAsync(ring + start * width, src, rb * part1, cudaMemcpyDefault, s));
  if (count > part1)
    UL_CUDA(cudaMemcpyAsync(ring, src + part1 * width, rb * (count - part1), cudaMemcpyDefault,
                            s));
  return UL_OK;
}

// Several device permutations in one launch (the update's per-epoch orders).
extern "C" int ul_device_permutations(int64_t n, int count, const uint64_t* host_keys,
                                      int64_t* out, int64_t ld, void* stream) {
  UL_CHECK_ARG(n >= 0 && n < (int64_t(1) << 62) && count >= 0 && count <= 16 && ld >= n,
               "permutations: bad n / count / ld");
  if (n == 0 || count == 0) return UL_OK;
  int bits = 1;
  while ((int64_t(1) << (2 * bits)) < n) ++bits;
  ul::PermKeys k{};
  for (int e = 0; e < count; ++e) k.key[e] = host_keys[e];
  int64_t blocks = ul::ceil_div(n, 256);
  const int64_t cap = ul::ceil_div(8 * ul::kNumSMs, count);
  blocks = blocks > cap ? cap : blocks;
  return ul::launch_pdl("feistel_perms_kernel", ul::feistel_perms_kernel,
                        dim3((unsigned)blocks, (unsigned)count), dim3(256), 0,
                        ul::as_stream(stream), n, bits, k, out, ld);
}

// Device minibatch permutation of [0, n) from a 64-bit key (performance mode).
extern "C" int ul_device_permutation(int64_t n, uint64_t key, int64_t* out, void* stream) {
  UL_CHECK_ARG(n >= 0 && n < (int64_t(1) << 62), "permutation: bad n");
  if (n == 0) return UL_OK;
  int bits = 1;
  while ((int64_t(1) << (2 * bits)) < n) ++bits;
  int64_t blocks = ul::ceil_div(n, 256);
  blocks = blocks > 8 * ul::kNumSMs ? 8 * ul::kNumSMs : blocks;
  ul::feistel_perm_kernel<<<(unsigned)blocks, 256, 0, ul::as_stream(stream)>>>(n, bits, key, out);
  return ul::check_launch("feistel_perm_kernel");
}

// f64 -> f32 narrowing of up to 8 device arrays in one launch (the pinned
// float64 per-step scalars of a rollout segment, landed as-is by the H2D:
// no host conversion, R:algos/segment.py field dtypes)
namespace ul {
namespace {
struct NarrowTable {
  const double* src[8];
  float* dst[8];
  int64_t n[8];
  int k;
};
__global__ void narrow_kernel(const __grid_constant__ NarrowTable t) {
  pdl_trigger();
  pdl_wait();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int a = 0; a < t.k; ++a)
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < t.n[a]; i += stride)
      t.dst[a][i] = (float)t.src[a][i];
}
}  // namespace
}  // namespace ul

extern "C" int ul_narrow_f64(int k, const double* const* src, float* const* dst,
                             const int64_t* n, void* stream) {
  UL_CHECK_ARG(k >= 0 && k <= 8, "narrow: 0..8 arrays");
  if (k == 0) return UL_OK;
  ul::NarrowTable t{};
  t.k = k;
  int64_t mx = 1;
  for (int a = 0; a < k; ++a) {
    t.src[a] = src[a];
    t.dst[a] = dst[a];
    t.n[a] = n[a];
    mx = n[a] > mx ? n[a] : mx;
  }
  int64_t blocks = ul::ceil_div(mx, 256);
  blocks = blocks > 4 * ul::kNumSMs ? 4 * ul::kNumSMs : blocks;
  return ul::launch_pdl("narrow_kernel", ul::narrow_kernel, dim3((unsigned)blocks), dim3(256), 0,
                        ul::as_stream(stream), t);
}

