// Shared helpers for libunilite_b200: status codes, error capture, launch checks.
// Status contract (include/unilite_b200.h): 0 OK, 1 ValueError, 2 IndexError,
// 3 DivergenceError, 4 SlotStateError, 5 CUDA error.  No C++ exception ever
// crosses the C ABI.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <utility>

#include "../../include/unilite_b200.h"

namespace ul {

void set_error(const char* fmt, ...);

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

inline int cuda_status(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return UL_OK;
  set_error("%s: %s", what, cudaGetErrorString(e));
  return UL_ERR_CUDA;
}

inline int check_launch(const char* what) { return cuda_status(cudaGetLastError(), what); }

constexpr int kNumSMs = 148;

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Programmatic dependent launch: kernels of the learner chain are launched
// with programmatic stream serialization, so a dependent kernel is scheduled
// while its predecessor drains and only its body waits (pdl_wait) for the
// predecessor's completion.  UL_PDL=0 turns it off.
inline bool pdl_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("UL_PDL");
    on = e ? atoi(e) != 0 : 1;
  }
  return on == 1;
}

// Launch `kern` (which must call pdl_wait() before touching global memory
// another kernel produces or consumes) with the PDL attribute.
template <typename... KArgs, typename... Args>
inline int launch_pdl(const char* what, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                      cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cuda_status(cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...), what);
}

}  // namespace ul

#define UL_CHECK_ARG(cond, ...)            \
  do {                                     \
    if (!(cond)) {                         \
      ::ul::set_error(__VA_ARGS__);        \
      return UL_ERR_VALUE;                 \
    }                                      \
  } while (0)

#define UL_TRY(expr)              \
  do {                            \
    int _st = (expr);             \
    if (_st != UL_OK) return _st; \
  } while (0)

#define UL_CUDA(expr) UL_TRY(::ul::cuda_status((expr), #expr))

// ----------------------------------------------------------------- device side
namespace ul {

// PDL: let the next kernel of the stream launch now / wait for the previous
// kernel's completion and memory.  Both are no-ops without the attribute.
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide sum of a double; result valid in thread 0.  `scratch` >= 32 doubles.
__device__ __forceinline__ double block_sum(double v, double* scratch) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) scratch[wid] = v;
  __syncthreads();
  double r = 0.0;
  if (wid == 0) {
    const int nw = (blockDim.x + 31) >> 5;
    r = lane < nw ? scratch[lane] : 0.0;
    r = warp_sum(r);
  }
  return r;
}

// "Last block done" ticket: returns true in exactly one block, after every
// block has published its partials (threadfence + atomic counter).  The
// counter self-resets so the kernel can be replayed inside a CUDA graph.
__device__ __forceinline__ bool last_block_ticket(unsigned int* counter, unsigned int nblocks) {
  __shared__ bool is_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned int prev = atomicAdd(counter, 1u);
    is_last = (prev == nblocks - 1);
    if (is_last) *counter = 0u;
  }
  __syncthreads();
  if (is_last) __threadfence();
  return is_last;
}

__device__ __forceinline__ float elu_f(float z) { return z > 0.f ? z : expm1f(fmaxf(z, -60.f)); }
__device__ __forceinline__ float elu_grad_from_act(float h) { return fminf(h, 0.f) + 1.f; }

}  // namespace ul
