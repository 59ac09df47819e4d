// Library-level C ABI: error string, version, device helpers.
#include <stdarg.h>

#include "common.cuh"

namespace ul {
namespace {
thread_local char g_err[1024] = {0};
}
void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}
}  // namespace ul

extern "C" const char* ul_last_error(void) { return ul::g_err; }

extern "C" int ul_version(void) { return UL_ABI_VERSION; }

extern "C" int ul_device_count(int* count) {
  return ul::cuda_status(cudaGetDeviceCount(count), "cudaGetDeviceCount");
}

extern "C" int ul_stream_sync(void* stream) {
  return ul::cuda_status(cudaStreamSynchronize(ul::as_stream(stream)), "cudaStreamSynchronize");
}

// Async copy on the given stream; kind is inferred from the pointers (UVA), so
// pinned-host -> device, device -> pinned-host and device -> device all work.
extern "C" int ul_memcpy_async(void* dst, const void* src, int64_t bytes, void* stream) {
  UL_CHECK_ARG(bytes >= 0, "memcpy: negative size");
  if (bytes == 0) return UL_OK;
  return ul::cuda_status(
      cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyDefault, ul::as_stream(stream)),
      "cudaMemcpyAsync");
}

// Async byte fill of device memory (allocation-time zeroing without a
// framework fill kernel)
extern "C" int ul_memset_async(void* dst, int value, int64_t bytes, void* stream) {
  UL_CHECK_ARG(bytes >= 0, "memset: negative size");
  if (bytes == 0) return UL_OK;
  return ul::cuda_status(cudaMemsetAsync(dst, value, (size_t)bytes, ul::as_stream(stream)),
                         "cudaMemsetAsync");
}

extern "C" int ul_memcpy2d_async(void* dst, int64_t dpitch, const void* src, int64_t spitch,
                                 int64_t width_bytes, int64_t rows, void* stream) {
  UL_CHECK_ARG(width_bytes >= 0 && rows >= 0 && dpitch >= width_bytes && spitch >= width_bytes,
               "memcpy2d: bad geometry");
  if (width_bytes == 0 || rows == 0) return UL_OK;
  return ul::cuda_status(cudaMemcpy2DAsync(dst, (size_t)dpitch, src, (size_t)spitch,
                                           (size_t)width_bytes, (size_t)rows, cudaMemcpyDefault,
                                           ul::as_stream(stream)),
                         "cudaMemcpy2DAsync");
}

extern "C" int ul_host_alloc_pinned(void** ptr, int64_t bytes) {
  UL_CHECK_ARG(bytes > 0, "pinned alloc: size must be > 0");
  return ul::cuda_status(cudaHostAlloc(ptr, (size_t)bytes, cudaHostAllocPortable),
                         "cudaHostAlloc");
}

extern "C" int ul_host_free_pinned(void* ptr) {
  return ul::cuda_status(cudaFreeHost(ptr), "cudaFreeHost");
}

extern "C" int ul_event_create(void** ev) {
  cudaEvent_t e;
  UL_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  *ev = (void*)e;
  return UL_OK;
}

extern "C" int ul_event_destroy(void* ev) {
  return ul::cuda_status(cudaEventDestroy((cudaEvent_t)ev), "cudaEventDestroy");
}

extern "C" int ul_event_record(void* ev, void* stream) {
  return ul::cuda_status(cudaEventRecord((cudaEvent_t)ev, ul::as_stream(stream)),
                         "cudaEventRecord");
}

extern "C" int ul_stream_wait_event(void* stream, void* ev) {
  return ul::cuda_status(cudaStreamWaitEvent(ul::as_stream(stream), (cudaEvent_t)ev, 0),
                         "cudaStreamWaitEvent");
}

// 1 = complete, 0 = pending
extern "C" int ul_event_query(void* ev, int* done) {
  cudaError_t e = cudaEventQuery((cudaEvent_t)ev);
  if (e == cudaSuccess) {
    *done = 1;
    return UL_OK;
  }
  if (e == cudaErrorNotReady) {
    (void)cudaGetLastError();
    *done = 0;
    return UL_OK;
  }
  return ul::cuda_status(e, "cudaEventQuery");
}

extern "C" int ul_event_sync(void* ev) {
  return ul::cuda_status(cudaEventSynchronize((cudaEvent_t)ev), "cudaEventSynchronize");
}
