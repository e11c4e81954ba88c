// peer.cu -- multi-GPU plumbing for the Ulysses exchange over peer memory:
// CUDA IPC export/import of caller-owned device buffers, copy-engine 2-D copies into a peer's buffer,
// and stream-ordered flags (a 32-bit write into a peer's flag word; a stream wait until every flag of
// a set reaches an epoch).  No arithmetic of the method and no NCCL on this path: a rank pushes its
// head slices straight into the peers' receive buffers over NVLink (DMA engines, no SMs), raises one
// flag per destination, and a consumer's compute stream waits on its flags before the kernels read.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <mutex>
#include <string>

#include "../../include/adaspa.h"

namespace {

thread_local std::string g_peer_error;

adaspa_status peer_fail(adaspa_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_peer_error = buf;
  return s;
}

typedef CUresult (*WriteValueFn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
typedef CUresult (*WaitValueFn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
typedef CUresult (*AddrRangeFn)(CUdeviceptr*, size_t*, CUdeviceptr);

template <class F>
F driver_fn(const char* name) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) == cudaSuccess && q == cudaDriverEntryPointSuccess)
    return reinterpret_cast<F>(p);
  return nullptr;
}

struct Driver {
  WriteValueFn write32 = nullptr;
  WaitValueFn wait32 = nullptr;
  AddrRangeFn range = nullptr;
};

const Driver& drv() {
  static Driver d;
  static std::once_flag once;
  std::call_once(once, [] {
    d.write32 = driver_fn<WriteValueFn>("cuStreamWriteValue32");
    d.wait32 = driver_fn<WaitValueFn>("cuStreamWaitValue32");
    d.range = driver_fn<AddrRangeFn>("cuMemGetAddressRange");
  });
  return d;
}

}  // namespace

const char* adaspa_peer_last_error(void) { return g_peer_error.c_str(); }

adaspa_status adaspa_peer_export(const void* dev_ptr, adaspa_peer_handle* out) {
  if (!dev_ptr || !out) return peer_fail(ADASPA_ERR_INVALID_ARG, "dev_ptr and out must not be NULL");
  const Driver& d = drv();
  if (!d.range) return peer_fail(ADASPA_ERR_CUDA, "cuMemGetAddressRange unavailable");
  CUdeviceptr base = 0;
  size_t size = 0;
  if (d.range(&base, &size, reinterpret_cast<CUdeviceptr>(dev_ptr)) != CUDA_SUCCESS)
    return peer_fail(ADASPA_ERR_INVALID_ARG, "dev_ptr is not device memory");
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base));
  if (e != cudaSuccess) return peer_fail(ADASPA_ERR_CUDA, "cudaIpcGetMemHandle: %s", cudaGetErrorString(e));
  static_assert(sizeof(h) <= sizeof(out->handle), "IPC handle outgrew adaspa_peer_handle");
  memset(out, 0, sizeof(*out));
  memcpy(out->handle, &h, sizeof(h));
  out->offset = static_cast<int64_t>(reinterpret_cast<CUdeviceptr>(dev_ptr) - base);
  return ADASPA_OK;
}

adaspa_status adaspa_peer_import(const adaspa_peer_handle* in, void** dev_ptr, void** base_out) {
  if (!in || !dev_ptr || !base_out) return peer_fail(ADASPA_ERR_INVALID_ARG, "arguments must not be NULL");
  cudaIpcMemHandle_t h;
  memcpy(&h, in->handle, sizeof(h));
  void* base = nullptr;
  cudaError_t e = cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) return peer_fail(ADASPA_ERR_CUDA, "cudaIpcOpenMemHandle: %s", cudaGetErrorString(e));
  *base_out = base;
  *dev_ptr = static_cast<char*>(base) + in->offset;
  return ADASPA_OK;
}

adaspa_status adaspa_peer_close(void* base) {
  if (!base) return peer_fail(ADASPA_ERR_INVALID_ARG, "base must not be NULL");
  cudaError_t e = cudaIpcCloseMemHandle(base);
  if (e != cudaSuccess) return peer_fail(ADASPA_ERR_CUDA, "cudaIpcCloseMemHandle: %s", cudaGetErrorString(e));
  return ADASPA_OK;
}

adaspa_status adaspa_peer_copy2d(void* dst, int64_t dst_pitch, const void* src, int64_t src_pitch,
                                 int64_t width_bytes, int64_t rows, adaspa_stream_t stream) {
  if (rows == 0 || width_bytes == 0) return ADASPA_OK;
  if (!dst || !src) return peer_fail(ADASPA_ERR_INVALID_ARG, "dst and src must not be NULL");
  if (rows < 0 || width_bytes < 0 || dst_pitch < width_bytes || src_pitch < width_bytes)
    return peer_fail(ADASPA_ERR_INVALID_ARG, "pitches must be >= width and sizes >= 0");
  cudaError_t e = cudaMemcpy2DAsync(dst, static_cast<size_t>(dst_pitch), src, static_cast<size_t>(src_pitch),
                                    static_cast<size_t>(width_bytes), static_cast<size_t>(rows), cudaMemcpyDefault,
                                    reinterpret_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return peer_fail(ADASPA_ERR_CUDA, "cudaMemcpy2DAsync: %s", cudaGetErrorString(e));
  return ADASPA_OK;
}

adaspa_status adaspa_peer_signal(uint32_t* flag, uint32_t value, adaspa_stream_t stream) {
  if (!flag) return peer_fail(ADASPA_ERR_INVALID_ARG, "flag must not be NULL");
  const Driver& d = drv();
  if (!d.write32) return peer_fail(ADASPA_ERR_CUDA, "cuStreamWriteValue32 unavailable");
  if (d.write32(reinterpret_cast<CUstream>(stream), reinterpret_cast<CUdeviceptr>(flag), value, 0) != CUDA_SUCCESS)
    return peer_fail(ADASPA_ERR_CUDA, "cuStreamWriteValue32 failed");
  return ADASPA_OK;
}

adaspa_status adaspa_peer_wait(const uint32_t* flags, int32_t n, uint32_t value, adaspa_stream_t stream) {
  if (n < 0 || (n > 0 && !flags)) return peer_fail(ADASPA_ERR_INVALID_ARG, "flags must hold n >= 0 words");
  const Driver& d = drv();
  if (!d.wait32) return peer_fail(ADASPA_ERR_CUDA, "cuStreamWaitValue32 unavailable");
  for (int i = 0; i < n; ++i)
    if (d.wait32(reinterpret_cast<CUstream>(stream), reinterpret_cast<CUdeviceptr>(flags + i), value,
                 CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS)
      return peer_fail(ADASPA_ERR_CUDA, "cuStreamWaitValue32 failed");
  return ADASPA_OK;
}
