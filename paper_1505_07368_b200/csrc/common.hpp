// Shared host-side helpers of libcafxg.so: status codes, thread-local error
// context, CUDA error mapping.
#pragma once
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdio>
#include <string>

#include "../../include/cafxg.h"

namespace cafxg {

void set_last_error(const char* fmt, ...);
void clear_last_error();

// Maps a CUDA failure to CAFXG_E_DOWN (the device or the actor behind it is
// unusable, cafx::errc::request_down) and records the context string.
inline int cuda_status(cudaError_t e, const char* what) {
  if (e == cudaSuccess)
    return CAFXG_OK;
  set_last_error("%s: %s (%s)", what, cudaGetErrorName(e), cudaGetErrorString(e));
  return CAFXG_E_DOWN;
}

#define CAFXG_CUDA_TRY(expr)                                  \
  do {                                                        \
    cudaError_t _e = (expr);                                  \
    if (_e != cudaSuccess)                                    \
      return ::cafxg::cuda_status(_e, #expr);                 \
  } while (0)

#define CAFXG_TRY(expr)                                       \
  do {                                                        \
    int _s = (expr);                                          \
    if (_s != CAFXG_OK)                                       \
      return _s;                                              \
  } while (0)

inline int fail(int status, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  set_last_error("%s", buf);
  return status;
}

// Scatter of a device staging buffer into reply buffers (copy.cu). One block
// per segment; 16-byte vector copies when src/dst/len allow.
struct CopySeg {
  const void* src;  // device
  void* dst;        // device-visible: device memory or mapped pinned host
  uint64_t bytes;
};
int copy_segments_launch(const CopySeg* segs_dev, uint32_t n, void* stream);
// Small batches pass their segment table by value in the kernel parameters
// (no allocation, upload or free per batch).
constexpr uint32_t kInlineSegs = 32;  // 768 B of parameters (launch cost grows with them)
int copy_segments_inline_launch(const CopySeg* segs_host, uint32_t n, void* stream);

}  // namespace cafxg
