// Shared plumbing for libptsbe_b200.so: error state, RAII device buffers,
// launch accounting.  sm_100a only; no other architecture is targeted.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/ptsbe_b200.h"

namespace ptsbe {

struct Failure : std::runtime_error {
  int code;
  Failure(int c, const std::string& what) : std::runtime_error(what), code(c) {}
};

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
  if (e != cudaSuccess) {
    char buf[512];
    snprintf(buf, sizeof buf, "CUDA failure %s at %s:%d: %s", what, file, line,
             cudaGetErrorString(e));
    throw Failure(PTSBE_EDEVICE, buf);
  }
}
#define CK(x) ::ptsbe::cuda_check((x), #x, __FILE__, __LINE__)

extern thread_local std::string g_last_error;
extern thread_local uint64_t g_launches;  // kernels launched on this thread since reset

// Stream-ordered device buffer.  Allocation goes through the device's default
// memory pool (release threshold raised at plan creation), so repeated runs
// reuse the same HBM without cudaMalloc latency.
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  cudaStream_t s = nullptr;
  DevBuf() {}
  DevBuf(size_t n, cudaStream_t st) { alloc(n, st); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), bytes(o.bytes), s(o.s) { o.p = nullptr; o.bytes = 0; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      release();
      p = o.p; bytes = o.bytes; s = o.s;
      o.p = nullptr; o.bytes = 0;
    }
    return *this;
  }
  void alloc(size_t n, cudaStream_t st) {
    release();
    s = st;
    bytes = n;
    if (n == 0) return;
    CK(cudaMallocAsync(&p, n, st));
  }
  void release() {
    if (p) cudaFreeAsync(p, s);
    p = nullptr;
    bytes = 0;
  }
  ~DevBuf() { release(); }
  template <typename T> T* as() const { return reinterpret_cast<T*>(p); }
};

// Deferred CUDA-event timing of spans on one stream: spans are recorded while the
// work is enqueued and read back after the next synchronisation point.
struct EventLog {
  struct Span { cudaEvent_t a, b; float* acc; };
  std::vector<Span> spans;
  cudaStream_t st = nullptr;
  explicit EventLog(cudaStream_t s) : st(s) {}
  void begin(float* acc) {
    Span sp;
    sp.acc = acc;
    CK(cudaEventCreate(&sp.a));
    CK(cudaEventCreate(&sp.b));
    CK(cudaEventRecord(sp.a, st));
    spans.push_back(sp);
  }
  void end() { CK(cudaEventRecord(spans.back().b, st)); }
  // call after the stream has been synchronised
  void flush() {
    for (auto& sp : spans) {
      float ms = 0;
      if (cudaEventElapsedTime(&ms, sp.a, sp.b) == cudaSuccess && sp.acc) *sp.acc += ms;
      cudaEventDestroy(sp.a);
      cudaEventDestroy(sp.b);
    }
    spans.clear();
  }
  ~EventLog() { for (auto& sp : spans) { cudaEventDestroy(sp.a); cudaEventDestroy(sp.b); } }
};

inline unsigned cdiv(uint64_t a, uint64_t b) { return (unsigned)((a + b - 1) / b); }

}  // namespace ptsbe
