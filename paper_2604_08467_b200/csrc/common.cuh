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

// Run-scoped device workspace: a bump allocator over a few big cudaMalloc'ed slabs that are
// kept between runs.  Every temporary of a sampling run (work lists, hoisted records,
// population vectors, sort buffers) comes from here, so the timed loop performs no device
// allocation at all once the slabs exist -- growing the stream-ordered pool by hundreds of
// MB inside the loop stalls the GPU for as long as the kernels themselves take.
struct Workspace {
  struct Slab { char* p; size_t size; };
  std::vector<Slab> slabs;
  size_t cur = 0, off = 0;
  static constexpr size_t kSlab = 1ull << 30;
  void* alloc(size_t bytes) {
    bytes = (bytes + 255) & ~size_t(255);
    if (bytes == 0) bytes = 256;
    for (; cur < slabs.size(); ++cur, off = 0)
      if (off + bytes <= slabs[cur].size) {
        void* r = slabs[cur].p + off;
        off += bytes;
        return r;
      }
    size_t want = bytes <= kSlab ? kSlab : ((bytes + bytes / 4 + (kSlab >> 2) - 1) / (kSlab >> 2)) * (kSlab >> 2);
    Slab sl;
    sl.size = want;
    if (cudaMalloc(reinterpret_cast<void**>(&sl.p), want) != cudaSuccess) {
      cudaGetLastError();
      sl.size = want = bytes;  // exact fit as a last resort
      cuda_check(cudaMalloc(reinterpret_cast<void**>(&sl.p), want), "cudaMalloc(workspace slab)", __FILE__, __LINE__);
    }
    slabs.push_back(sl);
    cur = slabs.size() - 1;
    off = bytes;
    return sl.p;
  }
  struct Mark { size_t cur, off; };
  Mark mark() const { return Mark{cur, off}; }
  void rewind(Mark m) { cur = m.cur; off = m.off; }
  void reset() { cur = 0; off = 0; }
  size_t reserved() const { size_t t = 0; for (auto& s : slabs) t += s.size; return t; }
  void destroy() { for (auto& s : slabs) cudaFree(s.p); slabs.clear(); reset(); }
  ~Workspace() { destroy(); }
};

// workspace that DevBuf allocations of the calling thread are served from (null: stream-ordered pool)
extern thread_local Workspace* g_ws;

// Device buffer.  Inside a sampling run (g_ws set) it is a view into the run's workspace and
// releasing it is free; elsewhere it is a stream-ordered allocation from the device's default
// memory pool (release threshold raised at plan creation).
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  cudaStream_t s = nullptr;
  bool owned = true;
  DevBuf() {}
  DevBuf(size_t n, cudaStream_t st) { alloc(n, st); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), bytes(o.bytes), s(o.s), owned(o.owned) { o.p = nullptr; o.bytes = 0; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      release();
      p = o.p; bytes = o.bytes; s = o.s; owned = o.owned;
      o.p = nullptr; o.bytes = 0;
    }
    return *this;
  }
  void alloc(size_t n, cudaStream_t st) {
    release();
    s = st;
    bytes = n;
    if (n == 0) return;
    if (g_ws) { p = g_ws->alloc(n); owned = false; return; }
    owned = true;
    CK(cudaMallocAsync(&p, n, st));
  }
  void alloc(size_t n, Workspace& ws) {
    release();
    bytes = n;
    owned = false;
    if (n) p = ws.alloc(n);
  }
  void release() {
    if (p && owned) cudaFreeAsync(p, s);
    p = nullptr;
    bytes = 0;
  }
  ~DevBuf() { release(); }
  template <typename T> T* as() const { return reinterpret_cast<T*>(p); }
};

struct WorkspaceScope {  // installs a workspace for DevBuf allocations of this thread
  Workspace* prev;
  explicit WorkspaceScope(Workspace* ws) : prev(g_ws) { g_ws = ws; }
  ~WorkspaceScope() { g_ws = prev; }
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
