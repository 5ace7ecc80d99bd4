// Histogram aggregation: sum counts per measured bitstring, output sorted by
// key (replaces merge_records, engine.py:815-829, for the count field; the
// `prob` tag only exists in non-proportional mode, which is out of scope).
//
// Keys are packed bitstrings of `words` u64 (qubit 0 = most significant bit of
// word 0), so numeric order of (word0, word1, ..) is the reference's sorted()
// order of bitstrings.  Sorting is an LSD pass per word with CUB's radix sort
// (library plumbing); segment heads, the u64 scan and the reduce are ours.
#pragma once
#include <cub/device/device_radix_sort.cuh>

#include "common.cuh"
#include "sampler.cuh"
#include "scan.cuh"

namespace ptsbe {

__global__ void gather_u64_kernel(const uint64_t* src, const uint32_t* perm, uint64_t* dst,
                                  uint64_t n) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[i] = src[perm[i]];
}

// head[i] = 1 when record i (in sorted order perm) starts a new key
__global__ void head_flags_kernel(const uint64_t* keys, uint64_t stride, uint32_t words,
                                  const uint32_t* perm, uint32_t* head, uint64_t n) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint32_t h = (i == 0);
  if (i) {
    const uint32_t a = perm[i], b = perm[i - 1];
    for (uint32_t w = 0; w < words; ++w) h |= keys[w * stride + a] != keys[w * stride + b];
  }
  head[i] = h;
}

__global__ void gather_counts_kernel(const uint32_t* counts, const uint32_t* perm, uint64_t* out,
                                     uint64_t n) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = counts[perm[i]];
}
__global__ void gather_counts64_kernel(const uint64_t* counts, const uint32_t* perm,
                                       uint64_t* out, uint64_t n) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = counts[perm[i]];
}

// seg[i] = exclusive scan of head (so seg of a head i is its output row + ... see below)
__global__ void emit_segments_kernel(const uint64_t* keys, uint64_t stride, uint32_t words,
                                     const uint32_t* perm, const uint32_t* head,
                                     const uint32_t* head_scan, const uint64_t* count_scan,
                                     uint64_t total_count, uint64_t n, uint64_t n_out,
                                     uint64_t* out_keys /*[n_out][words]*/,
                                     uint64_t* out_counts, uint64_t* seg_begin_scan) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (!head[i]) return;
  const uint32_t row = head_scan[i];  // heads before i
  for (uint32_t w = 0; w < words; ++w) out_keys[(uint64_t)row * words + w] = keys[w * stride + perm[i]];
  seg_begin_scan[row] = count_scan[i];
  (void)total_count; (void)n_out; (void)out_counts;
}
__global__ void segment_counts_kernel(const uint64_t* seg_begin_scan, uint64_t total_count,
                                      uint64_t n_out, uint64_t* out_counts) {
  const uint64_t r = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n_out) return;
  const uint64_t end = (r + 1 < n_out) ? seg_begin_scan[r + 1] : total_count;
  out_counts[r] = end - seg_begin_scan[r];
}

// row-major [n][words] -> SoA [words][n]
__global__ void transpose_keys_kernel(const uint64_t* in, uint64_t* out, uint64_t n, uint32_t words) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n * words) return;
  const uint64_t r = i / words, w = i - r * words;
  out[w * n + r] = in[i];
}

// SoA [words][n] -> row-major [n][words]
__global__ void untranspose_keys_kernel(const uint64_t* in, uint64_t* out, uint64_t n, uint32_t words) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n * words) return;
  const uint64_t r = i / words, w = i - r * words;
  out[i] = in[w * n + r];
}
__global__ void widen_counts_kernel(const uint32_t* in, uint64_t* out, uint64_t n) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = in[i];
}

struct Histogram {
  DevBuf keys;    // [n][words] row-major
  DevBuf counts;  // [n] u64
  uint64_t n = 0;
};

// keys: SoA [words][stride] u64 on device; counts u32 (counts64 == nullptr) or u64.
inline void reduce_by_key(const uint64_t* keys, uint64_t stride, uint32_t words,
                          const uint32_t* counts32, const uint64_t* counts64, uint64_t n,
                          uint32_t key_bits, Histogram& out, cudaStream_t st) {
  out.n = 0;
  if (n == 0) { out.keys.alloc(0, st); out.counts.alloc(0, st); return; }
  if (n >= (1ull << 32)) throw Failure(PTSBE_ECAPACITY, "more than 2^32 records in one reduce");
  const unsigned T = 256, G = cdiv(n, T);
  DevBuf perm_a(n * 4, st), perm_b(n * 4, st), kin(n * 8, st), kout(n * 8, st);
  iota_kernel<<<G, T, 0, st>>>(perm_a.as<uint32_t>(), (uint32_t)n, 0);
  g_launches++;
  uint32_t* pin = perm_a.as<uint32_t>();
  uint32_t* pout = perm_b.as<uint32_t>();
  DevBuf sorted_counts;
  if (words == 1 && counts32 && key_bits >= 1) {
    // one key word: sort the (key, count) pairs themselves; everything downstream then reads
    // sorted arrays through the identity permutation (coalesced) instead of gathering through one
    const int used = (int)std::min<uint32_t>(key_bits, 64);
    sorted_counts.alloc(n * 4, st);
    size_t tmp_bytes = 0;
    CK(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, keys, kout.as<uint64_t>(), counts32,
                                       sorted_counts.as<uint32_t>(), (int)n, 64 - used, 64, st));
    DevBuf tmp(tmp_bytes, st);
    CK(cub::DeviceRadixSort::SortPairs(tmp.p, tmp_bytes, keys, kout.as<uint64_t>(), counts32,
                                       sorted_counts.as<uint32_t>(), (int)n, 64 - used, 64, st));
    g_launches += 1 + (used + 7) / 8 * 2;
    keys = kout.as<uint64_t>();
    stride = n;
    counts32 = sorted_counts.as<uint32_t>();
  } else
  for (int w = (int)words - 1; w >= 0; --w) {
    // bits used in word w: qubits [64w, min(64w+64, key_bits)) occupy the top of the word
    const int used = (int)key_bits - 64 * w >= 64 ? 64 : (int)key_bits - 64 * w;
    if (used <= 0) continue;
    gather_u64_kernel<<<G, T, 0, st>>>(keys + (uint64_t)w * stride, pin, kin.as<uint64_t>(), n);
    g_launches++;
    size_t tmp_bytes = 0;
    CK(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, kin.as<uint64_t>(), kout.as<uint64_t>(),
                                       pin, pout, (int)n, 64 - used, 64, st));
    DevBuf tmp(tmp_bytes, st);
    CK(cub::DeviceRadixSort::SortPairs(tmp.p, tmp_bytes, kin.as<uint64_t>(), kout.as<uint64_t>(),
                                       pin, pout, (int)n, 64 - used, 64, st));
    g_launches += 1 + (used + 7) / 8 * 2;  // histogram + onesweep passes (library kernels)
    std::swap(pin, pout);
  }
  DevBuf head(n * 4, st), head_scan(n * 4, st), c64(n * 8, st), cscan(n * 8, st), tot(16, st);
  head_flags_kernel<<<G, T, 0, st>>>(keys, stride, words, pin, head.as<uint32_t>(), n);
  if (counts64) gather_counts64_kernel<<<G, T, 0, st>>>(counts64, pin, c64.as<uint64_t>(), n);
  else gather_counts_kernel<<<G, T, 0, st>>>(counts32, pin, c64.as<uint64_t>(), n);
  g_launches += 2;
  exclusive_scan<uint32_t, uint32_t>(head.as<uint32_t>(), head_scan.as<uint32_t>(), n,
                                     tot.as<uint32_t>(), st);
  exclusive_scan<uint64_t, uint64_t>(c64.as<uint64_t>(), cscan.as<uint64_t>(), n,
                                     tot.as<uint64_t>() + 1, st);
  struct { uint32_t heads; uint32_t pad; uint64_t total; } h;
  CK(cudaMemcpyAsync(&h, tot.p, 16, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  out.n = h.heads;
  out.keys.alloc((size_t)out.n * words * 8, st);
  out.counts.alloc((size_t)out.n * 8, st);
  DevBuf seg(out.n * 8, st);
  emit_segments_kernel<<<G, T, 0, st>>>(keys, stride, words, pin, head.as<uint32_t>(),
                                        head_scan.as<uint32_t>(), cscan.as<uint64_t>(), h.total,
                                        n, out.n, out.keys.as<uint64_t>(),
                                        out.counts.as<uint64_t>(), seg.as<uint64_t>());
  segment_counts_kernel<<<cdiv(out.n, T), T, 0, st>>>(seg.as<uint64_t>(), h.total, out.n,
                                                      out.counts.as<uint64_t>());
  g_launches += 2;
  CK(cudaGetLastError());
}

}  // namespace ptsbe
