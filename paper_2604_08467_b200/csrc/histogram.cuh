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

// ---- one-word keys, already sorted together with their u32 counts ----------------------------
// The segment heads, the head scan and the u64 count scan are done tile by tile straight from the
// sorted (key, count) arrays: one reduce pass, a scan of the per-tile totals, one emit pass.
constexpr int HT_THREADS = 256;
constexpr int HT_ITEMS = 8;
constexpr int HT_TILE = HT_THREADS * HT_ITEMS;

template <typename K>
__device__ __forceinline__ void hist_tile_load(const K* __restrict__ keys,
                                               const uint32_t* __restrict__ counts, uint64_t base,
                                               uint64_t n, K (&k)[HT_ITEMS],
                                               uint32_t (&c)[HT_ITEMS], K& prev) {
  if (base + HT_ITEMS <= n) {
    if constexpr (sizeof(K) == 8) {
      const ulonglong2* kp = reinterpret_cast<const ulonglong2*>(keys + base);
#pragma unroll
      for (int i = 0; i < HT_ITEMS / 2; ++i) { const ulonglong2 v = kp[i]; k[2 * i] = v.x; k[2 * i + 1] = v.y; }
    } else {
      const uint4* kp = reinterpret_cast<const uint4*>(keys + base);
#pragma unroll
      for (int i = 0; i < HT_ITEMS / 4; ++i) {
        const uint4 v = kp[i];
        k[4 * i] = v.x; k[4 * i + 1] = v.y; k[4 * i + 2] = v.z; k[4 * i + 3] = v.w;
      }
    }
    if (counts) {
      const uint4* cp = reinterpret_cast<const uint4*>(counts + base);
#pragma unroll
      for (int i = 0; i < HT_ITEMS / 4; ++i) {
        const uint4 v = cp[i];
        c[4 * i] = v.x; c[4 * i + 1] = v.y; c[4 * i + 2] = v.z; c[4 * i + 3] = v.w;
      }
    } else {  // records of one raw draw each
#pragma unroll
      for (int i = 0; i < HT_ITEMS; ++i) c[i] = 1;
    }
  } else {
#pragma unroll
    for (int i = 0; i < HT_ITEMS; ++i) {
      k[i] = base + i < n ? keys[base + i] : K(0);
      c[i] = base + i < n ? (counts ? counts[base + i] : 1u) : 0;
    }
  }
  prev = (base && base < n) ? keys[base - 1] : K(0);
}

// is item i of this thread (global index base + i) the first record of its key?
template <typename K>
__device__ __forceinline__ uint32_t hist_is_head(const K (&k)[HT_ITEMS], K prev,
                                                 uint64_t base, uint64_t n, int i) {
  if (base + i >= n) return 0;
  if (base + i == 0) return 1;
  return k[i] != (i ? k[i - 1] : prev);
}

template <typename K>
__global__ void __launch_bounds__(HT_THREADS)
hist_tile_reduce_kernel(const K* __restrict__ keys, const uint32_t* __restrict__ counts,
                        uint64_t n, uint32_t* __restrict__ tile_heads,
                        uint64_t* __restrict__ tile_sums) {
  __shared__ uint32_t wh[HT_THREADS / 32];
  __shared__ uint64_t wsum[HT_THREADS / 32];
  const uint64_t base = (uint64_t)blockIdx.x * HT_TILE + (uint64_t)threadIdx.x * HT_ITEMS;
  K k[HT_ITEMS], prev;
  uint32_t c[HT_ITEMS];
  hist_tile_load(keys, counts, base, n, k, c, prev);
  uint32_t heads = 0;
  uint64_t sum = 0;
#pragma unroll
  for (int i = 0; i < HT_ITEMS; ++i) { heads += hist_is_head(k, prev, base, n, i); sum += c[i]; }
#pragma unroll
  for (int d = 16; d; d >>= 1) {
    heads += __shfl_xor_sync(0xffffffffu, heads, d);
    sum += __shfl_xor_sync(0xffffffffu, sum, d);
  }
  if ((threadIdx.x & 31) == 0) { wh[threadIdx.x >> 5] = heads; wsum[threadIdx.x >> 5] = sum; }
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t h = 0;
    uint64_t t = 0;
#pragma unroll
    for (int w = 0; w < HT_THREADS / 32; ++w) { h += wh[w]; t += wsum[w]; }
    tile_heads[blockIdx.x] = h;
    tile_sums[blockIdx.x] = t;
  }
}

// 32-bit keys are the top halves of the packed bitstrings (key_bits <= 32)
__device__ __forceinline__ uint64_t hist_widen(uint64_t k) { return k; }
__device__ __forceinline__ uint64_t hist_widen(uint32_t k) { return (uint64_t)k << 32; }

__global__ void narrow_keys_kernel(const uint64_t* __restrict__ in, uint32_t* __restrict__ out, uint64_t n) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = (uint32_t)(in[i] >> 32);
}

template <typename K>
__global__ void __launch_bounds__(HT_THREADS)
hist_tile_emit_kernel(const K* __restrict__ keys, const uint32_t* __restrict__ counts,
                      uint64_t n, const uint32_t* __restrict__ tile_head_off,
                      const uint64_t* __restrict__ tile_sum_off, uint64_t* __restrict__ out_keys,
                      uint64_t* __restrict__ seg_begin) {
  __shared__ uint32_t ws32[33];
  __shared__ uint64_t ws64[33];
  const uint64_t base = (uint64_t)blockIdx.x * HT_TILE + (uint64_t)threadIdx.x * HT_ITEMS;
  K k[HT_ITEMS], prev;
  uint32_t c[HT_ITEMS];
  hist_tile_load(keys, counts, base, n, k, c, prev);
  uint32_t h[HT_ITEMS], heads = 0;
  uint64_t sum = 0;
#pragma unroll
  for (int i = 0; i < HT_ITEMS; ++i) { h[i] = hist_is_head(k, prev, base, n, i); heads += h[i]; sum += c[i]; }
  uint32_t th;
  uint64_t ts;
  uint32_t row = block_exclusive<uint32_t>(heads, ws32, &th) + tile_head_off[blockIdx.x];
  uint64_t run = block_exclusive<uint64_t>(sum, ws64, &ts) + tile_sum_off[blockIdx.x];
#pragma unroll
  for (int i = 0; i < HT_ITEMS; ++i) {
    if (h[i]) { out_keys[row] = hist_widen(k[i]); seg_begin[row] = run; ++row; }
    run += c[i];
  }
}

struct Histogram {
  DevBuf keys;    // [n][words] row-major
  DevBuf counts;  // [n] u64
  uint64_t n = 0;
};

// heads, head scan, u64 count scan and emission for sorted (key, count) pairs of one key word
template <typename K>
inline void sorted_pairs_tail(const K* sk, const uint32_t* sc, uint64_t n, Histogram& out, cudaStream_t st) {
  const unsigned T = 256;
  const unsigned tiles = (unsigned)cdiv(n, (uint64_t)HT_TILE);
  DevBuf th(tiles * 4, st), tho(tiles * 4, st), ts(tiles * 8, st), tso(tiles * 8, st), tot(16, st);
  hist_tile_reduce_kernel<K><<<tiles, HT_THREADS, 0, st>>>(sk, sc, n, th.as<uint32_t>(), ts.as<uint64_t>());
  g_launches++;
  exclusive_scan<uint32_t, uint32_t>(th.as<uint32_t>(), tho.as<uint32_t>(), tiles, tot.as<uint32_t>(), st);
  exclusive_scan<uint64_t, uint64_t>(ts.as<uint64_t>(), tso.as<uint64_t>(), tiles, tot.as<uint64_t>() + 1, st);
  struct { uint32_t heads; uint32_t pad; uint64_t total; } h;
  CK(cudaMemcpyAsync(&h, tot.p, 16, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  out.n = h.heads;
  out.keys.alloc((size_t)out.n * 8, st);
  out.counts.alloc((size_t)out.n * 8, st);
  DevBuf seg(out.n * 8, st);
  hist_tile_emit_kernel<K><<<tiles, HT_THREADS, 0, st>>>(sk, sc, n, tho.as<uint32_t>(), tso.as<uint64_t>(),
                                                         out.keys.as<uint64_t>(), seg.as<uint64_t>());
  segment_counts_kernel<<<cdiv(out.n, T), T, 0, st>>>(seg.as<uint64_t>(), h.total, out.n,
                                                      out.counts.as<uint64_t>());
  g_launches += 2;
  CK(cudaGetLastError());
}

// keys: SoA [words][stride] u64 on device; counts u32 (counts64 == nullptr) or u64.
inline void reduce_by_key(const uint64_t* keys, uint64_t stride, uint32_t words,
                          const uint32_t* counts32, const uint64_t* counts64, uint64_t n,
                          uint32_t key_bits, Histogram& out, cudaStream_t st, bool unit_counts = false) {
  out.n = 0;
  if (n == 0) { out.keys.alloc(0, st); out.counts.alloc(0, st); return; }
  if (n >= (1ull << 32)) throw Failure(PTSBE_ECAPACITY, "more than 2^32 records in one reduce");
  const unsigned T = 256, G = cdiv(n, T);
  DevBuf kout;
  DevBuf sorted_counts;
  if (words == 1 && counts32 && key_bits >= 1) {
    // one key word: sort the (key, count) pairs themselves, then reduce tile by tile from the
    // sorted arrays.  Keys of at most 32 bits are sorted as u32 (8 instead of 12 bytes per pair
    // and radix pass).
    const int used = (int)std::min<uint32_t>(key_bits, 64);
    size_t tmp_bytes = 0;
    if (unit_counts) {
      // every count is 1 (raw draws of a final descent stage): the sort moves keys alone and the tail
      // counts run lengths
      if (used <= 32) {
        DevBuf k32(n * 4, st), k32s(n * 4, st);
        narrow_keys_kernel<<<G, T, 0, st>>>(keys, k32.as<uint32_t>(), n);
        CK(cub::DeviceRadixSort::SortKeys(nullptr, tmp_bytes, k32.as<uint32_t>(), k32s.as<uint32_t>(), (int)n,
                                          32 - used, 32, st));
        DevBuf tmp(tmp_bytes, st);
        CK(cub::DeviceRadixSort::SortKeys(tmp.p, tmp_bytes, k32.as<uint32_t>(), k32s.as<uint32_t>(), (int)n,
                                          32 - used, 32, st));
        g_launches += 2 + (used + 7) / 8 * 2;
        sorted_pairs_tail<uint32_t>(k32s.as<uint32_t>(), nullptr, n, out, st);
      } else {
        kout.alloc(n * 8, st);
        CK(cub::DeviceRadixSort::SortKeys(nullptr, tmp_bytes, keys, kout.as<uint64_t>(), (int)n, 64 - used, 64, st));
        DevBuf tmp(tmp_bytes, st);
        CK(cub::DeviceRadixSort::SortKeys(tmp.p, tmp_bytes, keys, kout.as<uint64_t>(), (int)n, 64 - used, 64, st));
        g_launches += 1 + (used + 7) / 8 * 2;
        sorted_pairs_tail<uint64_t>(kout.as<uint64_t>(), nullptr, n, out, st);
      }
      return;
    }
    sorted_counts.alloc(n * 4, st);
    if (used <= 32) {
      DevBuf k32(n * 4, st), k32s(n * 4, st);
      narrow_keys_kernel<<<G, T, 0, st>>>(keys, k32.as<uint32_t>(), n);
      CK(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, k32.as<uint32_t>(), k32s.as<uint32_t>(), counts32,
                                         sorted_counts.as<uint32_t>(), (int)n, 32 - used, 32, st));
      DevBuf tmp(tmp_bytes, st);
      CK(cub::DeviceRadixSort::SortPairs(tmp.p, tmp_bytes, k32.as<uint32_t>(), k32s.as<uint32_t>(), counts32,
                                         sorted_counts.as<uint32_t>(), (int)n, 32 - used, 32, st));
      g_launches += 2 + (used + 7) / 8 * 2;
      sorted_pairs_tail<uint32_t>(k32s.as<uint32_t>(), sorted_counts.as<uint32_t>(), n, out, st);
    } else {
      kout.alloc(n * 8, st);
      CK(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, keys, kout.as<uint64_t>(), counts32,
                                         sorted_counts.as<uint32_t>(), (int)n, 64 - used, 64, st));
      DevBuf tmp(tmp_bytes, st);
      CK(cub::DeviceRadixSort::SortPairs(tmp.p, tmp_bytes, keys, kout.as<uint64_t>(), counts32,
                                         sorted_counts.as<uint32_t>(), (int)n, 64 - used, 64, st));
      g_launches += 1 + (used + 7) / 8 * 2;
      sorted_pairs_tail<uint64_t>(kout.as<uint64_t>(), sorted_counts.as<uint32_t>(), n, out, st);
    }
    return;
  }
  DevBuf perm_a(n * 4, st), perm_b(n * 4, st), kin(n * 8, st);
  kout.alloc(n * 8, st);
  iota_kernel<<<G, T, 0, st>>>(perm_a.as<uint32_t>(), (uint32_t)n, 0);
  g_launches++;
  uint32_t* pin = perm_a.as<uint32_t>();
  uint32_t* pout = perm_b.as<uint32_t>();
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
