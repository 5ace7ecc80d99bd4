// Order-preserving device scans used by the sampler's compaction and the
// histogram reduce-by-key.  Hand-written reduce-then-scan: warp shuffles inside
// a 256-thread block (8 consecutive elements per thread -> 128-bit coalesced
// loads for u32), recursion on the per-block totals.  Determinism matters more
// than the last few percent here: slot order defines the RNG stream of every
// child prefix, so no atomics are used anywhere in the compaction.
#pragma once
#include "common.cuh"

namespace ptsbe {

constexpr int SCAN_THREADS = 256;
constexpr int SCAN_ITEMS = 8;
constexpr int SCAN_TILE = SCAN_THREADS * SCAN_ITEMS;

template <typename T>
__device__ __forceinline__ T warp_inclusive(T v, int lane) {
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    T o = __shfl_up_sync(0xffffffffu, v, d);
    if (lane >= d) v += o;
  }
  return v;
}

// exclusive prefix of `v` over the block; *total = block sum. Needs warp_sums[32].
template <typename T>
__device__ __forceinline__ T block_exclusive(T v, T* warp_sums, T* total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  T inc = warp_inclusive(v, lane);
  if (lane == 31) warp_sums[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    T s = lane < nw ? warp_sums[lane] : T(0);
    T si = warp_inclusive(s, lane);
    warp_sums[lane] = si - s;  // exclusive warp offsets
    if (lane == 31) warp_sums[32] = si;
  }
  __syncthreads();
  T r = warp_sums[wid] + inc - v;
  *total = warp_sums[32];
  __syncthreads();
  return r;
}

// per-tile sums only (first pass of a multi-tile scan: nothing but the totals is written)
template <typename TI, typename TO>
__global__ void __launch_bounds__(SCAN_THREADS)
scan_reduce_kernel(const TI* __restrict__ in, TO* __restrict__ tile_sums, uint64_t n) {
  __shared__ TO ws[SCAN_THREADS / 32];
  const uint64_t base = (uint64_t)blockIdx.x * SCAN_TILE + (uint64_t)threadIdx.x * SCAN_ITEMS;
  TO local = 0;
#pragma unroll
  for (int i = 0; i < SCAN_ITEMS; ++i) local += (base + i < n) ? (TO)in[base + i] : TO(0);
#pragma unroll
  for (int d = 16; d; d >>= 1) local += __shfl_xor_sync(0xffffffffu, local, d);
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = local;
  __syncthreads();
  if (threadIdx.x == 0) {
    TO t = 0;
#pragma unroll
    for (int w = 0; w < SCAN_THREADS / 32; ++w) t += ws[w];
    tile_sums[blockIdx.x] = t;
  }
}

// scan of one tile, shifted by the tile's offset when given; writes the tile total when asked
template <typename TI, typename TO>
__global__ void __launch_bounds__(SCAN_THREADS)
scan_tile_kernel(const TI* in, TO* out, TO* __restrict__ tile_sums,
                 const TO* __restrict__ tile_offsets, uint64_t n) {
  __shared__ TO ws[33];
  const uint64_t base = (uint64_t)blockIdx.x * SCAN_TILE + (uint64_t)threadIdx.x * SCAN_ITEMS;
  TO v[SCAN_ITEMS];
  TO local = 0;
#pragma unroll
  for (int i = 0; i < SCAN_ITEMS; ++i) {
    v[i] = (base + i < n) ? (TO)in[base + i] : TO(0);
    local += v[i];
  }
  TO total;
  TO run = block_exclusive<TO>(local, ws, &total);
  if (tile_offsets) run += tile_offsets[blockIdx.x];
#pragma unroll
  for (int i = 0; i < SCAN_ITEMS; ++i) {
    if (base + i < n) out[base + i] = run;
    run += v[i];
  }
  if (threadIdx.x == 0 && tile_sums) tile_sums[blockIdx.x] = total;
}

template <typename TO>
__global__ void scan_total_kernel(const TO* __restrict__ tile_offsets,
                                  const TO* __restrict__ tile_sums, uint64_t n_tiles,
                                  TO* __restrict__ total) {
  if (threadIdx.x == 0 && blockIdx.x == 0)
    *total = n_tiles ? tile_offsets[n_tiles - 1] + tile_sums[n_tiles - 1] : TO(0);
}

// out[i] = sum_{k<i} in[k]; *total_dev (optional) = sum of all.  In-place allowed
// only when TI == TO.
template <typename TI, typename TO>
void exclusive_scan(const TI* in, TO* out, uint64_t n, TO* total_dev, cudaStream_t st) {
  if (n == 0) {
    if (total_dev) CK(cudaMemsetAsync(total_dev, 0, sizeof(TO), st));
    return;
  }
  const uint64_t tiles = (n + SCAN_TILE - 1) / SCAN_TILE;
  DevBuf sums(tiles * sizeof(TO), st);
  if (tiles > 1) {
    // reduce, scan the tile totals, scan every tile from its offset: 12 bytes per u32 element
    DevBuf offs(tiles * sizeof(TO), st);
    scan_reduce_kernel<TI, TO><<<(unsigned)tiles, SCAN_THREADS, 0, st>>>(in, sums.as<TO>(), n);
    exclusive_scan<TO, TO>(sums.as<TO>(), offs.as<TO>(), tiles, total_dev, st);
    scan_tile_kernel<TI, TO><<<(unsigned)tiles, SCAN_THREADS, 0, st>>>(in, out, nullptr, offs.as<TO>(), n);
    g_launches += 2;
  } else {
    scan_tile_kernel<TI, TO><<<1, SCAN_THREADS, 0, st>>>(in, out, sums.as<TO>(), nullptr, n);
    g_launches++;
    if (total_dev) CK(cudaMemcpyAsync(total_dev, sums.p, sizeof(TO), cudaMemcpyDeviceToDevice, st));
  }
  CK(cudaGetLastError());
}

__global__ void fill_u32_kernel(uint32_t* out, uint32_t n, uint32_t value) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = value;
}

// out[i] = in[i] + offset (error-set rows of a later chunk -> rows of the whole batch)
__global__ void add_offset_u32_kernel(const uint32_t* in, uint32_t* out, uint64_t n, uint32_t offset) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = in[i] + offset;
}

// probability tag of child c: slot (slot_off[parent] + position of c among its parent's children)
__global__ void gather_prob_kernel(const uint32_t* c_parent, const uint32_t* child_base,
                                   const uint32_t* p_slot_off, const double* slot_prob, double* out,
                                   uint32_t n) {
  const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n) return;
  const uint32_t p = c_parent[c];
  out[c] = slot_prob[p_slot_off[p] + (c - child_base[p])];
}

}  // namespace ptsbe
