// Batched stored-path contraction executor (north-star subsystem 2).
//
// One launch runs ONE compiled pass program (see include/ptsbe_b200.h) for a
// batch of work items (error set x measured prefix).  A work item is handled
// by one warp (small programs) or one CTA; every intermediate tensor of the
// path lives in that group's shared-memory arena, so the only HBM traffic of a
// work item is its Kraus-index row, its prefix words, the (L1/L2-resident)
// program tables and operand pool, and the final record.  Buffers that the
// compiler could not fit on chip are placed in a per-group global spill arena.
//
// Replaces, per work item: merge_errors (engine.py:284-313, as a table
// gather), marginal_network (engine.py:361-407, static operand table),
// execute_path/contract_pair (tensor.py:190-268) and the epilogue of
// _contract_marginal (engine.py:442-450).
#pragma once
#include "common.cuh"

namespace ptsbe {

constexpr int STEP_WORDS = 12;
constexpr int LEAF_WORDS = 4;

// Per-level view of the work-item lists (device memory, one entry per level,
// index 1..f+1).  Level L holds the unique prefixes entering stage L.
struct LevelDev {
  const uint32_t* eset;    // [n] error-set row inside the resident batch
  const uint32_t* parent;  // [n] index into level L-1 (unused for L == 1)
  const uint64_t* prefix;  // [words][n] packed measured bits
  const void* ext;         // records of hoist pass (L-1) of the CURRENT stage: [n][ext_rec]
  uint32_t n;
  uint32_t ext_rec;
};

enum ExecMode { EXEC_HOIST = 0, EXEC_MARGINAL = 1, EXEC_RAW = 2, EXEC_VECTOR = 3 };

struct ExecArgs {
  const uint32_t* leaves;
  const uint32_t* steps;
  const uint32_t* tables;
  const void* pool;
  const uint8_t* kraus;  // [sets][g]
  const LevelDev* levels;
  void* spill;   // [resident groups][arena_spill]
  void* out;     // HOIST: records [level n][out_elems] ; MARGINAL: real probs [items][out_elems]
                 // RAW: complex [items][out_elems] ; VECTOR: complex [items of this launch][out_elems]
  double* out_mass;  // MARGINAL: [items]
  double* out_min;   // MARGINAL: [items]
  uint32_t n_steps;
  uint32_t arena_fast;
  uint32_t arena_spill;
  uint32_t out_elems;
  uint32_t result_kind, result_ref;
  uint32_t level;       // L
  uint32_t first_item;  // items [first_item, first_item + n_items) of level L
  uint32_t n_items;
  uint32_t g;
  uint32_t words;
  uint32_t item_bytes;  // shared-memory footprint of one group
  uint32_t mode;
};

template <typename R> struct CxT;
template <> struct CxT<float> { using type = float2; };
template <> struct CxT<double> { using type = double2; };

template <typename C>
__device__ __forceinline__ void cmac(C& acc, const C a, const C b) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(a.y, b.x, acc.y);
}

// WARP = true : blockDim.x = 32 * groups, one warp per item, __syncwarp between steps
// WARP = false: one CTA per item, __syncthreads between steps
template <typename R, bool WARP>
__global__ void exec_kernel(const ExecArgs a) {
  using C = typename CxT<R>::type;
  extern __shared__ __align__(16) unsigned char smem_raw[];

  const int gsize = WARP ? 32 : blockDim.x;
  const int tid = WARP ? (threadIdx.x & 31) : threadIdx.x;
  const int group_in_block = WARP ? (threadIdx.x >> 5) : 0;
  const int groups_per_block = WARP ? (blockDim.x >> 5) : 1;
  const uint32_t group_global = blockIdx.x * groups_per_block + group_in_block;
  const uint32_t n_groups = gridDim.x * groups_per_block;

  unsigned char* my = smem_raw + (size_t)group_in_block * a.item_bytes;
  C* arena = reinterpret_cast<C*>(my);
  uint64_t* pfx = reinterpret_cast<uint64_t*>(my + (size_t)a.arena_fast * sizeof(C));
  uint32_t* anc = reinterpret_cast<uint32_t*>(pfx + a.words);
  uint8_t* sel = reinterpret_cast<uint8_t*>(anc + (a.level + 1));
  C* spill = reinterpret_cast<C*>(a.spill) + (size_t)group_global * a.arena_spill;
  const C* pool = reinterpret_cast<const C*>(a.pool);
  // scratch for CTA-wide reductions (marginal epilogue), placed after the groups
  double* red = reinterpret_cast<double*>(smem_raw + (size_t)groups_per_block * a.item_bytes);

  auto group_sync = [&]() {
    if (WARP) __syncwarp(); else __syncthreads();
  };

  for (uint32_t it = group_global; it < a.n_items; it += n_groups) {
    const uint32_t item = a.first_item + it;
    // ---- item context: ancestors, prefix words, Kraus-index row ----
    if (tid == 0) {
      uint32_t cur = item;
      anc[a.level] = cur;
      for (int l = (int)a.level; l > 1; --l) {
        cur = a.levels[l].parent[cur];
        anc[l - 1] = cur;
      }
    }
    const LevelDev lv = a.levels[a.level];
    const uint32_t e = lv.eset[item];
    for (uint32_t w = tid; w < a.words; w += gsize) pfx[w] = lv.prefix[(size_t)w * lv.n + item];
    {
      const uint8_t* row = a.kraus + (size_t)e * a.g;
      for (uint32_t s = tid; s < a.g; s += gsize) sel[s] = row[s];
    }
    group_sync();

    auto resolve = [&](uint32_t kind, uint32_t ref) -> const C* {
      if (kind == 0) return ref < a.arena_fast ? arena + ref : spill + (ref - a.arena_fast);
      if (kind == 1) {
        const uint32_t* lf = a.leaves + (size_t)ref * LEAF_WORDS;
        uint32_t v = 0;
        if (lf[2] == 1) v = sel[lf[3]];
        else if (lf[2] == 2) v = (uint32_t)((pfx[lf[3] >> 6] >> (63 - (lf[3] & 63))) & 1ull);
        return pool + lf[0] + (size_t)v * lf[1];
      }
      const uint32_t l = kind - 1;  // pass p = kind-2 iterates level p+1
      const LevelDev el = a.levels[l];
      return reinterpret_cast<const C*>(el.ext) + (size_t)anc[l] * el.ext_rec + ref;
    };

    // ---- replay the stored path ----
    for (uint32_t s = 0; s < a.n_steps; ++s) {
      const uint32_t* st = a.steps + (size_t)s * STEP_WORDS;
      const C* A = resolve(st[0], st[1]);
      const C* B = resolve(st[2], st[3]);
      C* O;
      if (st[4] == 0) O = st[5] < a.arena_fast ? arena + st[5] : spill + (st[5] - a.arena_fast);
      else O = reinterpret_cast<C*>(a.out) + (size_t)(a.mode == EXEC_VECTOR ? it : item) * a.out_elems + st[5];
      const uint32_t out_n = st[6], kn = st[7], lo_n = st[8], hi_n = st[9];
      const uint32_t* loA = a.tables + st[10];
      const uint32_t* loB = loA + lo_n;
      const uint32_t* hiA = loB + lo_n;
      const uint32_t* hiB = hiA + hi_n;
      const uint32_t* kA = hiB + hi_n;
      const uint32_t* kB = kA + kn;
      const bool pow2 = (lo_n & (lo_n - 1)) == 0;
      const int sh = 31 - __clz(lo_n);
      for (uint32_t c = tid; c < out_n; c += gsize) {
        uint32_t cl, ch;
        if (pow2) { cl = c & (lo_n - 1); ch = c >> sh; }
        else { ch = c / lo_n; cl = c - ch * lo_n; }
        uint32_t a0 = __ldg(loA + cl), b0 = __ldg(loB + cl);
        if (hi_n > 1) { a0 += __ldg(hiA + ch); b0 += __ldg(hiB + ch); }
        C acc; acc.x = 0; acc.y = 0;
        if (kn == 1) {
          cmac(acc, A[a0], B[b0]);
        } else {
          for (uint32_t k = 0; k < kn; ++k) cmac(acc, A[a0 + __ldg(kA + k)], B[b0 + __ldg(kB + k)]);
        }
        O[c] = acc;
      }
      group_sync();
    }

    // ---- epilogue ----
    if (a.mode == EXEC_MARGINAL || a.mode == EXEC_RAW) {
      const C* res = resolve(a.result_kind, a.result_ref);
      if (a.mode == EXEC_RAW) {
        C* o = reinterpret_cast<C*>(a.out) + (size_t)it * a.out_elems;
        for (uint32_t c = tid; c < a.out_elems; c += gsize) o[c] = res[c];
      } else {
        // real part, minimum before clamping, clamp, mass (engine.py:445-450)
        R* o = reinterpret_cast<R*>(a.out) + (size_t)it * a.out_elems;
        double mn = 1e300, sum = 0.0;
        for (uint32_t c = tid; c < a.out_elems; c += gsize) {
          R v = res[c].x;
          mn = fmin(mn, (double)v);
          v = v > R(0) ? v : R(0);
          sum += (double)v;
          o[c] = v;
        }
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) {
          mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, d));
          sum += __shfl_xor_sync(0xffffffffu, sum, d);
        }
        if (WARP) {
          if (tid == 0) { a.out_mass[it] = sum; a.out_min[it] = mn; }
        } else {
          const int wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
          if ((threadIdx.x & 31) == 0) { red[2 * wid] = mn; red[2 * wid + 1] = sum; }
          __syncthreads();
          if (threadIdx.x == 0) {
            for (int w = 1; w < nw; ++w) { mn = fmin(mn, red[2 * w]); sum += red[2 * w + 1]; }
            a.out_mass[it] = sum;
            a.out_min[it] = mn;
          }
        }
      }
    }
    group_sync();
  }
}

}  // namespace ptsbe
