// Per-qubit descent sampler for projection-form stages whose work items carry few
// shots each (north-star subsystem 3: "per-qubit conditional marginals once per
// distinct bitstring prefix").
//
// A projection-form stage has P[c] = Re(sum_d v[d] * M_e[d][c]), c < 2^b, with M_e
// fixed per error set (project.cuh).  Late stages of a wide circuit see almost one
// work item per shot, so materialising all 2^b populations to draw one or two
// outcomes from them wastes a factor 2^b / b: the probability of any SET of
// outcomes S is Re(v . sum_{c in S} M_e[:, c]), i.e. one D-term dot product with a
// column that depends on the error set only.  tree_build_kernel sums, once per
// error set, the columns of every "left half" of the binary tree over the b batch
// qubits (first batch qubit = root split = MSB of c, engine.py:489-490); a draw
// then walks the tree: at a node of probability p it evaluates the left child's
// probability pL (one dot product), goes left if r < pL, else right with
// r -= pL, p -= pL.  That is the inverse-CDF draw of rng.multinomial's categorical
// (engine.py:519) evaluated lazily: b dot products per draw instead of 2^b.
//
// The uniforms are the same Philox-4x32-10 counters as sample_kernel
// (draw, prefix rank, stage, global error-set id), so a work item's stream is
// independent of chunking and GPU count.  Guards as engine.py:445-450 /
// 475-476: vanishing mass relative to the trajectory weight, negative
// probabilities beyond tolerance flag the error set.
#pragma once
#include "common.cuh"
#include "executor.cuh"
#include "sampler.cuh"

namespace ptsbe {

constexpr int DS_THREADS = 256;
constexpr int DS_GS = 8;                       // lanes per work item
constexpr int DS_GROUPS = DS_THREADS / DS_GS;  // items in flight per CTA
constexpr int DS_TILE = 512;                   // consecutive items per tile (one table load per error-set run)

template <typename R> struct DsChunk;          // one 16-byte shared-memory load
template <> struct DsChunk<float> { using type = float4; static constexpr int CPC = 2; };
template <> struct DsChunk<double> { using type = double2; static constexpr int CPC = 1; };


struct TreeArgs {
  const void* rec0;     // pass-0 records [error sets][rec_stride] complex
  void* tree;           // out: [error sets][N][dpad] complex
  uint32_t rec_stride, m_off;
  uint32_t D, b, dpad;
  uint32_t n_sets;
};

// tree[e][idx][d]: idx 0 = all outcomes; idx = 2^(t-1) + parent (t = 1..b, parent < 2^(t-1)) =
// outcomes whose first t-1 batch bits spell `parent` and whose t-th bit is 0.
template <typename R>
__global__ void tree_build_kernel(const TreeArgs a) {
  using C = typename CxT<R>::type;
  const uint32_t N = 1u << a.b;
  const uint32_t e = blockIdx.x;
  const uint32_t x = blockIdx.y * blockDim.x + threadIdx.x;
  if (x >= N * a.dpad) return;
  const uint32_t idx = x / a.dpad, d = x % a.dpad;
  C* out = reinterpret_cast<C*>(a.tree) + ((size_t)e * N + idx) * a.dpad + d;
  C s; s.x = 0; s.y = 0;
  if (d < a.D) {
    uint32_t c0 = 0, width = N;
    if (idx) {
      const uint32_t t = 32 - __clz(idx);  // level 1..b
      const uint32_t parent = idx - (1u << (t - 1));
      width = N >> t;
      c0 = parent * 2 * width;
    }
    const C* M = reinterpret_cast<const C*>(a.rec0) + (size_t)e * a.rec_stride + a.m_off + (size_t)d * N + c0;
    double sx = 0.0, sy = 0.0;
    for (uint32_t c = 0; c < width; ++c) { sx += (double)M[c].x; sy += (double)M[c].y; }
    s.x = (R)sx; s.y = (R)sy;
  }
  *out = s;
}

// Same table for b <= TB_MAX_B, built as a reduction tree: a CTA owns TB_ROWS consecutive d of one
// error set, warp w reads row M[d0 + w][0 .. N) once (coalesced), sums pairs level by level in
// shared memory (double), and the CTA writes every node's TB_ROWS consecutive d as one 32/64-byte
// piece.  tree_build_kernel above reads each row b/2 + 1 times with a stride of N between lanes.
constexpr int TB_ROWS = 4;
constexpr int TB_MAX_B = 8;

template <typename R>
__global__ void __launch_bounds__(TB_ROWS * 32) tree_reduce_kernel(const TreeArgs a) {
  using C = typename CxT<R>::type;
  __shared__ double2 nodes[TB_ROWS][2 << TB_MAX_B];  // level k (blocks of 2^k columns) at off_k + q
  const uint32_t N = 1u << a.b;
  const uint32_t e = blockIdx.x, d0 = blockIdx.y * TB_ROWS;
  const uint32_t w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t d = d0 + w;
  double2* nd = nodes[w];
  if (d < a.D) {
    const C* M = reinterpret_cast<const C*>(a.rec0) + (size_t)e * a.rec_stride + a.m_off + (size_t)d * N;
    for (uint32_t c = lane; c < N; c += 32) { const C m = M[c]; nd[c] = make_double2((double)m.x, (double)m.y); }
  } else {
    for (uint32_t c = lane; c < N; c += 32) nd[c] = make_double2(0.0, 0.0);
  }
  __syncwarp();
  uint32_t off = 0;
  for (uint32_t k = 1; k <= a.b; ++k) {
    const uint32_t prev = off, n_prev = N >> (k - 1);
    off += n_prev;
    for (uint32_t q = lane; q < (n_prev >> 1); q += 32) {
      const double2 l = nd[prev + 2 * q], r = nd[prev + 2 * q + 1];
      nd[off + q] = make_double2(l.x + r.x, l.y + r.y);
    }
    __syncwarp();
  }
  __syncthreads();
  // node idx: 0 = all columns = level b, q 0; idx = 2^(t-1) + parent -> level b - t, q = 2 * parent
  C* out = reinterpret_cast<C*>(a.tree) + (size_t)e * N * a.dpad + d0;
  for (uint32_t i = threadIdx.x; i < N * TB_ROWS; i += TB_ROWS * 32) {
    const uint32_t idx = i / TB_ROWS, dd = i % TB_ROWS;
    if (d0 + dd >= a.dpad) continue;
    uint32_t k = a.b, q = 0;
    if (idx) {
      const uint32_t t = 32 - __clz(idx);
      k = a.b - t;
      q = 2 * (idx - (1u << (t - 1)));
    }
    const uint32_t lvl = 2 * N - (2 * N >> k);  // off_k = N + N/2 + ... = 2N (1 - 2^-k)
    const double2 v = nodes[dd][lvl + q];
    C o; o.x = (R)v.x; o.y = (R)v.y;
    out[(size_t)idx * a.dpad + dd] = o;
  }
}

struct DescentArgs {
  const void* v;            // [items of this launch][dpad] complex, row per item, zero padded
  const void* tree;         // [error sets][N][dpad] complex
  const uint32_t* eset;     // [level n] error-set row of every item
  const uint32_t* mult;     // [level n]
  const uint32_t* slot_off; // [level n]
  const uint32_t* eset_id;  // [level n] GLOBAL error-set id (RNG stream)
  const uint32_t* rank;     // [level n]
  uint32_t* slot_index;
  uint32_t* slot_count;
  uint32_t* nnz;
  unsigned long long* flag;
  uint32_t* flag_count;
  const double* set_mass;   // [error-set rows] stage-1 mass (trajectory weight)
  uint32_t first_item, n_items;
  uint32_t b, stage, k0, k1;
  double vanish, neg_abs, neg_rel;
};

template <typename R, int NCH>
__global__ void __launch_bounds__(DS_THREADS) descent_kernel(const DescentArgs a) {
  using CH = typename DsChunk<R>::type;
  constexpr uint32_t COL = DS_GS * NCH;  // 16-byte chunks per column (padded vector length / CPC)
  extern __shared__ __align__(16) unsigned char ds_smem[];
  const uint32_t N = 1u << a.b;
  CH* table = reinterpret_cast<CH*>(ds_smem);                              // [N][COL]
  uint32_t* counters = reinterpret_cast<uint32_t*>(table + (size_t)N * COL);  // [DS_GROUPS][N]
  __shared__ uint32_t s_end;
  const int tid = threadIdx.x, lane = tid & (DS_GS - 1), grp = tid / DS_GS;
  const unsigned gmask = 0xffu << (8 * ((tid & 31) / DS_GS));  // this group's lanes inside its warp
  uint32_t* cnt = counters + (size_t)grp * N;
  const uint32_t n_tiles = (a.n_items + DS_TILE - 1) / DS_TILE;
  const CH* V = reinterpret_cast<const CH*>(a.v);
  const CH* TREE = reinterpret_cast<const CH*>(a.tree);
  uint32_t loaded = 0xffffffffu;

  // Re(v . column) over the group's lanes; every lane of the group gets the same sum
  auto dot = [&](const CH (&v)[NCH], const CH* col) -> double {
    R acc = R(0);
#pragma unroll
    for (int i = 0; i < NCH; ++i) {
      const CH m = col[i * DS_GS + lane];
      if constexpr (DsChunk<R>::CPC == 2) {
        acc = fma(v[i].x, m.x, acc); acc = fma(-v[i].y, m.y, acc);
        acc = fma(v[i].z, m.z, acc); acc = fma(-v[i].w, m.w, acc);
      } else {
        acc = fma(v[i].x, m.x, acc); acc = fma(-v[i].y, m.y, acc);
      }
    }
#pragma unroll
    for (int d = DS_GS / 2; d > 0; d >>= 1) acc += __shfl_xor_sync(gmask, acc, d, DS_GS);
    return (double)acc;
  };

  // a CTA owns a contiguous range of tiles, so consecutive tiles mostly share the loaded table
  const uint32_t tiles_per = (n_tiles + gridDim.x - 1) / gridDim.x;
  const uint32_t tile_end = min(n_tiles, (blockIdx.x + 1) * tiles_per);
  for (uint32_t tile = blockIdx.x * tiles_per; tile < tile_end; ++tile) {
    const uint32_t t1 = min(a.n_items, (tile + 1) * DS_TILE);
    uint32_t pos = tile * DS_TILE;
    while (pos < t1) {
      // ---- the run of items [pos, end) that share error set e ----
      const uint32_t e = a.eset[a.first_item + pos];
      if (tid == 0) s_end = t1;
      __syncthreads();
      for (uint32_t i = pos + 1 + tid; i < t1; i += DS_THREADS)
        if (a.eset[a.first_item + i] != e) { atomicMin(&s_end, i); break; }
      if (e != loaded) {
        const CH* src = TREE + (size_t)e * N * COL;
        for (uint32_t x = tid; x < N * COL; x += DS_THREADS) table[x] = __ldg(src + x);
        loaded = e;
      }
      __syncthreads();
      const uint32_t end = s_end;

      for (uint32_t it = pos + grp; it < end; it += DS_GROUPS) {
        const uint32_t item = a.first_item + it;
        const uint32_t m = a.mult[item];
        CH v[NCH];
#pragma unroll
        for (int i = 0; i < NCH; ++i) v[i] = V[(size_t)it * COL + i * DS_GS + lane];
        const double mass = dot(v, table);
        const double floor_mass = a.vanish * a.set_mass[e];
        const double tol = a.neg_abs - a.neg_rel * mass;
        uint32_t bad = 0;
        if (!(mass >= floor_mass) || !(mass > 0.0)) bad = PTSBE_EIMPOSSIBLE;
        const uint32_t rk = a.rank[item], es = a.eset_id[item], slot0 = a.slot_off[item];

        // one draw: walk the b levels of the tree
        auto draw = [&](uint32_t t) -> uint32_t {
          const Philox4 x = philox4x32_10(t, rk, a.stage, es, a.k0, a.k1);
          const uint64_t x64 = ((uint64_t)x.v[1] << 32) | x.v[0];
          double p = mass;
          double r = (double)(x64 >> 11) * (1.0 / 9007199254740992.0) * mass;  // u in [0, 1)
          uint32_t node = 0;
          for (uint32_t lvl = 1; lvl <= a.b; ++lvl) {
            double pl = dot(v, table + (size_t)((1u << (lvl - 1)) + node) * COL);
            if (pl < tol || p - pl < tol) bad = PTSBE_ENUMERIC;
            pl = fmin(fmax(pl, 0.0), p);
            if (r < pl) { node = 2 * node; p = pl; }
            else { node = 2 * node + 1; r -= pl; p -= pl; }
          }
          return node;
        };

        if (!bad && m == 1) {
          const uint32_t c = draw(0);
          if (!bad && lane == 0) { a.slot_index[slot0] = c; a.slot_count[slot0] = 1; a.nnz[item] = 1; }
        } else if (!bad) {
          for (uint32_t k = lane; k < N; k += DS_GS) cnt[k] = 0;
          __syncwarp(gmask);
          for (uint32_t t = 0; t < m; ++t) {
            const uint32_t c = draw(t);
            if (lane == 0) cnt[c] += 1;
          }
          __syncwarp(gmask);
          if (!bad) {
            // ordered emission: lane owns the consecutive outcomes [lane*per, lane*per+per)
            const uint32_t per = N >= DS_GS ? N / DS_GS : 1;
            const uint32_t k0 = lane * per;
            const bool owns = k0 < N;
            uint32_t mine = 0;
            if (owns)
              for (uint32_t k = k0; k < k0 + per; ++k) mine += cnt[k] != 0;
            uint32_t posn = mine;
#pragma unroll
            for (int d = 1; d < DS_GS; d <<= 1) {
              const uint32_t o = __shfl_up_sync(gmask, posn, d, DS_GS);
              if (lane >= d) posn += o;
            }
            const uint32_t tot = __shfl_sync(gmask, posn, DS_GS - 1, DS_GS);
            posn -= mine;
            if (owns && mine)
              for (uint32_t k = k0; k < k0 + per; ++k) {
                const uint32_t c = cnt[k];
                if (c) { a.slot_index[slot0 + posn] = k; a.slot_count[slot0 + posn] = c; ++posn; }
              }
            if (lane == 0) a.nnz[item] = tot;
          }
          __syncwarp(gmask);
        }
        if (bad && lane == 0) {
          a.nnz[item] = 0;
          atomicMin(a.flag, ((unsigned long long)es << 16) | ((unsigned long long)(a.stage & 0xff) << 8) | bad);
          atomicAdd(a.flag_count, 1u);
        }
      }
      __syncthreads();
      pos = end;
    }
  }
}

}  // namespace ptsbe
