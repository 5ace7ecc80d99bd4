// Lane-per-item interpreter for the tiny per-prefix programs, and the fused
// "per-item steps + per-qubit descent" sampler built on it.
//
// The per-prefix passes of a stage (class >= 1 nodes of the stored path: the few
// contractions that depend on measured bits) are 2-20 steps over rank <= 4
// tensors -- a few hundred multiply-adds per work item, repeated for tens of
// millions of items.  With a group of lanes per item (executor.cuh) most issued
// instructions are step decoding replicated in every group.  Here ONE THREAD owns
// a work item: the step decode and every gather-table entry are warp-uniform
// (served from the program image in shared memory as broadcasts), only operand
// loads and the multiply-adds are per-lane work, and the item's intermediates
// live in a private slice of a warp-interleaved shared-memory arena
// (element e of lane t at [e * 40 + t]: conflict-free for "same element, all
// lanes" as well as for "same item, different elements").
//
// lane_descent_kernel additionally keeps the item's last intermediate on chip:
// the final step (the one that produces the projection vector v) is evaluated by
// the LN_GS-lane group that draws from it, straight into registers, so v never
// exists in memory.  A draw is the unit of work of the descent phase (no loop over an
// item's multiplicity, no idle groups next to a high-multiplicity item); the raw
// per-draw outcomes are merged into ordered (outcome, count) pairs by
// dedup_kernel afterwards.
//
// Same semantics as executor.cuh / descent.cuh (reference engine.py:361-450,
// 493-524); same Philox counters, so a work item's stream does not depend on the
// kernel that serves it.
#pragma once
#include "common.cuh"
#include "descent.cuh"
#include "executor.cuh"
#include "sampler.cuh"

namespace ptsbe {

constexpr int LN_THREADS = 256;
constexpr int LN_WARPS = LN_THREADS / 32;
constexpr int LN_AST = 40;          // arena row pitch in elements: lane t of element e at [e * 40 + t].  Pitch = 8
                                    // (mod 16) puts the elements a 4-lane group reads for one item, and the items of
                                    // the 8 groups of a warp, on disjoint bank pairs (33 gave 4-way conflicts)
constexpr int LN_MAX_LEVELS = 16;   // ancestors kept per lane
constexpr int LN_GS = 4;            // lanes per (item, draw) in the descent phase of the fused kernel
constexpr int LN_NG = 32 / LN_GS;   // such groups per warp
constexpr uint32_t LN_DEDUP_SERIAL = 48;  // draws per item merged by one thread; more: warp path

// shared-memory layout shared by the two kernels (offsets in bytes from the dynamic base)
struct LaneLayout {
  uint32_t steps_off, leaves_off, tables_off, levels_off, arena_off, anc_off, pfx_off, end;
};

__host__ __device__ inline LaneLayout lane_layout(uint32_t n_steps, uint32_t n_leaves, uint32_t n_table_words,
                                                  uint32_t n_levels, uint32_t arena_elems, uint32_t words,
                                                  uint32_t elem_bytes, uint32_t ast = LN_AST) {
  LaneLayout L;
  uint32_t o = 0;
  L.steps_off = o;  o += n_steps * STEP_WORDS * 4;
  L.leaves_off = o; o += n_leaves * LEAF_WORDS * 4;
  L.tables_off = o; o += n_table_words * 4;
  o = (o + 15) & ~15u;
  L.levels_off = o; o += n_levels * (uint32_t)sizeof(LevelDev);
  o = (o + 15) & ~15u;
  L.arena_off = o;  o += LN_WARPS * (arena_elems ? arena_elems : 1) * ast * elem_bytes;
  o = (o + 15) & ~15u;
  L.anc_off = o;    o += n_levels * LN_THREADS * 4;
  o = (o + 15) & ~15u;
  L.pfx_off = o;    o += words * LN_THREADS * 8;
  L.end = (o + 15) & ~15u;
  return L;
}

// One operand of a step as seen by one lane: a (generic) pointer and an element stride --
// LN_AST inside the lane's private arena slice, 1 for a leaf in the operand pool or a record
// of an earlier pass.  One code path serves both, so the inner loops carry no branch.
template <typename C>
struct LaneOp {
  const C* p;
  uint32_t stride;
};

template <typename R>
struct LaneCtx {
  using C = typename CxT<R>::type;
  const uint32_t* steps;
  const uint32_t* leaves;
  const uint32_t* tables;
  const LevelDev* levels;   // shared-memory copy
  C* arena_w;               // this warp's arena
  const uint32_t* anc;      // [level][LN_THREADS]
  const uint64_t* pfx;      // [word][LN_THREADS]
  const C* pool;
  const uint8_t* kraus;
  uint32_t g, arena_fast;
  uint32_t ast;             // arena row pitch: LN_AST (shared memory) or 32 (global arena, BIG)
  uint32_t tiny;            // steps with out_n * kn <= tiny (and kn <= 4) take the compact generic loop

  __device__ __forceinline__ uint32_t bit(uint32_t q, uint32_t slot) const {
    return (uint32_t)((pfx[(q >> 6) * LN_THREADS + slot] >> (63 - (q & 63))) & 1ull);
  }
  // operand (kind, ref) for the work item whose context sits in thread slot `slot`
  __device__ __forceinline__ LaneOp<C> resolve(uint32_t kind, uint32_t ref, uint32_t slot, uint32_t eset) const {
    LaneOp<C> o;
    if (kind == 0) {
      o.p = arena_w + ref * ast + (slot & 31);
      o.stride = ast;
      return o;
    }
    o.stride = 1;
    if (kind == 1) {
      const uint4 lf = reinterpret_cast<const uint4*>(leaves)[ref];
      uint32_t v = 0;
      if (lf.z == 1) v = __ldg(kraus + (size_t)eset * g + lf.w);
      else if (lf.z == 2) v = bit(lf.w, slot);
      o.p = pool + lf.x + (size_t)v * lf.y;
      return o;
    }
    const uint32_t l = kind - 1;
    o.p = reinterpret_cast<const C*>(levels[l].ext) + (size_t)anc[l * LN_THREADS + slot] * levels[l].ext_rec + ref;
    return o;
  }
};

// acc += a' * b' with a' = conj(a) if FA, b' = conj(b) if FB (sign flips fold into the FMAs)
template <bool FA, bool FB, typename C>
__device__ __forceinline__ void cmac_s(C& acc, const C a, const C b) {
  const auto ay = FA ? -a.y : a.y;
  const auto by = FB ? -b.y : b.y;
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(-ay, by, acc.x);
  acc.y = fma(a.x, by, acc.y);
  acc.y = fma(ay, b.x, acc.y);
}

// Decoded step (warp-uniform part)
struct LaneStep {
  uint4 s0, s1, s2;
  const uint32_t *loA, *loB, *hiA, *hiB, *kA, *kB, *dyn;
  uint32_t out_n, kn, lo_n, hi_n, flags;
};

__device__ __forceinline__ LaneStep lane_decode(const uint32_t* steps, const uint32_t* tables, uint32_t s) {
  LaneStep t;
  const uint4* st4 = reinterpret_cast<const uint4*>(steps + (size_t)s * STEP_WORDS);
  t.s0 = st4[0]; t.s1 = st4[1]; t.s2 = st4[2];
  t.out_n = t.s1.z; t.kn = t.s1.w; t.lo_n = t.s2.x; t.hi_n = t.s2.y; t.flags = t.s2.w;
  t.loA = tables + t.s2.z;
  t.loB = t.loA + t.lo_n;
  t.hiA = t.loB + t.lo_n;
  t.hiB = t.hiA + t.hi_n;
  t.kA = t.hiB + t.hi_n;
  t.kB = t.kA + t.kn;
  t.dyn = t.kB + t.kn;
  return t;
}

// Operands of a decoded step for the item in thread slot `slot` (slice views applied; for a
// slice step B is unused and A already points at the selected slice)
template <typename R>
__device__ __forceinline__ void lane_operands(const LaneCtx<R>& cx, const LaneStep& t, uint32_t slot, uint32_t eset,
                                              LaneOp<typename CxT<R>::type>& A, LaneOp<typename CxT<R>::type>& B) {
  A = cx.resolve(t.s0.x, t.s0.y, slot, eset);
  const bool slice = (t.flags & 4u) != 0;
  if (!slice) {
    B = cx.resolve(t.s0.z, t.s0.w, slot, eset);
  } else {
    // B is the basis vector e_x of a measured bit contracted over its only label: a gather
    const uint4 lf = reinterpret_cast<const uint4*>(cx.leaves)[t.s0.w];
    A.p += (cx.bit(lf.w, slot) ? t.kA[1] : t.kA[0]) * A.stride;
    B = A;
  }
  if (t.flags & 8u) {
    const uint32_t* dt = t.dyn;
    const uint32_t na = dt[0];
    uint32_t add = 0;
    for (uint32_t i = 0; i < na; ++i)
      if (cx.bit(dt[1 + 2 * i], slot)) add += dt[2 + 2 * i];
    A.p += add * A.stride;
    dt += 1 + 2 * na;
    const uint32_t nb = dt[0];
    add = 0;
    for (uint32_t i = 0; i < nb; ++i)
      if (cx.bit(dt[1 + 2 * i], slot)) add += dt[2 + 2 * i];
    if (!slice) B.p += add * B.stride;
  }
}

// value of output element c of a decoded step (generic form: tables read per element)
template <typename R>
__device__ __forceinline__ typename CxT<R>::type lane_element(
    const LaneStep& t, const LaneOp<typename CxT<R>::type>& A, const LaneOp<typename CxT<R>::type>& B, uint32_t c) {
  using C = typename CxT<R>::type;
  uint32_t cl = c, ch = 0;
  if (t.hi_n > 1) { ch = c / t.lo_n; cl = c - ch * t.lo_n; }
  uint32_t a0 = t.loA[cl], b0 = t.loB[cl];
  if (t.hi_n > 1) { a0 += t.hiA[ch]; b0 += t.hiB[ch]; }
  const bool fa = t.flags & 1u, fb = t.flags & 2u;
  if (t.flags & 4u) {
    C v = A.p[a0 * A.stride];
    if (fa) v.y = -v.y;
    return v;
  }
  C acc; acc.x = 0; acc.y = 0;
  for (uint32_t k = 0; k < t.kn; ++k) {
    C x = A.p[(a0 + t.kA[k]) * A.stride], y = B.p[(b0 + t.kB[k]) * B.stride];
    if (fa) x.y = -x.y;
    if (fb) y.y = -y.y;
    cmac(acc, x, y);
  }
  return acc;
}

// all outputs of a step with KN contracted entries: k-offsets in registers, conjugation folded
template <typename C, int KN, bool FA, bool FB, int U = 1>
__device__ __forceinline__ void lane_step_fixed(const LaneStep& t, const LaneOp<C>& A, const LaneOp<C>& B, C* O,
                                                uint32_t o_stride, bool store) {
  uint32_t ka[KN], kb[KN];
#pragma unroll
  for (int k = 0; k < KN; ++k) { ka[k] = t.kA[k] * A.stride; kb[k] = t.kB[k] * B.stride; }
  if ((t.flags & 32u) && KN <= 8) {
    // A does not depend on the output index (vector-matrix step): its KN elements are loaded once
    C av[KN];
#pragma unroll
    for (int k = 0; k < KN; ++k) av[k] = A.p[ka[k]];
    for (uint32_t ch = 0, c = 0; ch < t.hi_n; ++ch) {
      const uint32_t hb = t.hi_n > 1 ? t.hiB[ch] : 0u;
      for (uint32_t cl = 0; cl < t.lo_n; ++cl, ++c) {
        const C* pb = B.p + (t.loB[cl] + hb) * B.stride;
        C acc; acc.x = 0; acc.y = 0;
#pragma unroll
        for (int k = 0; k < KN; ++k) cmac_s<FA, FB>(acc, av[k], pb[kb[k]]);
        if (store) O[c * o_stride] = acc;
      }
    }
    return;
  }
  if ((t.flags & 64u) && KN <= 8) {
    // same with the roles swapped (matrix-vector step)
    C bv[KN];
#pragma unroll
    for (int k = 0; k < KN; ++k) bv[k] = B.p[kb[k]];
    for (uint32_t ch = 0, c = 0; ch < t.hi_n; ++ch) {
      const uint32_t ha = t.hi_n > 1 ? t.hiA[ch] : 0u;
      for (uint32_t cl = 0; cl < t.lo_n; ++cl, ++c) {
        const C* pa = A.p + (t.loA[cl] + ha) * A.stride;
        C acc; acc.x = 0; acc.y = 0;
#pragma unroll
        for (int k = 0; k < KN; ++k) cmac_s<FA, FB>(acc, pa[ka[k]], bv[k]);
        if (store) O[c * o_stride] = acc;
      }
    }
    return;
  }
  if constexpr (U > 1 && KN * U <= 16) {
    // U outputs at a time: all their operand loads are issued before the first multiply-add, so a thread
    // that waits on global memory (BIG: the arena is not in shared memory) has 2 * KN * U loads in flight
    // instead of 2 * KN.  Every output is still sum_k in the same order.
    for (uint32_t ch = 0, c = 0; ch < t.hi_n; ++ch) {
      const uint32_t ha = t.hi_n > 1 ? t.hiA[ch] : 0u, hb = t.hi_n > 1 ? t.hiB[ch] : 0u;
      for (uint32_t cl = 0; cl < t.lo_n; cl += U, c += U) {
        C av[U][KN], bv[U][KN];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint32_t cu = min(cl + u, t.lo_n - 1);
          const C* pa = A.p + (t.loA[cu] + ha) * A.stride;
          const C* pb = B.p + (t.loB[cu] + hb) * B.stride;
#pragma unroll
          for (int k = 0; k < KN; ++k) { av[u][k] = pa[ka[k]]; bv[u][k] = pb[kb[k]]; }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          C acc; acc.x = 0; acc.y = 0;
#pragma unroll
          for (int k = 0; k < KN; ++k) cmac_s<FA, FB>(acc, av[u][k], bv[u][k]);
          if (store && cl + u < t.lo_n) O[(c + u) * o_stride] = acc;
        }
      }
    }
    return;
  }
  for (uint32_t ch = 0, c = 0; ch < t.hi_n; ++ch) {
    const uint32_t ha = t.hi_n > 1 ? t.hiA[ch] : 0u, hb = t.hi_n > 1 ? t.hiB[ch] : 0u;
    for (uint32_t cl = 0; cl < t.lo_n; ++cl, ++c) {
      const C* pa = A.p + (t.loA[cl] + ha) * A.stride;
      const C* pb = B.p + (t.loB[cl] + hb) * B.stride;
      C acc; acc.x = 0; acc.y = 0;
#pragma unroll
      for (int k = 0; k < KN; ++k) cmac_s<FA, FB>(acc, pa[ka[k]], pb[kb[k]]);
      if (store) O[c * o_stride] = acc;
    }
  }
}

template <typename C, int KN, int U = 1>
__device__ __forceinline__ void lane_step_kn(const LaneStep& t, const LaneOp<C>& A, const LaneOp<C>& B, C* O,
                                             uint32_t o_stride, bool store) {
  switch (t.flags & 3u) {
    case 0: lane_step_fixed<C, KN, false, false, U>(t, A, B, O, o_stride, store); break;
    case 1: lane_step_fixed<C, KN, true, false, U>(t, A, B, O, o_stride, store); break;
    case 2: lane_step_fixed<C, KN, false, true, U>(t, A, B, O, o_stride, store); break;
    default: lane_step_fixed<C, KN, true, true, U>(t, A, B, O, o_stride, store); break;
  }
}

struct LaneArgs {
  ExecArgs e;               // program, lists, output (HOIST record or VECTOR row per item)
  uint32_t n_leaves, n_table_words, n_levels;
  uint32_t tiny;            // steps of at most this many multiply-adds (kn <= 4) run through the compact generic loop
                            // instead of their unrolled variant: programs of many tiny steps (cfg5) otherwise stall
                            // on instruction fetch across the interpreter's 60 specialised loops
  uint32_t ast;             // arena row pitch in elements; 0: LN_AST.  Kernels whose lanes only ever touch their
                            // own item's slice (lane_x.cuh) run with 32: a fifth less shared memory
};

// Loads the program image and the level table into shared memory (all threads), returns the context.
template <typename R>
__device__ __forceinline__ LaneCtx<R> lane_setup(const LaneArgs& a, unsigned char* smem, const LaneLayout& L,
                                                 bool big = false) {
  using C = typename CxT<R>::type;
  uint32_t* img = reinterpret_cast<uint32_t*>(smem);
  // big: the gather tables stay in global memory (warp-uniform reads, L1-resident) and the arena is global
  const uint32_t ns = a.e.n_steps * STEP_WORDS, nl = a.n_leaves * LEAF_WORDS, nt = big ? 0u : a.n_table_words;
  for (uint32_t i = threadIdx.x; i < ns; i += blockDim.x) img[L.steps_off / 4 + i] = __ldg(a.e.steps + i);
  for (uint32_t i = threadIdx.x; i < nl; i += blockDim.x) img[L.leaves_off / 4 + i] = __ldg(a.e.leaves + i);
  for (uint32_t i = threadIdx.x; i < nt; i += blockDim.x) img[L.tables_off / 4 + i] = __ldg(a.e.tables + i);
  const uint32_t lw = a.n_levels * (uint32_t)(sizeof(LevelDev) / 4);
  const uint32_t* lsrc = reinterpret_cast<const uint32_t*>(a.e.levels);
  for (uint32_t i = threadIdx.x; i < lw; i += blockDim.x) img[L.levels_off / 4 + i] = __ldg(lsrc + i);
  LaneCtx<R> cx;
  cx.steps = img + L.steps_off / 4;
  cx.leaves = img + L.leaves_off / 4;
  cx.tables = big ? a.e.tables : img + L.tables_off / 4;
  cx.levels = reinterpret_cast<const LevelDev*>(smem + L.levels_off);
  cx.ast = big ? 32u : (a.ast ? a.ast : (uint32_t)LN_AST);
  cx.tiny = a.tiny;
  cx.arena_w = big ? reinterpret_cast<C*>(a.e.spill) +
                         ((size_t)blockIdx.x * LN_WARPS + (threadIdx.x >> 5)) * a.e.arena_fast * 32
                   : reinterpret_cast<C*>(smem + L.arena_off) +
                         (size_t)(threadIdx.x >> 5) * (a.e.arena_fast ? a.e.arena_fast : 1) * cx.ast;
  cx.anc = reinterpret_cast<const uint32_t*>(smem + L.anc_off);
  cx.pfx = reinterpret_cast<const uint64_t*>(smem + L.pfx_off);
  cx.pool = reinterpret_cast<const C*>(a.e.pool);
  cx.kraus = a.e.kraus;
  cx.g = a.e.g;
  cx.arena_fast = a.e.arena_fast;
  return cx;
}

// Item context of this thread's slot: ancestors and prefix words -> shared memory.  Returns the
// error-set row.
template <typename R>
__device__ __forceinline__ uint32_t lane_item_context(const LaneArgs& a, const LaneCtx<R>& cx, unsigned char* smem,
                                                      const LaneLayout& L, uint32_t item) {
  uint32_t* anc = reinterpret_cast<uint32_t*>(smem + L.anc_off);
  uint64_t* pfx = reinterpret_cast<uint64_t*>(smem + L.pfx_off);
  const uint32_t slot = threadIdx.x;
  uint32_t cur = item;
  anc[a.e.level * LN_THREADS + slot] = cur;
  for (int l = (int)a.e.level; l > 1; --l) {
    cur = __ldg(cx.levels[l].parent + cur);
    anc[(l - 1) * LN_THREADS + slot] = cur;
  }
  const LevelDev& lv = cx.levels[a.e.level];
  for (uint32_t w = 0; w < a.e.words; ++w) pfx[w * LN_THREADS + slot] = __ldg(lv.prefix + (size_t)w * lv.n + item);
  return __ldg(lv.eset + item);
}

// Runs steps [s0, s1) for the item of this thread.  Outputs of kind 0 go to the private arena;
// outputs of kind 1 to `rec` (this item's record / vector row) when `live`.
template <typename R, int U = 1>
__device__ __forceinline__ void lane_run(const LaneCtx<R>& cx, uint32_t s0, uint32_t s1, uint32_t eset,
                                         typename CxT<R>::type* rec, bool live) {
  using C = typename CxT<R>::type;
  const uint32_t slot = threadIdx.x, ls = threadIdx.x & 31;
  for (uint32_t s = s0; s < s1; ++s) {
    const LaneStep t = lane_decode(cx.steps, cx.tables, s);
    LaneOp<C> A, B;
    lane_operands<R>(cx, t, slot, eset, A, B);
    const bool to_arena = t.s1.x == 0;
    C* O = to_arena ? cx.arena_w + t.s1.y * cx.ast + ls : rec + t.s1.y;
    const uint32_t o_stride = to_arena ? cx.ast : 1u;
    const bool store = to_arena || live;
    if (t.flags & 4u) {
      for (uint32_t c = 0; c < t.out_n; ++c) {
        const C v = lane_element<R>(t, A, B, c);
        if (store) O[c * o_stride] = v;
      }
    } else if (t.kn <= 4 && t.out_n * t.kn <= cx.tiny) {
      for (uint32_t c = 0; c < t.out_n; ++c) {
        const C v = lane_element<R>(t, A, B, c);
        if (store) O[c * o_stride] = v;
      }
    } else {
      switch (t.kn) {
        case 1: lane_step_kn<C, 1, U>(t, A, B, O, o_stride, store); break;
        case 2: lane_step_kn<C, 2, U>(t, A, B, O, o_stride, store); break;
        case 4: lane_step_kn<C, 4, U>(t, A, B, O, o_stride, store); break;
        case 8: lane_step_kn<C, 8, U>(t, A, B, O, o_stride, store); break;
        case 16: lane_step_kn<C, 16>(t, A, B, O, o_stride, store); break;
        default:
          for (uint32_t c = 0; c < t.out_n; ++c) {
            const C v = lane_element<R>(t, A, B, c);
            if (store) O[c * o_stride] = v;
          }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// standalone: hoist passes p >= 1 and vector rows, one thread per work item
// ---------------------------------------------------------------------------
// Marginal epilogue of a lane-owned item (reference engine.py:445-450: real part, minimum before
// clamping, clamp, mass), bit-compatible with the GS-lane epilogue of exec_kernel: that one gives lane t
// the elements c = t (mod GS), sums them in double in increasing c and folds the GS partial sums with
// xor-butterflies of distance GS/2 .. 1.  Here one thread keeps the GS partial sums itself and folds
// them in the same tree, so the mass does not depend on which kernel served the error set.
template <typename R, int GS>
__device__ __forceinline__ void lane_marginal_epilogue(const typename CxT<R>::type* res, uint32_t res_stride,
                                                       uint32_t n, R* o, bool live, double& mass, double& mn_out) {
  double part[GS];
#pragma unroll
  for (int t = 0; t < GS; ++t) part[t] = 0.0;
  double mn = 1e300;
  for (uint32_t c0 = 0; c0 < n; c0 += GS) {
#pragma unroll
    for (int t = 0; t < GS; ++t) {
      const uint32_t c = c0 + t;
      if (c < n) {
        R v = res[(size_t)c * res_stride].x;
        mn = fmin(mn, (double)v);
        v = v > R(0) ? v : R(0);
        part[t] += (double)v;
        if (live) o[c] = v;
      }
    }
  }
#pragma unroll
  for (int d = GS / 2; d > 0; d >>= 1)
#pragma unroll
    for (int t = 0; t < d; ++t) part[t] += part[t + d];
  mass = part[0];
  mn_out = mn;
}

// BIG: class-0 programs of hundreds of steps over arenas of kilobytes (cfg5: 320-560 steps, 650-1600
// elements) when the batch holds tens of thousands of error sets.  A group of lanes per item spends ~100
// issued instructions per step on decoding for a handful of multiply-adds; with one thread per error set the
// decode is shared by 32 items and the arena moves to global memory, interleaved [element][lane] so that every
// access of a warp is one or two full cache lines (a.e.spill: [resident warps][arena_fast][32]).
template <typename R, bool BIG = false>
__global__ void __launch_bounds__(LN_THREADS) exec_lane_kernel(const LaneArgs a) {
  using C = typename CxT<R>::type;
  extern __shared__ __align__(16) unsigned char ln_smem[];
  const LaneLayout L = lane_layout(a.e.n_steps, a.n_leaves, BIG ? 0u : a.n_table_words, a.n_levels,
                                   BIG ? 0u : a.e.arena_fast, a.e.words, (uint32_t)sizeof(C));
  const LaneCtx<R> cx = lane_setup<R>(a, ln_smem, L, BIG);
  __syncthreads();
  const uint32_t per_round = gridDim.x * LN_THREADS;
  const uint32_t rounds = (a.e.n_items + per_round - 1) / per_round;
  for (uint32_t r = 0; r < rounds; ++r) {
    uint32_t it = r * per_round + blockIdx.x * LN_THREADS + threadIdx.x;
    const bool live = it < a.e.n_items;
    if (!live) it = a.e.n_items - 1;
    const uint32_t item = a.e.first_item + it;
    const uint32_t eset = lane_item_context<R>(a, cx, ln_smem, L, item);
    __syncwarp();
    C* rec = a.e.mode == EXEC_VECTOR ? reinterpret_cast<C*>(a.e.out) + (size_t)it * a.e.vec_row
                                     : reinterpret_cast<C*>(a.e.out) + (size_t)item * a.e.out_elems;
    lane_run<R>(cx, 0, a.e.n_steps, eset, rec, live);  // U > 1 (outputs in flight) measured slower: registers
    if constexpr (BIG) {
      if (a.e.mode == EXEC_MARGINAL) {
        // stage-1 marginal pass: the root sits in this lane's arena slice
        const C* res = cx.arena_w + (size_t)a.e.result_ref * 32 + (threadIdx.x & 31);
        R* o = reinterpret_cast<R*>(a.e.out) + (size_t)it * a.e.out_elems;
        double mass, mn;
        switch (a.e.item_bytes) {  // lanes per item of the group kernel this one stands in for
          case 8: lane_marginal_epilogue<R, 8>(res, 32, a.e.out_elems, o, live, mass, mn); break;
          case 16: lane_marginal_epilogue<R, 16>(res, 32, a.e.out_elems, o, live, mass, mn); break;
          default: lane_marginal_epilogue<R, 32>(res, 32, a.e.out_elems, o, live, mass, mn); break;
        }
        if (live) { a.e.out_mass[it] = mass; a.e.out_min[it] = mn; }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// fused: per-item steps (thread per item) + per-qubit descent (LN_GS lanes per draw)
// ---------------------------------------------------------------------------
struct LaneDescentArgs {
  LaneArgs l;               // l.e.out unused; the last step of the program produces v
  DescentArgs d;            // d.v unused
  uint32_t* big_list;       // items with more than LN_DEDUP_SERIAL draws (merged by dedup_big_kernel)
  uint32_t* big_count;
  uint32_t tile;            // consecutive items a CTA takes at a time (multiple of LN_THREADS)
  uint32_t warp_runs;       // non-zero: every warp walks its own share of the tile with a private copy of the
                            // tree table (short runs of items per error set: cfg5 has <= 100), instead of the
                            // CTA serving one error set at a time between two barriers
  const uint32_t* herm_map; // HERM: [D] real slot -> c | c' << 12 | kind << 24 (kind 0: Re v_c, 1: Im v_c)
};

// Hermitian packing (HERM).  When the projection vector is v = x (x) conj(x) (the ket / bra halves
// of the cut are mirror images), v[c'] = conj(v[c]) for the transposed index c', so
//   Re sum_c v_c C_c = sum_diag v_c Re C_c + sum_{c < c'} Re v_c (Re C_c + Re C_c') - Im v_c (Im C_c - Im C_c'):
// D REAL products instead of D complex ones.  The tree columns are packed accordingly by
// herm_pack_kernel, which halves both the table in shared memory and the work of every tree level.
struct HermPackArgs {
  const void* tree;         // [sets][N][dpad_c] complex columns (tree_build_kernel)
  void* packed;             // [sets][N][dpad_r] reals
  const uint32_t* map;      // [D] c | c' << 12 | kind << 24
  const uint32_t* canon;    // null, or [D]: slot s is stored at position canon[s] & 0xffff, negated if bit 31 is
                            // set (canonical order of lane_x.cuh)
  uint32_t D, dpad_c, dpad_r, b;
};

template <typename R>
__global__ void herm_pack_kernel(const HermPackArgs a) {
  using C = typename CxT<R>::type;
  const uint32_t N = 1u << a.b;
  const uint32_t e = blockIdx.x;
  const uint32_t x = blockIdx.y * blockDim.x + threadIdx.x;
  if (x >= N * a.dpad_r) return;
  const uint32_t node = x / a.dpad_r, s = x % a.dpad_r;
  R out = R(0);
  uint32_t dst = s;
  if (s < a.D) {
    const uint32_t m = __ldg(a.map + s);
    const uint32_t c = m & 0xfffu, c2 = (m >> 12) & 0xfffu, kind = m >> 24;
    const C* col = reinterpret_cast<const C*>(a.tree) + ((size_t)e * N + node) * a.dpad_c;
    const C u = col[c], w = col[c2];
    if (kind == 0) out = (c == c2) ? u.x : u.x + w.x;
    else if (kind == 1) out = -(u.y - w.y);
    if (a.canon) {
      const uint32_t cm = __ldg(a.canon + s);
      dst = cm & 0xffffu;
      if (cm >> 31) out = -out;
    }
  }
  reinterpret_cast<R*>(a.packed)[((size_t)e * N + node) * a.dpad_r + dst] = out;
}

// tree_reduce_kernel + herm_pack_kernel in one pass for small tables (cfg5: 64 nodes x 16 reals per error set,
// 10^5 error sets per stage, ~100 work items each): a warp owns an error set, reduces the D rows of M one after
// the other (pairwise sums in double, as tree_reduce_kernel) into a [D][N] table of rounded node values in
// shared memory and writes the packed columns coalesced.  The two-kernel path launched 4 x 10^5 CTAs of 128
// threads for the trees, wrote them to HBM and read them back: 7.4 of cfg5's 54 ms per step.  Same values.
struct TreeHermArgs {
  const void* rec0;         // pass-0 records [error sets][rec_stride] complex
  void* packed;             // out: [sets][N][dpad_r] reals
  const uint32_t* map;      // [D] c | c' << 12 | kind << 24
  const uint32_t* canon;    // null or [D] (HermPackArgs)
  uint32_t rec_stride, m_off, D, b, dpad_r, n_sets;
};
constexpr int TH_WARPS = 4;

template <typename R>
__global__ void __launch_bounds__(TH_WARPS * 32) tree_herm_kernel(const TreeHermArgs a) {
  using C = typename CxT<R>::type;
  extern __shared__ __align__(16) unsigned char th_smem[];
  const uint32_t N = 1u << a.b;
  const uint32_t w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const size_t per_warp = (size_t)2 * N * sizeof(double2) + (size_t)a.D * N * sizeof(C);
  double2* nd = reinterpret_cast<double2*>(th_smem + w * per_warp);   // reduction tree of one row
  C* tr = reinterpret_cast<C*>(nd + 2 * N);                           // [D][N] node values, rounded
  for (uint32_t e = blockIdx.x * TH_WARPS + w; e < a.n_sets; e += gridDim.x * TH_WARPS) {
    const C* M0 = reinterpret_cast<const C*>(a.rec0) + (size_t)e * a.rec_stride + a.m_off;
    for (uint32_t d = 0; d < a.D; ++d) {
      const C* M = M0 + (size_t)d * N;
      for (uint32_t c = lane; c < N; c += 32) { const C m = M[c]; nd[c] = make_double2((double)m.x, (double)m.y); }
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
      // node idx: 0 = all columns = level b, q 0; idx = 2^(t-1) + parent -> level b - t, q = 2 * parent
      for (uint32_t idx = lane; idx < N; idx += 32) {
        uint32_t k = a.b, q = 0;
        if (idx) {
          const uint32_t t = 32 - __clz(idx);
          k = a.b - t;
          q = 2 * (idx - (1u << (t - 1)));
        }
        const double2 v = nd[2 * N - (2 * N >> k) + q];
        C o; o.x = (R)v.x; o.y = (R)v.y;
        tr[d * N + idx] = o;
      }
      __syncwarp();
    }
    R* out = reinterpret_cast<R*>(a.packed) + (size_t)e * N * a.dpad_r;
    const uint32_t dsh = 31 - __clz(a.dpad_r);  // dpad_r = lanes x chunks x reals per chunk: a power of two
    for (uint32_t x = lane; x < N * a.dpad_r; x += 32) {
      const uint32_t node = x >> dsh, sl = x & (a.dpad_r - 1);
      R val = R(0);
      uint32_t dst = sl;
      if (sl < a.D) {
        const uint32_t m = __ldg(a.map + sl);
        const uint32_t c = m & 0xfffu, c2 = (m >> 12) & 0xfffu, kind = m >> 24;
        const C u = tr[c * N + node], v2 = tr[c2 * N + node];
        if (kind == 0) val = (c == c2) ? u.x : u.x + v2.x;
        else if (kind == 1) val = -(u.y - v2.y);
        if (a.canon) {
          const uint32_t cm = __ldg(a.canon + sl);
          dst = cm & 0xffffu;
          if (cm >> 31) val = -val;
        }
      }
      out[(size_t)node * a.dpad_r + dst] = val;
    }
    __syncwarp();
  }
}

template <typename R, int NCH, bool HERM>
__global__ void __launch_bounds__(LN_THREADS, 2) lane_descent_kernel(const LaneDescentArgs a) {
  using C = typename CxT<R>::type;
  using CH = typename DsChunk<R>::type;
  constexpr int CPC = HERM ? 2 * DsChunk<R>::CPC : DsChunk<R>::CPC;  // vector elements per 16-byte chunk
  constexpr uint32_t COL = LN_GS * NCH;
  // Shared-memory row pitch of the tree table.  A 4-lane group reads 64 contiguous bytes (16 banks) of its
  // node's row per chunk; the 8 groups of a warp read 8 different rows.  With an even chunk count the rows are
  // unpadded (every row starts at bank 0, chunk i covers the bank half i & 1) and the groups walk the chunks in
  // an order rotated by their parity (ROT below): at every step four groups hit each half -> 4 wavefronts per
  // 512-byte warp access, the minimum, for ANY combination of rows.  (One chunk of padding, the previous
  // layout, left ~1.5x the ideal wavefronts on this load, the largest shared-memory consumer of the kernel.)
  constexpr uint32_t COLP = NCH >= 2 ? COL : COL + 1;
  extern __shared__ __align__(16) unsigned char ln_smem[];
  const ExecArgs& e = a.l.e;
  const DescentArgs& d = a.d;
  const LaneLayout L = lane_layout(e.n_steps, a.l.n_leaves, a.l.n_table_words, a.l.n_levels, e.arena_fast, e.words,
                                   (uint32_t)sizeof(C));
  const LaneCtx<R> cx = lane_setup<R>(a.l, ln_smem, L);
  const uint32_t N = 1u << d.b;
  // after the interpreter's region: per-warp scratch, then the tree table
  double* mass_s = reinterpret_cast<double*>(ln_smem + L.end);                 // [LN_THREADS]
  uint32_t* cum_s = reinterpret_cast<uint32_t*>(mass_s + LN_THREADS);          // [LN_THREADS]
  uint32_t* slot0_s = cum_s + LN_THREADS;                                      // [LN_THREADS]
  uint32_t* eset_s = slot0_s + LN_THREADS;                                     // [LN_THREADS]
  uint32_t* bad_s = eset_s + LN_THREADS;                                       // [LN_THREADS]
  uint32_t* rank_s = bad_s + LN_THREADS;                                       // [LN_THREADS]
  uint32_t* gid_s = rank_s + LN_THREADS;                                       // [LN_THREADS]
  const int tid = threadIdx.x, lane32 = tid & 31, warp = tid >> 5;
  const bool WR = a.warp_runs != 0;
  CH* table = reinterpret_cast<CH*>(gid_s + LN_THREADS) + (WR ? (size_t)warp * N * COLP : 0);  // [N][COLP]
  __shared__ uint32_t s_end;
  const int lane = tid & (LN_GS - 1), grp = lane32 / LN_GS;                    // LN_GS-lane groups
  const unsigned gmask = ((1u << LN_GS) - 1u) << (LN_GS * grp);
  const int ROT = NCH >= 2 ? (grp & 1) : 0;  // register slot i of v holds logical chunk i ^ ROT
  const uint32_t wbase = warp * 32;
  const CH* TREE = reinterpret_cast<const CH*>(d.tree);
  uint32_t loaded = 0xffffffffu;
  __syncthreads();  // program image complete
  const LaneStep last = lane_decode(cx.steps, cx.tables, e.n_steps - 1);

  // v of the item in warp slot i, distributed over this group's lanes: lane holds the 16-byte
  // chunks {k * LN_GS + lane}, i.e. elements CPC * (k * LN_GS + lane) + {0, CPC - 1}.
  // Common case (v = x (x) conj(x): one multiply per element, no slice): the gather offsets of
  // this lane's elements do not depend on the item -- resolved once per kernel.
  const bool fast_last = HERM || (last.kn == 1 && !(last.flags & 4u) && last.hi_n == 1);
  const uint32_t last_sa = last.s0.x == 0 ? LN_AST : 1u, last_sb = last.s0.z == 0 ? LN_AST : 1u;
  uint32_t via[NCH * CPC], vib[NCH * CPC];
  uint32_t vim = 0;  // HERM: bit k set -> slot k takes the imaginary part
#pragma unroll
  for (int k = 0; k < NCH * CPC; ++k) {
    uint32_t c = CPC * (((k / CPC) ^ ROT) * LN_GS + lane) + (k % CPC);
    bool ok = fast_last && c < last.out_n;
    if constexpr (HERM) {
      if (ok) {
        const uint32_t m = __ldg(a.herm_map + c);  // c | c' << 12 | kind << 24
        c = m & 0xfffu;
        if ((m >> 24) == 1u) vim |= 1u << k;
        ok = (m >> 24) < 2u;
      }
    }
    via[k] = ok ? (last.loA[c] + last.kA[0]) * last_sa : 0xffffffffu;
    vib[k] = ok ? (last.loB[c] + last.kB[0]) * last_sb : 0u;
  }
  const R sgn_a = (last.flags & 1u) ? R(-1) : R(1), sgn_b = (last.flags & 2u) ? R(-1) : R(1);
  auto vector_of = [&](uint32_t i, CH (&v)[NCH]) {
    const uint32_t slot = wbase + i;
    LaneOp<C> A, B;
    lane_operands<R>(cx, last, slot, eset_s[slot], A, B);
    C x[NCH * CPC];
#pragma unroll
    for (int k = 0; k < NCH * CPC; ++k) {
      x[k].x = 0; x[k].y = 0;
      if (fast_last) {
        if (via[k] != 0xffffffffu) {
          C p = A.p[via[k]], q = B.p[vib[k]];
          p.y *= sgn_a; q.y *= sgn_b;
          cmac(x[k], p, q);
        }
      } else {
        const uint32_t c = CPC * (((k / CPC) ^ ROT) * LN_GS + lane) + (k % CPC);
        if (c < last.out_n) x[k] = lane_element<R>(last, A, B, c);
      }
    }
    if constexpr (HERM) {
      // real slots: Re or Im of the selected element
      R w[NCH * CPC];
#pragma unroll
      for (int k = 0; k < NCH * CPC; ++k) w[k] = ((vim >> k) & 1u) ? x[k].y : x[k].x;
#pragma unroll
      for (int k = 0; k < NCH; ++k) {
        if constexpr (CPC == 4) { v[k].x = w[4 * k]; v[k].y = w[4 * k + 1]; v[k].z = w[4 * k + 2]; v[k].w = w[4 * k + 3]; }
        else { v[k].x = w[2 * k]; v[k].y = w[2 * k + 1]; }
      }
    } else {
#pragma unroll
      for (int k = 0; k < NCH; ++k) {
        if constexpr (CPC == 2) { v[k].x = x[2 * k].x; v[k].y = x[2 * k].y; v[k].z = x[2 * k + 1].x; v[k].w = x[2 * k + 1].y; }
        else { v[k].x = x[k].x; v[k].y = x[k].y; }
      }
    }
  };
  // One partial sum per chunk (independent FMA chains), pairs of chunks added first: a + b is commutative, so
  // the result does not depend on the group's chunk order (ROT) -- an item's draws are the same whichever
  // group of whichever warp serves it.
  auto dot = [&](const CH (&v)[NCH], const CH* col) -> R {
    R part[NCH];
#pragma unroll
    for (int i = 0; i < NCH; ++i) {
      const CH m = col[(i ^ ROT) * LN_GS + lane];
      R acc;
      if constexpr (HERM) {
        acc = v[i].x * m.x; acc = fma(v[i].y, m.y, acc);
        if constexpr (CPC == 4) { acc = fma(v[i].z, m.z, acc); acc = fma(v[i].w, m.w, acc); }
      } else if constexpr (CPC == 2) {
        acc = v[i].x * m.x; acc = fma(-v[i].y, m.y, acc);
        acc = fma(v[i].z, m.z, acc); acc = fma(-v[i].w, m.w, acc);
      } else {
        acc = v[i].x * m.x; acc = fma(-v[i].y, m.y, acc);
      }
      part[i] = acc;
    }
    R acc = part[0];
    if constexpr (NCH >= 2) {
      acc += part[1];
#pragma unroll
      for (int i = 2; i < NCH; i += 2) acc += part[i] + part[i + 1];
    }
#pragma unroll
    for (int s = LN_GS / 2; s > 0; s >>= 1) acc += __shfl_xor_sync(gmask, acc, s, LN_GS);
    return acc;
  };

  const uint32_t n_tiles = (d.n_items + a.tile - 1) / a.tile;
  const uint32_t tiles_per = (n_tiles + gridDim.x - 1) / gridDim.x;
  const uint32_t tile_end = min(n_tiles, (blockIdx.x + 1) * tiles_per);
  __syncthreads();
  for (uint32_t tile = blockIdx.x * tiles_per; tile < tile_end; ++tile) {
    uint32_t t1 = min(d.n_items, (tile + 1) * a.tile);
    uint32_t pos = tile * a.tile;
    if (WR) {  // this warp's share of the tile
      const uint32_t per = ((t1 - pos + LN_WARPS - 1) / LN_WARPS + 31) & ~31u;
      pos = min(t1, pos + warp * per);
      t1 = min(t1, pos + per);
    }
    while (pos < t1) {
      // ---- the run of items [pos, end) that share error set er ----
      const uint32_t er = d.eset[d.first_item + pos];
      uint32_t end = t1;
      if (WR) {
        for (uint32_t i0 = pos + 1; i0 < t1; i0 += 32) {
          const uint32_t i = i0 + lane32;
          const unsigned differs = __ballot_sync(0xffffffffu, i < t1 && d.eset[d.first_item + i] != er);
          if (differs) { end = i0 + __ffs(differs) - 1; break; }
        }
        if (er != loaded) {
          const CH* src = TREE + (size_t)er * N * COL;
          for (uint32_t x = lane32; x < N * COL; x += 32) table[(x / COL) * COLP + (x % COL)] = __ldg(src + x);
          loaded = er;
        }
        __syncwarp();
      } else {
        if (tid == 0) s_end = t1;
        __syncthreads();
        for (uint32_t i = pos + 1 + tid; i < t1; i += LN_THREADS)
          if (d.eset[d.first_item + i] != er) { atomicMin(&s_end, i); break; }
        if (er != loaded) {
          const CH* src = TREE + (size_t)er * N * COL;
          for (uint32_t x = tid; x < N * COL; x += LN_THREADS) table[(x / COL) * COLP + (x % COL)] = __ldg(src + x);
          loaded = er;
        }
        __syncthreads();
        end = s_end;
      }
      const double floor_mass = d.vanish * d.set_mass[er];

      for (uint32_t w0 = pos + (WR ? 0u : wbase); w0 < end; w0 += (WR ? 32u : (uint32_t)LN_THREADS)) {
        // ---- phase A: this lane's item, every step but the last ----
        const uint32_t it = w0 + lane32;
        const bool live = it < end;
        const uint32_t item = d.first_item + (live ? it : end - 1);
        const uint32_t es_row = lane_item_context<R>(a.l, cx, ln_smem, L, item);
        eset_s[tid] = es_row;
        __syncwarp();
        lane_run<R>(cx, 0, e.n_steps - 1, es_row, nullptr, false);
        uint32_t m = live ? d.mult[item] : 0u;
        slot0_s[tid] = d.slot_off[item];
        rank_s[tid] = d.rank[item];     // Philox counter words of this lane's item: staged here so a
        gid_s[tid] = d.eset_id[item];   // draw does not start with an L2 round trip
        bad_s[tid] = 0;
        __syncwarp();
        // one descent from v: decisions in the arithmetic type of the path (float for complex64: the
        // conditional marginals carry 1e-5 relative error anyway; double for complex128, compatible
        // with the oracle's float64 inverse-CDF walk)
        auto descend = [&](const CH (&v)[NCH], R mass, uint32_t t, uint32_t i, uint32_t& bad) -> uint32_t {
          const R tol = (R)(d.neg_abs - d.neg_rel * (double)mass);
          const Philox4 x = philox4x32_10(t, rank_s[wbase + i], d.stage, gid_s[wbase + i], d.k0, d.k1);
          const uint64_t x64 = ((uint64_t)x.v[1] << 32) | x.v[0];
          R p = mass;
          R r = (R)((double)(x64 >> 11) * (1.0 / 9007199254740992.0)) * mass;  // u in [0, 1)
          if (sizeof(R) == 4 && !(r < mass)) r = nextafterf((float)mass, 0.0f);  // u rounded up to 1.0f
          uint32_t node = 0;
          for (uint32_t lvl = 1; lvl <= d.b; ++lvl) {
            R pl = dot(v, table + (size_t)((1u << (lvl - 1)) + node) * COLP);
            if (pl < tol || p - pl < tol) bad = PTSBE_ENUMERIC;
            pl = fmin(fmax(pl, R(0)), p);
            if (r < pl) { node = 2 * node; p = pl; }
            else { node = 2 * node + 1; r -= pl; p -= pl; }
          }
          return node;
        };
        // draws 1.. of the items that carry more than one shot: inclusive scan of (m - 1)
        uint32_t incl = m > 1 ? m - 1 : 0u;
#pragma unroll
        for (int s = 1; s < 32; s <<= 1) {
          const uint32_t o = __shfl_up_sync(0xffffffffu, incl, s);
          if (lane32 >= s) incl += o;
        }
        cum_s[tid] = incl;
        const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
        __syncwarp();
        // ---- phase B: one (item, draw) per LN_GS-lane group and round.  Rounds [0, item_rounds): the
        // warp's items in order -- v, mass (guards as descent.cuh) and draw 0; later rounds: the
        // remaining draws of multi-shot items, v recomputed, mass from shared memory ----
        const uint32_t n_live = min(32u, end - w0);
        const uint32_t item_rounds = (n_live + LN_NG - 1) / LN_NG, rounds = item_rounds + (total + LN_NG - 1) / LN_NG;
        for (uint32_t rd = 0; rd < rounds; ++rd) {
          const bool first = rd < item_rounds;  // warp-uniform
          bool active;
          uint32_t i, t;
          if (first) {
            active = rd * LN_NG + grp < n_live;
            i = active ? rd * LN_NG + grp : n_live - 1;
            t = 0;
          } else {
            const uint32_t d0 = (rd - item_rounds) * LN_NG;
            active = d0 + grp < total;
            const uint32_t dr = active ? d0 + grp : total - 1;
            uint32_t lo = 0, hi = 31;  // smallest i with cum[i] > dr
            while (lo < hi) {
              const uint32_t mid = (lo + hi) >> 1;
              if (cum_s[wbase + mid] > dr) hi = mid; else lo = mid + 1;
            }
            i = lo;
            t = 1 + dr - (i ? cum_s[wbase + i - 1] : 0u);
          }
          CH v[NCH];
          vector_of(i, v);
          uint32_t bad = 0;
          R mass;
          if (first) {
            mass = dot(v, table);
            if (!((double)mass >= floor_mass) || !(mass > R(0))) bad = PTSBE_EIMPOSSIBLE;
          } else {
            mass = (R)mass_s[wbase + i];
            bad = bad_s[wbase + i] == PTSBE_EIMPOSSIBLE ? PTSBE_EIMPOSSIBLE : 0u;
          }
          uint32_t node = 0;
          if (!bad) node = descend(v, mass, t, i, bad);  // group-uniform branch
          if (active && lane == 0) {
            if (first) mass_s[wbase + i] = (double)mass;
            if (bad) {
              bad_s[wbase + i] = bad;
            } else {
              const uint32_t sl = slot0_s[wbase + i] + t;
              d.slot_index[sl] = node;
              d.slot_count[sl] = 1;
            }
          }
          if (first && rd + 1 == item_rounds) __syncwarp();  // masses and flags visible to the later rounds
        }
        __syncwarp();
        // ---- per item: number of raw children, flags, hand-over of long draw lists ----
        if (live) {
          const uint32_t bad = bad_s[tid];
          if (bad) {
            d.nnz[item] = 0;
            atomicMin(d.flag, ((unsigned long long)d.eset_id[item] << 16) |
                                  ((unsigned long long)(d.stage & 0xff) << 8) | bad);
            atomicAdd(d.flag_count, 1u);
          } else {
            d.nnz[item] = m;
            if (m > LN_DEDUP_SERIAL) a.big_list[atomicAdd(a.big_count, 1u)] = item;
          }
        }
        __syncwarp();
      }
      if (WR) __syncwarp(); else __syncthreads();
      pos = end;
    }
  }
}

// ---------------------------------------------------------------------------
// raw per-draw outcomes -> ordered (outcome, count) pairs
// ---------------------------------------------------------------------------
struct DedupArgs {
  const uint32_t* slot_off;
  uint32_t* slot_index;
  uint32_t* slot_count;
  uint32_t* nnz;
  const uint32_t* big_list;
  const uint32_t* big_count;
  uint32_t first_item, n_items, b;
};

// one thread per item with 2..LN_DEDUP_SERIAL draws: insertion sort + run-length merge in place
__global__ void dedup_kernel(const DedupArgs a) {
  const uint32_t it = blockIdx.x * blockDim.x + threadIdx.x;
  if (it >= a.n_items) return;
  const uint32_t item = a.first_item + it;
  const uint32_t m = a.nnz[item];
  if (m < 2 || m > LN_DEDUP_SERIAL) return;
  uint32_t* idx = a.slot_index + a.slot_off[item];
  uint32_t* cnt = a.slot_count + a.slot_off[item];
  if (m <= 8) {
    // the common case: all draws in registers (one round of independent loads), 19-comparator
    // odd-even merge network, run-length merge straight from the registers
    uint32_t v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = (uint32_t)i < m ? idx[i] : 0xFFFFFFFFu;
#define PTSBE_CE(i, j) { const uint32_t lo = min(v[i], v[j]), hi = max(v[i], v[j]); v[i] = lo; v[j] = hi; }
    PTSBE_CE(0, 1) PTSBE_CE(2, 3) PTSBE_CE(4, 5) PTSBE_CE(6, 7)
    PTSBE_CE(0, 2) PTSBE_CE(1, 3) PTSBE_CE(4, 6) PTSBE_CE(5, 7)
    PTSBE_CE(1, 2) PTSBE_CE(5, 6)
    PTSBE_CE(0, 4) PTSBE_CE(1, 5) PTSBE_CE(2, 6) PTSBE_CE(3, 7)
    PTSBE_CE(2, 4) PTSBE_CE(3, 5)
    PTSBE_CE(1, 2) PTSBE_CE(3, 4) PTSBE_CE(5, 6)
#undef PTSBE_CE
    uint32_t out = 0, run = 1;
#pragma unroll
    for (int i = 1; i <= 8; ++i) {
      if ((uint32_t)i <= m) {
        const bool same = (uint32_t)i < m && v[i < 8 ? i : 7] == v[i - 1];
        if (same) {
          ++run;
        } else {
          idx[out] = v[i - 1];
          cnt[out] = run;
          ++out;
          run = 1;
        }
      }
    }
    a.nnz[item] = out;
    return;
  }
  for (uint32_t i = 1; i < m; ++i) {
    const uint32_t x = idx[i];
    uint32_t j = i;
    while (j > 0 && idx[j - 1] > x) { idx[j] = idx[j - 1]; --j; }
    idx[j] = x;
  }
  uint32_t out = 0, run = 1;
  for (uint32_t i = 1; i <= m; ++i) {
    if (i < m && idx[i] == idx[i - 1]) { ++run; continue; }
    idx[out] = idx[i - 1];
    cnt[out] = run;
    ++out;
    run = 1;
  }
  a.nnz[item] = out;
}

// one CTA per item with more draws than that: shared-memory counters, ordered emission
__global__ void __launch_bounds__(256) dedup_big_kernel(const DedupArgs a) {
  extern __shared__ uint32_t dd_cnt[];
  __shared__ uint32_t s_scan[256];
  const uint32_t N = 1u << a.b, n_big = *a.big_count;
  for (uint32_t k = blockIdx.x; k < n_big; k += gridDim.x) {
    const uint32_t item = a.big_list[k];
    const uint32_t m = a.nnz[item];
    uint32_t* idx = a.slot_index + a.slot_off[item];
    uint32_t* cnt = a.slot_count + a.slot_off[item];
    for (uint32_t c = threadIdx.x; c < N; c += 256) dd_cnt[c] = 0;
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < m; i += 256) atomicAdd(&dd_cnt[idx[i]], 1u);
    __syncthreads();
    // thread owns the consecutive outcomes [t * per, t * per + per)
    const uint32_t per = (N + 255) / 256, c0 = threadIdx.x * per;
    uint32_t mine = 0;
    for (uint32_t c = c0; c < min(N, c0 + per); ++c) mine += dd_cnt[c] != 0;
    s_scan[threadIdx.x] = mine;
    __syncthreads();
    for (int s = 1; s < 256; s <<= 1) {
      const uint32_t o = threadIdx.x >= (unsigned)s ? s_scan[threadIdx.x - s] : 0u;
      __syncthreads();
      s_scan[threadIdx.x] += o;
      __syncthreads();
    }
    uint32_t posn = s_scan[threadIdx.x] - mine;
    for (uint32_t c = c0; c < min(N, c0 + per); ++c)
      if (dd_cnt[c]) { idx[posn] = c; cnt[posn] = dd_cnt[c]; ++posn; }
    if (threadIdx.x == 255) a.nnz[item] = s_scan[255];
    __syncthreads();
  }
}

}  // namespace ptsbe
