// Batched stored-path contraction executor (north-star subsystem 2).
//
// One launch runs ONE compiled pass program (see include/ptsbe_b200.h) for a
// batch of work items (error set x measured prefix).  A work item is handled
// by a group of GS lanes (GS = 8, 16 or 32: 4, 2 or 1 items per warp, all
// running the same step list in lockstep) or by one CTA; every intermediate
// tensor of the path lives in that group's shared-memory arena, so the only
// HBM traffic of a work item is its Kraus-index row, its prefix words, the
// (L1/L2-resident) program tables and operand pool, records of earlier passes
// and the final record.  Buffers that the compiler could not fit on chip are
// placed in a per-group global spill arena.
//
// Replaces, per work item: merge_errors (engine.py:284-313, as a table
// gather), marginal_network (engine.py:361-407, static operand table),
// execute_path/contract_pair (tensor.py:190-268) and the epilogue of
// _contract_marginal (engine.py:442-450).
#pragma once
#include "common.cuh"
#include "project_tc.cuh"  // tcgen05 / mbarrier PTX wrappers, TF32 split

namespace ptsbe {

constexpr int STEP_WORDS = 20;
constexpr uint32_t MEMO_NONE = 0xFFFFu;
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

enum ExecMode { EXEC_HOIST = 0, EXEC_MARGINAL = 1, EXEC_RAW = 2, EXEC_VECTOR = 3, EXEC_MEMO_BUILD = 4 };

// shared memory of the variant-0 memo bookkeeping: dirty + run bitmaps, the compacted list of
// steps to run (u16) and its length
__host__ __device__ inline uint32_t memo_words(uint32_t n_steps) { return (n_steps + 31) / 32; }
__host__ __device__ inline uint32_t memo_smem_bytes(uint32_t n_steps) {
  return (2 * memo_words(n_steps) * 4 + n_steps * 2 + 16 + 15) & ~15u;
}

struct ExecArgs {
  const uint32_t* leaves;
  const uint32_t* steps;
  const uint32_t* tables;
  const void* pool;
  const uint8_t* kraus;  // [sets][g]
  const LevelDev* levels;
  void* spill;   // [resident groups][arena_spill]
  void* out;     // HOIST: records [level n][out_elems] ; MARGINAL: real probs [items][out_elems]
                 // RAW: complex [items][out_elems]
                 // VECTOR: complex, TRANSPOSED [out_elems][vec_stride] (column = item of this launch)
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
  uint32_t vec_stride;  // VECTOR: row pitch (items, padded) of the transposed output
  uint32_t vec_row;     // VECTOR: non-zero -> one row of vec_row elements per item instead (descent.cuh)
  // variant-0 memo (class-0 programs run one CTA per error set)
  void* memo;                // [memo_elems] value of every step with Kraus index 0 at every site
  const uint32_t* memo_ptr;  // [n_memo_sites + 2] CSR: steps depending on site s; last row: always-run
  const uint32_t* memo_idx;
  uint32_t n_memo_sites;
  // CTA-per-item programs: step descriptors staged in shared memory (the step loop is a chain
  // of dependent loads otherwise: descriptor -> table -> operand)
  uint32_t desc_off;   // byte offset of the staging area from the dynamic shared-memory base
  uint32_t desc_cap;   // steps it holds (0: none)
  uint32_t n_leaves, n_table_words;  // STAGED: the whole program image goes to the staging area
  uint32_t tile_min;   // TILED: 4 x 4 register tiles for steps with at least this many of them, 2 x 2 below
  uint32_t tc_off;     // TC: byte offset of the tensor-core tiles (TCS_BYTES) from the dynamic shared-memory base
};

constexpr uint32_t DESC_CAP = 192;  // staged step descriptors per CTA (x 80 bytes)

__device__ __forceinline__ void prefetch_l1(const void* p) {
  asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}

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

// program words (steps, leaves, gather tables): read-only global memory, or -- STAGED -- the copy a CTA
// keeps in shared memory (generic pointer, so no ld.global.nc)
template <bool STAGED>
__device__ __forceinline__ uint32_t ldt(const uint32_t* p) { return STAGED ? *p : __ldg(p); }
template <bool STAGED>
__device__ __forceinline__ uint4 ldt4(const uint4* p) { return STAGED ? *p : __ldg(p); }

struct StepTables {
  const uint32_t *loA, *loB, *hiA, *hiB, *kA, *kB;
  uint32_t out_n, lo_n, hi_n;
  uint32_t conj;  // bit 0: use conj(A), bit 1: use conj(B) -- operand is the conjugate twin of a computed node
};

template <typename C>
__device__ __forceinline__ C ld_conj(const C* p, bool flip) {
  C v = *p;
  if (flip) v.y = -v.y;
  return v;
}

// inner product over KN shared labels with the k-offsets held in registers
template <typename C, int KN, bool STAGED = false>
__device__ __forceinline__ void step_fixed_k(const C* __restrict__ A, const C* __restrict__ B, C* O,
                                             size_t o_stride, const StepTables& t, int tid,
                                             int gsize, bool store) {
  uint32_t ka[KN], kb[KN];
#pragma unroll
  for (int k = 0; k < KN; ++k) { ka[k] = ldt<STAGED>(t.kA + k); kb[k] = ldt<STAGED>(t.kB + k); }
  const int sh = 31 - __clz(t.lo_n);
  const bool pow2 = (t.lo_n & (t.lo_n - 1)) == 0;
  const bool fa = t.conj & 1, fb = t.conj & 2;
  for (uint32_t c = tid; c < t.out_n; c += gsize) {
    uint32_t cl, ch;
    if (pow2) { cl = c & (t.lo_n - 1); ch = c >> sh; }
    else { ch = c / t.lo_n; cl = c - ch * t.lo_n; }
    uint32_t a0 = ldt<STAGED>(t.loA + cl), b0 = ldt<STAGED>(t.loB + cl);
    if (t.hi_n > 1) { a0 += ldt<STAGED>(t.hiA + ch); b0 += ldt<STAGED>(t.hiB + ch); }
    C acc; acc.x = 0; acc.y = 0;
#pragma unroll
    for (int k = 0; k < KN; ++k) cmac(acc, ld_conj(A + a0 + ka[k], fa), ld_conj(B + b0 + kb[k], fb));
    if (store) O[(size_t)c * o_stride] = acc;
  }
}

// Separable (GEMM) form of a large step, one CTA: out[oA[a] + oB[b]] = sum_k A[aOff[a] + kA[k]] *
// B[bOff[b] + kB[k]].  A thread owns a TM x TN register tile, so each loaded operand element
// feeds TN (or TM) multiply-adds instead of one; neighbouring threads share the tile row (their A
// loads are shared-memory broadcasts).  The k order of every output is that of the plain form,
// so the values are bit-identical.
template <typename C, bool FA, bool FB, int TM = 4, int TN = 4>
__device__ __forceinline__ void tiled_step(const C* __restrict__ A, const C* __restrict__ B, C* O,
                                           const uint32_t* __restrict__ g, uint32_t M, uint32_t N,
                                           const uint32_t* __restrict__ kA, const uint32_t* __restrict__ kB,
                                           uint32_t kn, int tid, int nthreads, bool store) {
  const uint32_t *aOff = g, *bOff = g + M, *oA = g + M + N, *oB = g + 2 * M + N;
  const uint32_t tn = (N + TN - 1) / TN, tm = (M + TM - 1) / TM;
  for (uint32_t tile = tid; tile < tm * tn; tile += nthreads) {
    const uint32_t ta = tile / tn, tb = tile - ta * tn;
    uint32_t ao[TM], bo[TN];
#pragma unroll
    for (int i = 0; i < TM; ++i) ao[i] = __ldg(aOff + min(ta * TM + i, M - 1));
#pragma unroll
    for (int j = 0; j < TN; ++j) bo[j] = __ldg(bOff + min(tb * TN + j, N - 1));
    C acc[TM][TN];
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
      for (int j = 0; j < TN; ++j) { acc[i][j].x = 0; acc[i][j].y = 0; }
    for (uint32_t k = 0; k < kn; ++k) {
      const uint32_t ka = __ldg(kA + k), kb = __ldg(kB + k);
      C av[TM], bv[TN];
#pragma unroll
      for (int i = 0; i < TM; ++i) { av[i] = A[ao[i] + ka]; if (FA) av[i].y = -av[i].y; }
#pragma unroll
      for (int j = 0; j < TN; ++j) { bv[j] = B[bo[j] + kb]; if (FB) bv[j].y = -bv[j].y; }
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) cmac(acc[i][j], av[i], bv[j]);
    }
    if (store) {
#pragma unroll
      for (int i = 0; i < TM; ++i) {
        if (ta * TM + i >= M) break;
        const uint32_t oa = __ldg(oA + ta * TM + i);
#pragma unroll
        for (int j = 0; j < TN; ++j)
          if (tb * TN + j < N) O[oa + __ldg(oB + tb * TN + j)] = acc[i][j];
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Large separable steps on the 5th-generation tensor cores (complex64, CTA-per-item programs).
//
// The same step as tiled_step -- out[oA[a] + oB[b]] = sum_k A[aOff[a] + kA[k]] * B[bOff[b] + kB[k]], the
// np.tensordot of reference tensor.py:190-216 -- written as a REAL product D[M x 2N] = A'[M x 2K] B'[2N x 2K]^T:
//     A'[a][2k] = Re A, A'[a][2k+1] = Im A;   B'[2b][2k] = Re B, B'[2b][2k+1] = -Im B  (real part of out),
//                                             B'[2b+1][2k] = Im B, B'[2b+1][2k+1] = Re B (imaginary part),
// so a row of D is the row of complex outputs, interleaved.  Operands are gather-addressed per error set, so
// there is no TMA: all 256 threads gather, split x = hi + lo on the TF32 mantissa (project_tc.cuh) and store
// 16-byte chunks into K-major tiles with the 128-byte swizzle the UMMA descriptors of project_tc.cuh expect
// (chunk j of row r at (r / 8) * 1024 + (r % 8) * 128 + ((j ^ (r % 8)) * 16)); one thread issues
// tcgen05.mma.kind::tf32 (M = 128, N' <= 64, K = 8) for hi*hi + hi*lo, the A tile is overwritten with its lo
// part for lo*hi (one A buffer: shared memory decides how many CTAs stay resident), the accumulator lives in
// TMEM and comes back with tcgen05.ld, thread = output row.  3 x TF32 keeps ~2^-21 per product.
constexpr uint32_t TCS_A_BYTES = 128 * 128;      // 128 rows x 32 floats
constexpr uint32_t TCS_NP = 64;                  // real output columns per pass (32 complex)
constexpr uint32_t TCS_B_BYTES = TCS_NP * 128;
constexpr uint32_t TCS_BYTES = TCS_A_BYTES + 2 * TCS_B_BYTES + 1024 /* alignment */ + 64 /* mbarrier, TMEM slot */;
constexpr uint32_t TCS_TMEM_COLS = 64;

__device__ __forceinline__ void tc_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr)
      : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

struct TcStepCtx {
  unsigned char* tiles;   // 1024-byte aligned: A | B_hi | B_lo
  uint32_t bar;           // shared-memory address of the mbarrier (count 1)
  uint32_t tmem;          // TMEM base of this CTA's TCS_TMEM_COLS columns
  uint32_t phase;         // parity of the next barrier completion (uniform over the CTA)
};

__device__ __forceinline__ uint32_t tcs_swz(uint32_t r, uint32_t j) {
  return (r >> 3) * 1024u + (r & 7u) * 128u + ((j ^ (r & 7u)) << 4);
}

// CTA-wide; every thread of the 256 must call it (barriers inside)
__device__ __forceinline__ void tc_step(TcStepCtx& cx, const float2* __restrict__ A, const float2* __restrict__ B,
                                        float2* O, const uint32_t* __restrict__ g, uint32_t M, uint32_t N,
                                        const uint32_t* __restrict__ kA, const uint32_t* __restrict__ kB, uint32_t kn,
                                        bool fa, bool fb, int tid, bool store) {
  const uint32_t *aOff = g, *bOff = g + M, *oA = g + M + N, *oB = g + 2 * M + N;
  unsigned char* a_tile = cx.tiles;
  unsigned char* bh_tile = cx.tiles + TCS_A_BYTES;
  unsigned char* bl_tile = bh_tile + TCS_B_BYTES;
  const uint32_t a_s = tc_smem(a_tile), bh_s = tc_smem(bh_tile), bl_s = tc_smem(bl_tile);
  const uint32_t kblocks = (kn + 15) / 16;
  const int warp = tid >> 5, lane = tid & 31;
  for (uint32_t m0 = 0; m0 < M; m0 += 128) {
    for (uint32_t n0 = 0; n0 < N; n0 += TCS_NP / 2) {
      const uint32_t np = min(TCS_NP / 2, N - n0);                 // complex columns of this pass
      const uint32_t nprime = max(16u, 2u * ((np + 7u) & ~7u));    // UMMA N: multiple of 16
      const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((nprime >> 3) << 17) | ((128u >> 4) << 24);
      for (uint32_t kb = 0; kb < kblocks; ++kb) {
        // ---- gather + split: A (hi to the tile, lo kept in registers), B (hi and lo tiles) ----
        float4 alo[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const uint32_t idx = tid + 256 * i, r = idx >> 3, j = idx & 7, k0 = kb * 16 + 2 * j;
          const uint32_t row = m0 + r;
          float2 x0 = make_float2(0.f, 0.f), x1 = x0;
          if (row < M) {
            const uint32_t ao = __ldg(aOff + row);
            if (k0 < kn) x0 = A[ao + __ldg(kA + k0)];
            if (k0 + 1 < kn) x1 = A[ao + __ldg(kA + k0 + 1)];
          }
          if (fa) { x0.y = -x0.y; x1.y = -x1.y; }
          float4 h, l;
          tc_split(x0.x, h.x, l.x); tc_split(x0.y, h.y, l.y); tc_split(x1.x, h.z, l.z); tc_split(x1.y, h.w, l.w);
          *reinterpret_cast<float4*>(a_tile + tcs_swz(r, j)) = h;
          alo[i] = l;
        }
        for (uint32_t idx = tid; idx < nprime * 8; idx += 256) {
          const uint32_t r = idx >> 3, j = idx & 7, k0 = kb * 16 + 2 * j, b = r >> 1;
          float2 y0 = make_float2(0.f, 0.f), y1 = y0;
          if (b < np) {
            const uint32_t bo = __ldg(bOff + n0 + b);
            if (k0 < kn) y0 = B[bo + __ldg(kB + k0)];
            if (k0 + 1 < kn) y1 = B[bo + __ldg(kB + k0 + 1)];
          }
          if (fb) { y0.y = -y0.y; y1.y = -y1.y; }
          float4 v;
          if (r & 1u) v = make_float4(y0.y, y0.x, y1.y, y1.x);      // imaginary part of the output
          else v = make_float4(y0.x, -y0.y, y1.x, -y1.y);           // real part
          float4 h, l;
          tc_split(v.x, h.x, l.x); tc_split(v.y, h.y, l.y); tc_split(v.z, h.z, l.z); tc_split(v.w, h.w, l.w);
          *reinterpret_cast<float4*>(bh_tile + tcs_swz(r, j)) = h;
          *reinterpret_cast<float4*>(bl_tile + tcs_swz(r, j)) = l;
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> tensor-core reads
        __syncthreads();
        const uint32_t ksteps = min(4u, (2u * kn - kb * 32u + 7u) / 8u);
        if (tid == 0) {
          tc_fence_after();
          for (uint32_t k = 0; k < ksteps; ++k) {
            tc_mma_tf32(cx.tmem, tc_desc(a_s + k * 32), tc_desc(bh_s + k * 32), idesc, (kb | k) ? 1u : 0u);
            tc_mma_tf32(cx.tmem, tc_desc(a_s + k * 32), tc_desc(bl_s + k * 32), idesc, 1u);
          }
          tc_commit(cx.bar);
        }
        mbar_wait(cx.bar, cx.phase);
        cx.phase ^= 1u;
        // ---- A_lo over the same buffer, times B_hi ----
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const uint32_t idx = tid + 256 * i;
          *reinterpret_cast<float4*>(a_tile + tcs_swz(idx >> 3, idx & 7)) = alo[i];
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        if (tid == 0) {
          tc_fence_after();
          for (uint32_t k = 0; k < ksteps; ++k)
            tc_mma_tf32(cx.tmem, tc_desc(a_s + k * 32), tc_desc(bh_s + k * 32), idesc, 1u);
          tc_commit(cx.bar);
        }
        mbar_wait(cx.bar, cx.phase);
        cx.phase ^= 1u;
      }
      // ---- accumulator -> registers -> out: thread = row (TMEM lane), warps 0-3 = lane quadrants ----
      tc_fence_after();
      if (warp < 4) {
        const uint32_t row = m0 + 32 * warp + lane;
        const uint32_t oa = row < M ? __ldg(oA + row) : 0u;
        for (uint32_t c0 = 0; c0 < nprime; c0 += 16) {
          uint32_t r[16];
          tc_ld16(cx.tmem + ((32u * warp) << 16) + c0, r);
          if (store && row < M) {
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              const uint32_t b = c0 / 2 + q;
              if (b < np) O[oa + __ldg(oB + n0 + b)] = make_float2(__uint_as_float(r[2 * q]), __uint_as_float(r[2 * q + 1]));
            }
          }
        }
      }
      tc_fence_before();
      __syncthreads();  // accumulator and tiles free for the next pass; outputs visible to the CTA
    }
  }
}

// GS > 0 : sub-warp mapping, GS lanes per item, 32 / GS items per warp, __syncwarp between steps
// GS == 0: one CTA per item, __syncthreads between steps
// MEMO    : (GS == 0 only) class-0 program with a variant-0 memo.  UPV leaves every tensor of the
//           template untouched except at the sites where this error set realised an operator, so
//           only the steps above those sites are re-executed; everything else is read from the
//           memo that was computed once per plan.
// TILED   : (with MEMO) large steps run in their separable form with register tiles; costs
//           registers, so only programs dominated by such steps use it
// STAGED  : (GS > 0 only) the program image -- steps, leaves, gather tables -- is copied to shared memory
//           once per CTA.  A step of a lane-group program is a chain of dependent reads (descriptor ->
//           tables -> leaf row -> Kraus index -> operand); from global memory that chain costs ~2000
//           cycles per step, which is all there is when a batch holds few error sets (cfg5 at E <= 10^4).
// TC      : (GS == 0, TILED, complex64) large separable steps on the tensor cores (tc_step above)
template <typename R, int GS, bool MEMO, bool TILED = false, bool STAGED = false, bool TC = false>
__global__ void __launch_bounds__(256, TILED ? (TC ? 2 : 3) : 5) exec_kernel(const ExecArgs a) {
  using C = typename CxT<R>::type;
  constexpr bool WARP = GS > 0;
  constexpr int GSD = GS > 0 ? GS : 1;
  extern __shared__ __align__(16) unsigned char smem_raw[];

  const int gsize = WARP ? GS : blockDim.x;
  const int tid = WARP ? (threadIdx.x & (GSD - 1)) : threadIdx.x;
  const int group_in_block = WARP ? (threadIdx.x / GSD) : 0;
  const int groups_per_block = WARP ? (blockDim.x / GSD) : 1;
  const uint32_t group_global = blockIdx.x * groups_per_block + group_in_block;
  const uint32_t n_groups = gridDim.x * groups_per_block;

  unsigned char* my = smem_raw + (size_t)group_in_block * a.item_bytes;
  C* arena = reinterpret_cast<C*>(my);
  uint64_t* pfx = reinterpret_cast<uint64_t*>(my + (size_t)a.arena_fast * sizeof(C));
  uint32_t* anc = reinterpret_cast<uint32_t*>(pfx + a.words);
  C* spill = reinterpret_cast<C*>(a.spill) + (size_t)group_global * a.arena_spill;
  const C* pool = reinterpret_cast<const C*>(a.pool);
  // scratch for CTA-wide reductions (marginal epilogue), placed after the groups
  double* red = reinterpret_cast<double*>(smem_raw + (size_t)groups_per_block * a.item_bytes);
  // memo bookkeeping, after the reduction scratch
  const uint32_t mw = MEMO ? memo_words(a.n_steps) : 0;
  uint32_t* dirty = reinterpret_cast<uint32_t*>(smem_raw + (size_t)groups_per_block * a.item_bytes + 1024);
  uint32_t* runb = dirty + mw;
  uint32_t* n_run_s = runb + mw;
  uint16_t* run_list = reinterpret_cast<uint16_t*>(n_run_s + 4);
  const C* memo = reinterpret_cast<const C*>(a.memo);
  const bool build = MEMO && a.mode == EXEC_MEMO_BUILD;
  uint32_t* desc_s = reinterpret_cast<uint32_t*>(smem_raw + a.desc_off);
  const C** pre_s = reinterpret_cast<const C**>(smem_raw + a.desc_off + (size_t)a.desc_cap * STEP_WORDS * 4);
  uint32_t n_staged = 0;
  const uint32_t* steps_p = a.steps;
  const uint32_t* leaves_p = a.leaves;
  const uint32_t* tables_p = a.tables;
  if constexpr (STAGED) {
    uint32_t* img = reinterpret_cast<uint32_t*>(smem_raw + a.desc_off);
    const uint32_t ns = a.n_steps * STEP_WORDS, nl = a.n_leaves * LEAF_WORDS, nt = a.n_table_words;
    for (uint32_t i = threadIdx.x; i < ns; i += blockDim.x) img[i] = __ldg(a.steps + i);
    for (uint32_t i = threadIdx.x; i < nl; i += blockDim.x) img[ns + i] = __ldg(a.leaves + i);
    for (uint32_t i = threadIdx.x; i < nt; i += blockDim.x) img[ns + nl + i] = __ldg(a.tables + i);
    __syncthreads();
    steps_p = img;
    leaves_p = img + ns;
    tables_p = img + ns + nl;
  }
  if (!WARP && !MEMO && a.desc_cap) {
    // same step list for every item: staged once
    n_staged = min(a.n_steps, a.desc_cap);
    for (uint32_t i = threadIdx.x; i < n_staged * STEP_WORDS; i += blockDim.x) desc_s[i] = __ldg(a.steps + i);
    __syncthreads();
  }

  TcStepCtx tcx;
  tcx.tiles = nullptr; tcx.bar = 0; tcx.tmem = 0; tcx.phase = 0;
  if constexpr (TC) {
    unsigned char* raw = smem_raw + a.tc_off;
    tcx.tiles = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bar = reinterpret_cast<uint64_t*>(tcx.tiles + TCS_A_BYTES + 2 * TCS_B_BYTES);
    uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 1);
    tcx.bar = tc_smem(bar);
    if (threadIdx.x == 0) {
      mbar_init(tcx.bar, 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (threadIdx.x < 32) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tc_smem(slot)),
                   "r"(TCS_TMEM_COLS)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    tcx.tmem = *slot;
  }

  auto group_sync = [&]() {
    if (WARP) __syncwarp(); else __syncthreads();
  };

  // every group of a warp runs the same number of rounds (lockstep __syncwarp): groups past
  // the end redo the last item with their stores to global memory masked off
  const uint32_t rounds = (a.n_items + n_groups - 1) / n_groups;
  for (uint32_t r = 0; r < rounds; ++r) {
    uint32_t it = r * n_groups + group_global;
    const bool live = it < a.n_items;
    if (!live) it = a.n_items - 1;
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
    const uint8_t* sel = a.kraus + (size_t)e * a.g;  // Kraus-index row: shared by all items of the error set (L1/L2)
    if constexpr (MEMO) {
      for (uint32_t w = tid; w < 2 * mw; w += gsize) dirty[w] = build ? (w >= mw ? 0xffffffffu : 0u) : 0u;
      __syncthreads();
      if (!build) {
        // mark the steps above every site that carries an operator, and the always-run steps
        for (uint32_t site = tid; site <= a.n_memo_sites; site += gsize) {
          const bool always = site == a.n_memo_sites;
          if (!always && __ldg(sel + site) == 0) continue;
          uint32_t* bits = always ? runb : dirty;
          const uint32_t k1 = __ldg(a.memo_ptr + site + 1);
          for (uint32_t k = __ldg(a.memo_ptr + site); k < k1; ++k) {
            const uint32_t idx = __ldg(a.memo_idx + k);
            atomicOr(bits + (idx >> 5), 1u << (idx & 31));
          }
        }
        __syncthreads();
      }
      // compact (dirty | always) into an ordered list of step indices
      if (threadIdx.x < 32) {
        uint32_t base = 0;
        for (uint32_t w0 = 0; w0 < mw; w0 += 32) {
          const uint32_t w = w0 + threadIdx.x;
          uint32_t word = w < mw ? (dirty[w] | runb[w]) : 0u;
          if (w == mw - 1 && (a.n_steps & 31)) word &= (1u << (a.n_steps & 31)) - 1u;
          const uint32_t cnt = __popc(word);
          uint32_t incl = cnt;
#pragma unroll
          for (int d = 1; d < 32; d <<= 1) {
            const uint32_t o = __shfl_up_sync(0xffffffffu, incl, d);
            if ((int)threadIdx.x >= d) incl += o;
          }
          uint32_t pos = base + incl - cnt;
          while (word) {
            const uint32_t bit = __ffs(word) - 1;
            run_list[pos++] = (uint16_t)(w * 32 + bit);
            word &= word - 1;
          }
          base += __shfl_sync(0xffffffffu, incl, 31);
        }
        if (threadIdx.x == 0) *n_run_s = base;
      }
    }
    group_sync();
    const uint32_t n_run = MEMO ? *n_run_s : a.n_steps;
    if constexpr (MEMO) {
      // descriptors of the steps this item runs: one round of parallel loads instead of one
      // dependent load chain per step
      n_staged = min(n_run, a.desc_cap);
      for (uint32_t i = threadIdx.x; i < n_staged * STEP_WORDS; i += blockDim.x) {
        const uint32_t si = i / STEP_WORDS, w = i - si * STEP_WORDS;
        desc_s[i] = __ldg(a.steps + (size_t)run_list[si] * STEP_WORDS + w);
      }
      __syncthreads();
      // leaf operands of the staged steps resolved in parallel (leaf row -> Kraus index -> pool
      // address is two dependent loads that would otherwise sit in front of every small step)
      for (uint32_t i = threadIdx.x; i < n_staged * 2; i += blockDim.x) {
        const uint32_t* dsc = desc_s + (size_t)(i >> 1) * STEP_WORDS + (i & 1) * 2;
        const C* ptr = nullptr;
        if (dsc[0] == 1) {
          const uint4 lf = __ldg(reinterpret_cast<const uint4*>(a.leaves) + dsc[1]);
          if (lf.z < 2) ptr = pool + lf.x + (size_t)(lf.z == 1 ? __ldg(sel + lf.w) : 0u) * lf.y;
        }
        pre_s[i] = ptr;
      }
      __syncthreads();
    }

    // measured bit selected by a prefix-projector leaf (slice steps read the bit, not the vector)
    auto leaf_bit = [&](uint32_t ref) -> uint32_t {
      const uint4 lf = ldt4<STAGED>(reinterpret_cast<const uint4*>(leaves_p) + ref);
      return (uint32_t)((pfx[lf.w >> 6] >> (63 - (lf.w & 63))) & 1ull);
    };
    auto resolve = [&](uint32_t kind, uint32_t ref) -> const C* {
      if (kind == 0) return ref < a.arena_fast ? arena + ref : spill + (ref - a.arena_fast);
      if (kind == 1) {
        const uint4 lf = ldt4<STAGED>(reinterpret_cast<const uint4*>(leaves_p) + ref);
        uint32_t v = 0;
        if (lf.z == 1) v = __ldg(sel + lf.w);
        else if (lf.z == 2) v = (uint32_t)((pfx[lf.w >> 6] >> (63 - (lf.w & 63))) & 1ull);
        return pool + lf.x + (size_t)v * lf.y;
      }
      const uint32_t l = kind - 1;  // pass p = kind-2 iterates level p+1
      const LevelDev el = a.levels[l];
      return reinterpret_cast<const C*>(el.ext) + (size_t)anc[l] * el.ext_rec + ref;
    };

    // ---- replay the stored path ----
    for (uint32_t si = 0; si < n_run; ++si) {
      const uint32_t s = MEMO ? run_list[si] : si;
      // s0 = {a_kind, a_ref, b_kind, b_ref}, s1 = {o_kind, o_ref, out_n, k_n}, s2 = {lo_n, hi_n, tab_off, flags}
      // s3 = {a_memo, b_memo, a_prod | b_prod << 16, own_memo}, s4 = {gemm_off, gemm_m, gemm_n, -}
      uint4 s0, s1, s2, s3, s4;
      s3 = make_uint4(0, 0, 0, 0); s4 = s3;
      if (si < n_staged) {
        const uint4* st4 = reinterpret_cast<const uint4*>(desc_s + (size_t)si * STEP_WORDS);
        s0 = st4[0]; s1 = st4[1]; s2 = st4[2];
        if (MEMO) s3 = st4[3];
        if (TILED) s4 = st4[4];
        if (threadIdx.x == 0 && si + 1 < n_staged) {
          // warm L1 with the next step's gather tables while this step computes
          const uint32_t* nd = desc_s + (size_t)(si + 1) * STEP_WORDS;
          prefetch_l1(a.tables + nd[10]);
          if (TILED && nd[17]) prefetch_l1(a.tables + nd[16]);
        }
      } else {
        const uint4* st4 = reinterpret_cast<const uint4*>(steps_p + (size_t)s * STEP_WORDS);
        s0 = ldt4<STAGED>(st4); s1 = ldt4<STAGED>(st4 + 1); s2 = ldt4<STAGED>(st4 + 2);
        if (MEMO) s3 = ldt4<STAGED>(st4 + 3);
        if (TILED) s4 = ldt4<STAGED>(st4 + 4);
      }
      const bool slice = (s2.w & 4u) != 0;
      const C* A = nullptr;
      const C* B = nullptr;
      if (MEMO && si < n_staged) { A = pre_s[2 * si]; B = pre_s[2 * si + 1]; }
      if (!A) A = resolve(s0.x, s0.y);
      if (!B && !slice) B = resolve(s0.z, s0.w);
      C* O;
      size_t o_stride = 1;
      bool store = true;
      bool copy_memo = false;
      uint32_t own_memo = 0;
      if (MEMO) {
        const uint32_t pa = s3.z & 0xFFFFu, pb = s3.z >> 16;
        if (pa != MEMO_NONE && !((dirty[pa >> 5] >> (pa & 31)) & 1u)) A = memo + s3.x;
        if (pb != MEMO_NONE && !((dirty[pb >> 5] >> (pb & 31)) & 1u)) B = memo + s3.y;
        own_memo = s3.w;
        // an always-run step whose inputs are clean: its value is the memo's
        copy_memo = !build && !((dirty[s >> 5] >> (s & 31)) & 1u);
      }
      if (build) {
        O = const_cast<C*>(memo) + own_memo;
      } else if (s1.x == 0) {
        O = s1.y < a.arena_fast ? arena + s1.y : spill + (s1.y - a.arena_fast);
      } else if (a.mode == EXEC_VECTOR) {
        if (a.vec_row) {
          O = reinterpret_cast<C*>(a.out) + (size_t)it * a.vec_row + s1.y;
        } else {
          O = reinterpret_cast<C*>(a.out) + (size_t)s1.y * a.vec_stride + it;
          o_stride = a.vec_stride;
        }
        store = live;
      } else {
        O = reinterpret_cast<C*>(a.out) + (size_t)item * a.out_elems + s1.y;
        store = live;
      }
      StepTables t;
      t.out_n = s1.z;
      t.lo_n = s2.x;
      t.hi_n = s2.y;
      t.conj = s2.w;
      const uint32_t kn = s1.w;
      t.loA = tables_p + s2.z;
      t.loB = t.loA + t.lo_n;
      t.hiA = t.loB + t.lo_n;
      t.hiB = t.hiA + t.hi_n;
      t.kA = t.hiB + t.hi_n;
      t.kB = t.kA + kn;
      if (t.conj & 8u) {
        // slice views: the operand is T[.., bit(q), ..] of a stored tensor -- add bit * stride
        // per sliced leg to the base instead of materialising the slice
        const uint32_t* dt = t.kB + kn;
        const uint32_t na = ldt<STAGED>(dt);
        for (uint32_t i = 0; i < na; ++i) {
          const uint32_t q = ldt<STAGED>(dt + 1 + 2 * i);
          if ((pfx[q >> 6] >> (63 - (q & 63))) & 1ull) A += ldt<STAGED>(dt + 2 + 2 * i);
        }
        dt += 1 + 2 * na;
        const uint32_t nb = ldt<STAGED>(dt);
        for (uint32_t i = 0; i < nb; ++i) {
          const uint32_t q = ldt<STAGED>(dt + 1 + 2 * i);
          if ((pfx[q >> 6] >> (63 - (q & 63))) & 1ull) B += ldt<STAGED>(dt + 2 + 2 * i);
        }
      }
      if (MEMO && copy_memo) {
        const C* src = memo + own_memo;
        for (uint32_t c = tid; c < t.out_n; c += gsize)
          if (store) O[(size_t)c * o_stride] = src[c];
      } else if (TC && TILED && o_stride == 1 && s4.y >= 64 && s4.z >= 4 && kn >= 4 &&
                 (uint64_t)s4.y * s4.z * kn >= 16384) {
        // large step on the tensor cores
        if constexpr (TC)
          tc_step(tcx, reinterpret_cast<const float2*>(A), reinterpret_cast<const float2*>(B),
                  reinterpret_cast<float2*>(O), a.tables + s4.x, s4.y, s4.z, t.kA, t.kB, kn, (t.conj & 1u) != 0,
                  (t.conj & 2u) != 0, tid, store);
      } else if (TILED && o_stride == 1 && s4.y != 0) {
        // large step: separable form with register tiles
        const uint32_t* gt = a.tables + s4.x;
        // 4 x 4 tiles when they keep most of the CTA busy; steps of a few hundred outputs (2-32 k MACs, K up
        // to 64) would otherwise run on one or two warps while the rest waits at the barrier: 2 x 2 tiles
        if (((s4.y + 3) / 4) * ((s4.z + 3) / 4) >= a.tile_min) {
          switch (t.conj & 3u) {
            case 0: tiled_step<C, false, false>(A, B, O, gt, s4.y, s4.z, t.kA, t.kB, kn, tid, gsize, store); break;
            case 1: tiled_step<C, true, false>(A, B, O, gt, s4.y, s4.z, t.kA, t.kB, kn, tid, gsize, store); break;
            case 2: tiled_step<C, false, true>(A, B, O, gt, s4.y, s4.z, t.kA, t.kB, kn, tid, gsize, store); break;
            default: tiled_step<C, true, true>(A, B, O, gt, s4.y, s4.z, t.kA, t.kB, kn, tid, gsize, store); break;
          }
        } else {
          switch (t.conj & 3u) {
            case 0: tiled_step<C, false, false, 2, 2>(A, B, O, gt, s4.y, s4.z, t.kA, t.kB, kn, tid, gsize, store); break;
            case 1: tiled_step<C, true, false, 2, 2>(A, B, O, gt, s4.y, s4.z, t.kA, t.kB, kn, tid, gsize, store); break;
            case 2: tiled_step<C, false, true, 2, 2>(A, B, O, gt, s4.y, s4.z, t.kA, t.kB, kn, tid, gsize, store); break;
            default: tiled_step<C, true, true, 2, 2>(A, B, O, gt, s4.y, s4.z, t.kA, t.kB, kn, tid, gsize, store); break;
          }
        }
      } else if (slice) {
        // B is the basis vector e_x of a measured bit, contracted over its only label:
        // out[c] = A[a0(c) + kA[x]] -- a gather, no multiply-adds
        const uint32_t k0 = ldt<STAGED>(t.kA), k1 = ldt<STAGED>(t.kA + 1);
        const uint32_t off = leaf_bit(s0.w) ? k1 : k0;
        const bool pow2 = (t.lo_n & (t.lo_n - 1)) == 0;
        const int sh = 31 - __clz(t.lo_n);
        const bool fa = t.conj & 1;
        for (uint32_t c = tid; c < t.out_n; c += gsize) {
          uint32_t cl, ch;
          if (pow2) { cl = c & (t.lo_n - 1); ch = c >> sh; }
          else { ch = c / t.lo_n; cl = c - ch * t.lo_n; }
          uint32_t a0 = ldt<STAGED>(t.loA + cl);
          if (t.hi_n > 1) a0 += ldt<STAGED>(t.hiA + ch);
          const C v = ld_conj(A + a0 + off, fa);
          if (store) O[(size_t)c * o_stride] = v;
        }
      } else
      switch (kn) {
        case 1: step_fixed_k<C, 1, STAGED>(A, B, O, o_stride, t, tid, gsize, store); break;
        case 2: step_fixed_k<C, 2, STAGED>(A, B, O, o_stride, t, tid, gsize, store); break;
        case 4: step_fixed_k<C, 4, STAGED>(A, B, O, o_stride, t, tid, gsize, store); break;
        case 8: step_fixed_k<C, 8, STAGED>(A, B, O, o_stride, t, tid, gsize, store); break;
        default: {
          const bool pow2 = (t.lo_n & (t.lo_n - 1)) == 0;
          const int sh = 31 - __clz(t.lo_n);
          const bool fa = t.conj & 1, fb = t.conj & 2;
          for (uint32_t c = tid; c < t.out_n; c += gsize) {
            uint32_t cl, ch;
            if (pow2) { cl = c & (t.lo_n - 1); ch = c >> sh; }
            else { ch = c / t.lo_n; cl = c - ch * t.lo_n; }
            uint32_t a0 = ldt<STAGED>(t.loA + cl), b0 = ldt<STAGED>(t.loB + cl);
            if (t.hi_n > 1) { a0 += ldt<STAGED>(t.hiA + ch); b0 += ldt<STAGED>(t.hiB + ch); }
            C acc; acc.x = 0; acc.y = 0;
            for (uint32_t k = 0; k < kn; ++k)
              cmac(acc, ld_conj(A + a0 + ldt<STAGED>(t.kA + k), fa), ld_conj(B + b0 + ldt<STAGED>(t.kB + k), fb));
            if (store) O[(size_t)c * o_stride] = acc;
          }
        }
      }
      group_sync();
    }

    // ---- epilogue ----
    if (a.mode == EXEC_MARGINAL || a.mode == EXEC_RAW) {
      const C* res = resolve(a.result_kind, a.result_ref);
      if (a.mode == EXEC_RAW) {
        C* o = reinterpret_cast<C*>(a.out) + (size_t)it * a.out_elems;
        if (live)
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
          if (live) o[c] = v;
        }
        constexpr int RED = WARP ? GSD : 32;
#pragma unroll
        for (int d = RED / 2; d > 0; d >>= 1) {
          mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, d));
          sum += __shfl_xor_sync(0xffffffffu, sum, d);
        }
        if (WARP) {
          if (tid == 0 && live) { a.out_mass[it] = sum; a.out_min[it] = mn; }
        } else {
          const int wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
          if ((threadIdx.x & 31) == 0) { red[2 * wid] = mn; red[2 * wid + 1] = sum; }
          __syncthreads();
          if (threadIdx.x == 0 && live) {
            for (int w = 1; w < nw; ++w) { mn = fmin(mn, red[2 * w]); sum += red[2 * w + 1]; }
            a.out_mass[it] = sum;
            a.out_min[it] = mn;
          }
        }
      }
    }
    group_sync();
  }
  if constexpr (TC) {
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) {
      tc_fence_after();
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tcx.tmem), "r"(TCS_TMEM_COLS) : "memory");
    }
  }
}

}  // namespace ptsbe
