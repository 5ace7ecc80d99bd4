// Dense projection step of a stage (north-star subsystem 2, "the steps that are
// genuinely dense contractions"):
//
//     P[i][c] = Re( sum_d v_i[d] * M_e(i)[d][c] ),   d < D, c < N = 2^b
//
// v_i is the per-work-item vector left by the stored path's per-item steps
// (exec_kernel, EXEC_VECTOR), M_e the record the path's error-set-only part
// produced once per error set (exec_kernel, EXEC_HOIST, pass 0).  Work items
// are sorted by error set, so a tile of TI consecutive items almost always
// shares one M: the product over all items of an error set is a real GEMM
// [items x 2D] x [2D x N] (only the real part of the complex product is
// needed: two FMAs per complex pair instead of four).
//
// This version runs on the FP32 / FP64 FMA pipes: 1e-5 (complex64) and 1e-11
// (complex128) on the marginals rule out single-pass TF32, and a split-
// precision tcgen05 path is listed as next work in DESIGN.md.
//
// Replaces, for those stages, the last np.tensordot of execute_path
// (tensor.py:236-259) plus transpose/real of _contract_marginal
// (engine.py:442-445); clamp/mass/min guards run in the sampler.
#pragma once
#include "common.cuh"
#include "executor.cuh"

namespace ptsbe {

struct ProjectArgs {
  const void* vt;         // [D][v_stride] complex, TRANSPOSED: column = item - first_item
  const void* rec0;       // pass-0 records: [error sets][rec_stride] complex
  const uint32_t* eset;   // [level n] error-set row of every item
  void* out;              // [n_items][N] real, raw (unclamped)
  uint32_t first_item, n_items;
  uint32_t D, N;
  uint32_t v_stride;      // row pitch of vt in elements (multiple of 2)
  uint32_t rec_stride;    // elements per error-set record
  uint32_t m_off;         // offset of M inside the record
};

constexpr int PJ_TI = 64;    // items per tile
constexpr int PJ_TN = 128;   // columns per tile
constexpr int PJ_THREADS = 256;
constexpr int PJ_RI = 4;     // items per thread (consecutive)
constexpr int PJ_RN = 8;     // columns per thread: 4 pairs, pair p at columns 2 * (p * 16 + tn) + {0, 1}

template <typename R> struct ProjK { static constexpr int KC = 16; };   // k-chunk of one ring slot
template <> struct ProjK<double> { static constexpr int KC = 8; };

template <typename R> struct Cx2;  // two complex numbers, one 16/32-byte load
template <> struct Cx2<float> { using type = float4; };
template <> struct Cx2<double> { using type = double4; };

// 16-byte asynchronous global -> shared copy (LDGSTS); src_bytes == 0 zero-fills the slot.
__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc, uint32_t src_bytes) {
  const uint32_t d = (uint32_t)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(gsrc), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// Both operands are k-major (vt[d][item], M[d][c]), so the tiles go to shared memory with
// straight, coalesced, conflict-free 16-byte copies: Vs[KC][TI], Ms[KC][TN].  The copies are
// asynchronous (cp.async) into a two-deep ring, so the loads of k-chunk n+1 (or of the next
// tile) overlap the FMAs of chunk n.  A warp is 2 (item groups) x 16 (column groups): the V
// reads of a k are two broadcasts, the M reads are 16 consecutive pairs -> no bank conflicts.
//
// TN is 64 for N <= 64 (no dead columns) and 128 otherwise.  Items are sorted by error set; a
// tile whose items span a few error sets is computed once per RUN of equal error sets with that
// run's M (rows outside the run are discarded), so only tiles with more than PJ_MAX_RUNS error
// sets (or unaligned records) take the per-item path that reads every M entry from L2.
constexpr uint32_t PJ_MAX_RUNS = 8;

template <typename R, int TN>
__global__ void __launch_bounds__(PJ_THREADS) project_kernel(const ProjectArgs a) {
  using C = typename CxT<R>::type;
  using C2 = typename Cx2<R>::type;
  constexpr int KC = ProjK<R>::KC;
  constexpr int RN = TN / 16;                      // columns per thread
  constexpr int PER16 = 16 / sizeof(C);            // complex elements per 16-byte copy (2 or 1)
  constexpr int STAGE = KC * (PJ_TI + TN);         // elements of one ring slot
  extern __shared__ __align__(32) unsigned char pj_smem[];
  C* ring = reinterpret_cast<C*>(pj_smem);
  const int tid = threadIdx.x;
  const int tn = tid & 15, ti = tid >> 4;  // 16 x 16 thread grid
  const uint32_t n_tiles_i = (a.n_items + PJ_TI - 1) / PJ_TI;
  const uint32_t n_tiles_n = (a.N + TN - 1) / TN;
  const uint32_t n_tiles = n_tiles_i * n_tiles_n;
  const uint32_t n_chunks = (a.D + KC - 1) / KC;
  const C* VT = reinterpret_cast<const C*>(a.vt);
  const C* REC = reinterpret_cast<const C*>(a.rec0);
  R* OUT = reinterpret_cast<R*>(a.out);
  const bool aligned_all = (a.N % PER16) == 0 && (a.rec_stride % PER16) == 0 && (a.m_off % PER16) == 0;

  // work of this CTA: tiles blockIdx.x, +gridDim.x, ...; a "job" is one k-chunk of one run of one
  // tile (or a whole tile on the per-item path).  All of this state is uniform over the CTA.
  const uint32_t my_tiles = blockIdx.x < n_tiles ? (n_tiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  struct Job {
    uint32_t tile_k, it0, c0, ni;  // tile
    uint32_t s, s_end;             // run of equal error sets, tile-relative [s, s_end)
    uint32_t chunk, slot;
    bool fast, done;
    const C* M;
  };
  auto run_end = [&](const Job& q, uint32_t s) -> uint32_t {
    const uint32_t* es = a.eset + a.first_item + q.it0;
    const uint32_t e = es[s];
    if (es[q.ni - 1] == e) return q.ni;
    uint32_t lo = s + 1, hi = q.ni - 1;  // es[hi] != e: first index whose error set differs
    while (lo < hi) {
      const uint32_t mid = (lo + hi) >> 1;
      if (es[mid] != e) hi = mid; else lo = mid + 1;
    }
    return lo;
  };
  auto enter_tile = [&](Job& q) {
    q.s = 0;
    q.chunk = 0;
    if (q.tile_k >= my_tiles) { q.done = true; q.fast = false; return; }
    const uint32_t tile = blockIdx.x + q.tile_k * gridDim.x;
    q.it0 = (tile / n_tiles_n) * PJ_TI;
    q.c0 = (tile % n_tiles_n) * TN;
    q.ni = min((uint32_t)PJ_TI, a.n_items - q.it0);
    const uint32_t* es = a.eset + a.first_item + q.it0;
    const uint32_t e_first = es[0], e_last = es[q.ni - 1];
    const size_t off = (size_t)e_first * a.rec_stride + a.m_off;
    q.M = REC + off;
    q.s_end = q.ni;
    if (e_first == e_last) {
      q.fast = (a.N % PER16) == 0 && (off % PER16) == 0;
    } else {
      const int boundary = tid > 0 && (uint32_t)tid < q.ni && es[tid] != es[tid - 1];
      const uint32_t runs = 1 + __syncthreads_count(boundary);
      q.fast = aligned_all && runs <= PJ_MAX_RUNS;
      if (q.fast) q.s_end = run_end(q, 0);
    }
  };
  auto advance = [&](Job& q) {
    q.slot ^= 1;
    if (q.fast && ++q.chunk < n_chunks) return;
    q.chunk = 0;
    if (q.fast && q.s_end < q.ni) {  // next run of the same tile
      q.s = q.s_end;
      q.s_end = run_end(q, q.s);
      q.M = REC + (size_t)a.eset[a.first_item + q.it0 + q.s] * a.rec_stride + a.m_off;
      return;
    }
    ++q.tile_k;
    enter_tile(q);
  };
  auto issue = [&](const Job& q) {  // asynchronous copies of one job into its ring slot
    if (!q.done && q.fast) {
      const uint32_t k0 = q.chunk * KC;
      C* Vs = ring + (size_t)q.slot * STAGE;
      C* Ms = Vs + KC * PJ_TI;
      for (int x = tid; x < KC * PJ_TI / PER16; x += PJ_THREADS) {
        const int k = x / (PJ_TI / PER16), i = (x % (PJ_TI / PER16)) * PER16;
        const bool ok = k0 + k < a.D;  // v_stride is padded: tail columns exist
        cp_async16(Vs + k * PJ_TI + i, VT + (size_t)(ok ? k0 + k : 0) * a.v_stride + q.it0 + i, ok ? 16u : 0u);
      }
      for (int x = tid; x < KC * TN / PER16; x += PJ_THREADS) {
        const int k = x / (TN / PER16), c = (x % (TN / PER16)) * PER16;
        const bool ok = k0 + k < a.D && q.c0 + c < a.N;
        cp_async16(Ms + k * TN + c, q.M + (size_t)(ok ? k0 + k : 0) * a.N + (ok ? q.c0 + c : 0), ok ? 16u : 0u);
      }
    }
    cp_async_commit();  // one group per job, empty for per-item tiles and past the end
  };

  R acc[PJ_RI][RN];
  Job cur;
  cur.tile_k = 0;
  cur.slot = 0;
  cur.done = false;
  enter_tile(cur);
  issue(cur);
  while (!cur.done) {
    Job nxt = cur;
    advance(nxt);
    issue(nxt);
    cp_async_wait<1>();   // everything but the newest group has landed: cur's slot is ready
    __syncthreads();
    if (cur.fast) {
      const C* Vs = ring + (size_t)cur.slot * STAGE;
      const C* Ms = Vs + KC * PJ_TI;
      if (cur.chunk == 0) {
#pragma unroll
        for (int i = 0; i < PJ_RI; ++i)
#pragma unroll
          for (int j = 0; j < RN; ++j) acc[i][j] = R(0);
      }
#pragma unroll 8
      for (int k = 0; k < KC; ++k) {
        C vr[PJ_RI], mr[RN];
#pragma unroll
        for (int i = 0; i < PJ_RI; i += 2) {
          const C2 v2 = *reinterpret_cast<const C2*>(Vs + k * PJ_TI + ti * PJ_RI + i);
          vr[i].x = v2.x; vr[i].y = v2.y; vr[i + 1].x = v2.z; vr[i + 1].y = v2.w;
        }
#pragma unroll
        for (int p = 0; p < RN / 2; ++p) {
          const C2 m2 = *reinterpret_cast<const C2*>(Ms + k * TN + 2 * (p * 16 + tn));
          mr[2 * p].x = m2.x; mr[2 * p].y = m2.y; mr[2 * p + 1].x = m2.z; mr[2 * p + 1].y = m2.w;
        }
#pragma unroll
        for (int i = 0; i < PJ_RI; ++i)
#pragma unroll
          for (int j = 0; j < RN; ++j) {
            acc[i][j] = fma(vr[i].x, mr[j].x, acc[i][j]);
            acc[i][j] = fma(-vr[i].y, mr[j].y, acc[i][j]);
          }
      }
      if (cur.chunk + 1 == n_chunks) {  // last chunk of the run: write its population rows
#pragma unroll
        for (int i = 0; i < PJ_RI; ++i) {
          const uint32_t li = ti * PJ_RI + i;
          if (li < cur.s || li >= cur.s_end) continue;  // s_end <= ni: also the ragged last tile
          const uint32_t item = cur.it0 + li;
#pragma unroll
          for (int p = 0; p < RN / 2; ++p) {
            const uint32_t c = cur.c0 + 2 * (p * 16 + tn);
            R* o = OUT + (size_t)item * a.N + c;
            if (c + 1 < a.N) { o[0] = acc[i][2 * p]; o[1] = acc[i][2 * p + 1]; }
            else if (c < a.N) o[0] = acc[i][2 * p];
          }
        }
      }
    } else {
      // ---- many error sets in the tile (or unaligned M): every item reads its own M from L2 ----
      for (uint32_t x = tid; x < cur.ni * TN; x += PJ_THREADS) {
        const uint32_t i = x / TN, c = cur.c0 + x % TN;
        if (c >= a.N) continue;
        const uint32_t item = cur.it0 + i;
        const C* Mi = REC + (size_t)a.eset[a.first_item + item] * a.rec_stride + a.m_off;
        R s = R(0);
        for (uint32_t d = 0; d < a.D; ++d) {
          const C v = VT[(size_t)d * a.v_stride + item], m = Mi[(size_t)d * a.N + c];
          s = fma(v.x, m.x, s);
          s = fma(-v.y, m.y, s);
        }
        OUT[(size_t)item * a.N + c] = s;
      }
    }
    __syncthreads();  // the slot may be overwritten by the copies issued next iteration
    cur = nxt;
  }
  cp_async_wait<0>();
}

// min before clamping, clamp in place, mass (engine.py:445-450) of raw rows; one warp per row.
template <typename R>
__global__ void row_stats_kernel(R* probs, uint32_t n_rows, uint32_t N, double* mass, double* minv) {
  const uint32_t row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (row >= n_rows) return;
  R* p = probs + (size_t)row * N;
  double mn = 1e300, sum = 0.0;
  for (uint32_t c = lane; c < N; c += 32) {
    R v = p[c];
    mn = fmin(mn, (double)v);
    v = v > R(0) ? v : R(0);
    sum += (double)v;
    p[c] = v;
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, d));
    sum += __shfl_xor_sync(0xffffffffu, sum, d);
  }
  if (lane == 0) { mass[row] = sum; minv[row] = mn; }
}

}  // namespace ptsbe
