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
template <typename R>
__global__ void __launch_bounds__(PJ_THREADS) project_kernel(const ProjectArgs a) {
  using C = typename CxT<R>::type;
  using C2 = typename Cx2<R>::type;
  constexpr int KC = ProjK<R>::KC;
  constexpr int PER16 = 16 / sizeof(C);            // complex elements per 16-byte copy (2 or 1)
  constexpr int STAGE = KC * (PJ_TI + PJ_TN);      // elements of one ring slot
  extern __shared__ __align__(32) unsigned char pj_smem[];
  C* ring = reinterpret_cast<C*>(pj_smem);
  const int tid = threadIdx.x;
  const int tn = tid & 15, ti = tid >> 4;  // 16 x 16 thread grid
  const uint32_t n_tiles_i = (a.n_items + PJ_TI - 1) / PJ_TI;
  const uint32_t n_tiles_n = (a.N + PJ_TN - 1) / PJ_TN;
  const uint32_t n_tiles = n_tiles_i * n_tiles_n;
  const uint32_t n_chunks = (a.D + KC - 1) / KC;
  const C* VT = reinterpret_cast<const C*>(a.vt);
  const C* REC = reinterpret_cast<const C*>(a.rec0);
  R* OUT = reinterpret_cast<R*>(a.out);

  // work of this CTA: tiles blockIdx.x, +gridDim.x, ...; a "job" is one k-chunk of one tile
  const uint32_t my_tiles = blockIdx.x < n_tiles ? (n_tiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  const uint32_t n_jobs = my_tiles * n_chunks;

  auto tile_of = [&](uint32_t job, uint32_t& it0, uint32_t& c0, uint32_t& ni, uint32_t& k0) {
    const uint32_t tile = blockIdx.x + (job / n_chunks) * gridDim.x;
    it0 = (tile / n_tiles_n) * PJ_TI;
    c0 = (tile % n_tiles_n) * PJ_TN;
    ni = min((uint32_t)PJ_TI, a.n_items - it0);
    k0 = (job % n_chunks) * KC;
  };
  // uniform tile <=> all its items share one error set (one M); fast path needs aligned M rows
  auto uniform_m = [&](uint32_t it0, uint32_t ni, const C*& M) -> bool {
    const uint32_t e_first = a.eset[a.first_item + it0], e_last = a.eset[a.first_item + it0 + ni - 1];
    const size_t off = (size_t)e_first * a.rec_stride + a.m_off;
    M = REC + off;
    return e_first == e_last && (a.N % PER16) == 0 && (off % PER16) == 0;
  };
  auto issue = [&](uint32_t job) {  // asynchronous copies of one job into ring slot job & 1
    if (job < n_jobs) {
      uint32_t it0, c0, ni, k0;
      tile_of(job, it0, c0, ni, k0);
      const C* M;
      if (uniform_m(it0, ni, M)) {
        C* Vs = ring + (size_t)(job & 1) * STAGE;
        C* Ms = Vs + KC * PJ_TI;
        for (int x = tid; x < KC * PJ_TI / PER16; x += PJ_THREADS) {
          const int k = x / (PJ_TI / PER16), i = (x % (PJ_TI / PER16)) * PER16;
          const bool ok = k0 + k < a.D;  // v_stride is padded: tail columns exist
          cp_async16(Vs + k * PJ_TI + i, VT + (size_t)(ok ? k0 + k : 0) * a.v_stride + it0 + i, ok ? 16u : 0u);
        }
        for (int x = tid; x < KC * PJ_TN / PER16; x += PJ_THREADS) {
          const int k = x / (PJ_TN / PER16), c = (x % (PJ_TN / PER16)) * PER16;
          const bool ok = k0 + k < a.D && c0 + c < a.N;
          cp_async16(Ms + k * PJ_TN + c, M + (size_t)(ok ? k0 + k : 0) * a.N + (ok ? c0 + c : 0), ok ? 16u : 0u);
        }
      }
    }
    cp_async_commit();  // one group per job, empty for slow-path tiles and past the end
  };

  R acc[PJ_RI][PJ_RN];
  issue(0);
  for (uint32_t job = 0; job < n_jobs; ++job) {
    issue(job + 1);
    cp_async_wait<1>();   // everything but the newest group has landed: job's slot is ready
    __syncthreads();
    uint32_t it0, c0, ni, k0;
    tile_of(job, it0, c0, ni, k0);
    const C* M;
    const bool fast = uniform_m(it0, ni, M);
    if (fast) {
      const C* Vs = ring + (size_t)(job & 1) * STAGE;
      const C* Ms = Vs + KC * PJ_TI;
      if (k0 == 0) {
#pragma unroll
        for (int i = 0; i < PJ_RI; ++i)
#pragma unroll
          for (int j = 0; j < PJ_RN; ++j) acc[i][j] = R(0);
      }
#pragma unroll 8
      for (int k = 0; k < KC; ++k) {
        C vr[PJ_RI], mr[PJ_RN];
#pragma unroll
        for (int i = 0; i < PJ_RI; i += 2) {
          const C2 v2 = *reinterpret_cast<const C2*>(Vs + k * PJ_TI + ti * PJ_RI + i);
          vr[i].x = v2.x; vr[i].y = v2.y; vr[i + 1].x = v2.z; vr[i + 1].y = v2.w;
        }
#pragma unroll
        for (int p = 0; p < PJ_RN / 2; ++p) {
          const C2 m2 = *reinterpret_cast<const C2*>(Ms + k * PJ_TN + 2 * (p * 16 + tn));
          mr[2 * p].x = m2.x; mr[2 * p].y = m2.y; mr[2 * p + 1].x = m2.z; mr[2 * p + 1].y = m2.w;
        }
#pragma unroll
        for (int i = 0; i < PJ_RI; ++i)
#pragma unroll
          for (int j = 0; j < PJ_RN; ++j) {
            acc[i][j] = fma(vr[i].x, mr[j].x, acc[i][j]);
            acc[i][j] = fma(-vr[i].y, mr[j].y, acc[i][j]);
          }
      }
      if (k0 + KC >= a.D) {  // last chunk of the tile: write the population rows
#pragma unroll
        for (int i = 0; i < PJ_RI; ++i) {
          const uint32_t item = it0 + ti * PJ_RI + i;
          if (item >= a.n_items) continue;
#pragma unroll
          for (int p = 0; p < PJ_RN / 2; ++p) {
            const uint32_t c = c0 + 2 * (p * 16 + tn);
            R* o = OUT + (size_t)item * a.N + c;
            if (c + 1 < a.N) { o[0] = acc[i][2 * p]; o[1] = acc[i][2 * p + 1]; }
            else if (c < a.N) o[0] = acc[i][2 * p];
          }
        }
      }
    } else if (k0 == 0) {
      // ---- tile straddles error sets (or unaligned M): every item reads its own M from L2 ----
      for (uint32_t x = tid; x < ni * PJ_TN; x += PJ_THREADS) {
        const uint32_t i = x / PJ_TN, c = c0 + x % PJ_TN;
        if (c >= a.N) continue;
        const uint32_t item = it0 + i;
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
