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

template <typename R> struct ProjK { static constexpr int KC = 32; };
template <> struct ProjK<double> { static constexpr int KC = 16; };

template <typename R> struct Cx2;  // two complex numbers, one 16/32-byte load
template <> struct Cx2<float> { using type = float4; };
template <> struct Cx2<double> { using type = double4; };

// Both operands are k-major (vt[d][item], M[d][c]), so the tiles go to shared memory with
// straight, coalesced, conflict-free vector copies: Vs[KC][TI], Ms[KC][TN].  A warp is
// 2 (item groups) x 16 (column groups): the V reads of a k are two broadcasts, the M reads
// are 16 consecutive pairs -> no bank conflicts on either side.
template <typename R>
__global__ void __launch_bounds__(PJ_THREADS) project_kernel(const ProjectArgs a) {
  using C = typename CxT<R>::type;
  using C2 = typename Cx2<R>::type;
  constexpr int KC = ProjK<R>::KC;
  extern __shared__ __align__(32) unsigned char pj_smem[];
  C* Vs = reinterpret_cast<C*>(pj_smem);
  C* Ms = Vs + KC * PJ_TI;
  const int tid = threadIdx.x;
  const int tn = tid & 15, ti = tid >> 4;  // 16 x 16 thread grid
  const uint32_t n_tiles_i = (a.n_items + PJ_TI - 1) / PJ_TI;
  const uint32_t n_tiles_n = (a.N + PJ_TN - 1) / PJ_TN;
  const C* VT = reinterpret_cast<const C*>(a.vt);
  const C* REC = reinterpret_cast<const C*>(a.rec0);
  R* OUT = reinterpret_cast<R*>(a.out);

  for (uint32_t tile = blockIdx.x; tile < n_tiles_i * n_tiles_n; tile += gridDim.x) {
    // column tiles of one item tile are adjacent in the schedule: its V columns stay in L1/L2
    const uint32_t it0 = (tile / n_tiles_n) * PJ_TI, c0 = (tile % n_tiles_n) * PJ_TN;
    const uint32_t ni = min((uint32_t)PJ_TI, a.n_items - it0);
    const uint32_t e_first = a.eset[a.first_item + it0], e_last = a.eset[a.first_item + it0 + ni - 1];
    if (e_first == e_last) {
      // ---- uniform tile: one M for all items ----
      const C* M = REC + (size_t)e_first * a.rec_stride + a.m_off;
      R acc[PJ_RI][PJ_RN];
#pragma unroll
      for (int i = 0; i < PJ_RI; ++i)
#pragma unroll
        for (int j = 0; j < PJ_RN; ++j) acc[i][j] = R(0);
      for (uint32_t k0 = 0; k0 < a.D; k0 += KC) {
        __syncthreads();
        // V chunk: rows k0.., columns it0.. (v_stride is padded, so the tail columns exist)
        for (int x = tid; x < KC * PJ_TI / 2; x += PJ_THREADS) {
          const int k = x / (PJ_TI / 2), i2 = x % (PJ_TI / 2);
          C2 val = {};
          if (k0 + k < a.D)
            val = *reinterpret_cast<const C2*>(VT + (size_t)(k0 + k) * a.v_stride + it0 + 2 * i2);
          *reinterpret_cast<C2*>(Vs + k * PJ_TI + 2 * i2) = val;
        }
        // M chunk
        if (c0 + PJ_TN <= a.N && (a.N & 1) == 0 && (((size_t)e_first * a.rec_stride + a.m_off) & 1) == 0) {
          for (int x = tid; x < KC * PJ_TN / 2; x += PJ_THREADS) {
            const int k = x / (PJ_TN / 2), c2 = x % (PJ_TN / 2);
            C2 val = {};
            if (k0 + k < a.D) val = *reinterpret_cast<const C2*>(M + (size_t)(k0 + k) * a.N + c0 + 2 * c2);
            *reinterpret_cast<C2*>(Ms + k * PJ_TN + 2 * c2) = val;
          }
        } else {
          for (int x = tid; x < KC * PJ_TN; x += PJ_THREADS) {
            const int k = x / PJ_TN, c = x % PJ_TN;
            C val; val.x = 0; val.y = 0;
            if (c0 + c < a.N && k0 + k < a.D) val = M[(size_t)(k0 + k) * a.N + c0 + c];
            Ms[k * PJ_TN + c] = val;
          }
        }
        __syncthreads();
#pragma unroll 4
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
      }
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
    } else {
      // ---- tile straddles error sets: every item reads its own M from L2 ----
      for (uint32_t x = tid; x < ni * PJ_TN; x += PJ_THREADS) {
        const uint32_t i = x / PJ_TN, c = c0 + x % PJ_TN;
        if (c >= a.N) continue;
        const uint32_t item = it0 + i;
        const C* M = REC + (size_t)a.eset[a.first_item + item] * a.rec_stride + a.m_off;
        R s = R(0);
        for (uint32_t d = 0; d < a.D; ++d) {
          const C v = VT[(size_t)d * a.v_stride + item], m = M[(size_t)d * a.N + c];
          s = fma(v.x, m.x, s);
          s = fma(-v.y, m.y, s);
        }
        OUT[(size_t)item * a.N + c] = s;
      }
    }
  }
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
