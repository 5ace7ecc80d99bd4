// Dense projection step on the 5th-generation tensor cores (tcgen05 + TMEM + TMA), complex64:
//
//     P[i][c] = Re( sum_d v_i[d] * M_e(i)[d][c] ),   d < D, c < N = 2^b
//
// -- the same product as project.cuh (the last np.tensordot of execute_path, reference
// tensor.py:190-216, plus transposed/real of _contract_marginal, engine.py:442-445), written
// as a REAL GEMM  P[items x N] = A[items x K] * B_e[K x N],  K = 2 D:
//
//     A[i][2d] = Re v_i[d], A[i][2d+1] = Im v_i[d]      (the item's vector as the executor
//                                                        writes it: one row of D complex)
//     B_e[2d][c] = Re M_e[d][c], B_e[2d+1][c] = -Im M_e[d][c]
//
// Precision: the north star asks 1e-5 relative on marginals, which a single TF32 pass
// (2^-11) cannot give.  Both operands are split  x = hi + lo  with hi = x truncated to the 10
// explicit mantissa bits of TF32 and lo = (x - hi) rounded to them (both exactly
// representable, so the tensor core's own conversion of the inputs changes nothing), and
//     P = A_hi B_hi + A_lo B_hi + A_hi B_lo          (fp32 accumulation in TMEM)
// drops only lo*lo and the truncation of lo: ~2^-21 relative to |a||b| per term.
//
// Data path (one persistent CTA per SM, 10 warps):
//   warp 0     TMA producer: cp.async.bulk.tensor (128-byte swizzle) of the A tile
//              [128 items x 32 floats] and of the hi / lo tiles of B_e [N x 32 floats] per
//              k-block into a ring of shared-memory stages; mbarrier complete_tx.
//   warps 2-5  split A in place (hi) and into a second tile (lo), fence.proxy.async.
//   warp 1     one elected thread issues tcgen05.mma.kind::tf32 (M = 128, N, K = 8) from
//              shared-memory descriptors; the accumulator [128 lanes x N columns] lives in
//              TMEM (double buffered); tcgen05.commit releases stages / publishes tiles.
//   warps 6-9  epilogue: tcgen05.ld of the accumulator, transposed through shared memory,
//              coalesced stores of the rows that belong to the job's error set.
// B_e depends on the error set only: the hi / lo K-major images are built once per error set
// and stage by tc_prep_b_kernel.  Work items are sorted by error set; a tile of 128
// consecutive items is multiplied once per RUN of equal error sets inside it (a "job").
#pragma once
#include <cuda.h>

#include "common.cuh"

namespace ptsbe {

constexpr int TC_BM = 128;       // items per tile (UMMA M)
constexpr int TC_BK = 32;        // floats per k-block: one 128-byte swizzle atom
constexpr int TC_THREADS = 320;  // 10 warps
constexpr int TC_MAX_STAGES = 4;
constexpr uint32_t TC_A_BYTES = TC_BM * TC_BK * 4;  // 16 KB

struct TcProjectArgs {
  const uint32_t* eset;  // [level n] error-set row of every item
  float* out;            // [n_items][N] raw (unclamped) populations
  uint32_t first_item, n_items;
  uint32_t N;            // 32 .. 256, power of two
  uint32_t kb;           // k-blocks: K / 32
  uint32_t stages;       // ring depth (fits shared memory)
  uint32_t tmem_cols;    // power of two >= 2 N, >= 32
};

// ---- PTX wrappers -----------------------------------------------------------------------
__device__ __forceinline__ uint32_t tc_smem(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
  } while (!ok);
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* tm, uint32_t bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
      ::"r"(dst), "l"(tm), "r"(bar), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}
// D[tmem] (+)= A[smem] * B[smem], TF32 inputs, fp32 accumulate; issued by ONE thread
__device__ __forceinline__ void tc_mma_tf32(uint32_t tmem_d, uint64_t desc_a, uint64_t desc_b, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
      ::"r"(tmem_d), "l"(desc_a), "l"(desc_b), "r"(idesc), "r"(accumulate)
      : "memory");
}
// K-major operand tile with 128-byte swizzle: rows of 128 bytes, 8-row groups 1024 bytes apart
// (cute::UMMA::SmemDescriptor: start >> 4 at [0,14), LBO at [16,30), SBO at [32,46), version 1
// at [46,48), layout SWIZZLE_128B = 2 at [61,64))
__device__ __forceinline__ uint64_t tc_desc(uint32_t smem_addr) {
  return (uint64_t)((smem_addr >> 4) & 0x3FFFu) | (1ull << 16) | (64ull << 32) | (1ull << 46) | (2ull << 61);
}
__device__ __forceinline__ void tc_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
      "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr)
      : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// ---- B images: once per error set and stage ---------------------------------------------
struct TcPrepArgs {
  const float2* rec0;   // pass-0 records [error sets][rec_stride] complex64
  float* b_hi;          // [error sets][N][K] K-major
  float* b_lo;
  uint32_t n_sets, D, N, K, rec_stride, m_off;
};

__device__ __forceinline__ void tc_split(float x, float& hi, float& lo) {
  hi = __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
  // lo: rounded to nearest on the 10 explicit TF32 mantissa bits (unbiased; the carry may bump the exponent)
  lo = __uint_as_float((__float_as_uint(x - hi) + 0x1000u) & 0xFFFFE000u);
}

// one CTA per (error set, 32 columns): coalesced reads of M[d][c..c+31], transposed through
// shared memory, coalesced writes of B[c][k]
__global__ void __launch_bounds__(256) tc_prep_b_kernel(const TcPrepArgs a) {
  __shared__ float2 tile[32][33];
  const uint32_t e = blockIdx.x, c0 = blockIdx.y * 32;
  const float2* M = a.rec0 + (size_t)e * a.rec_stride + a.m_off;
  float* hi = a.b_hi + (size_t)e * a.N * a.K;
  float* lo = a.b_lo + (size_t)e * a.N * a.K;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
  for (uint32_t d0 = 0; d0 < a.K / 2; d0 += 32) {
    for (int r = ty; r < 32; r += 8) {
      const uint32_t d = d0 + r;
      tile[r][tx] = (d < a.D && c0 + tx < a.N) ? M[(size_t)d * a.N + c0 + tx] : make_float2(0.f, 0.f);
    }
    __syncthreads();
    for (int r = ty; r < 32; r += 8) {  // r: column, tx: d
      const uint32_t c = c0 + r, d = d0 + tx;
      if (c < a.N && 2 * d + 1 < a.K) {
        const float2 m = tile[tx][r];
        float h0, l0, h1, l1;
        tc_split(m.x, h0, l0);
        tc_split(-m.y, h1, l1);
        *reinterpret_cast<float2*>(hi + (size_t)c * a.K + 2 * d) = make_float2(h0, h1);
        *reinterpret_cast<float2*>(lo + (size_t)c * a.K + 2 * d) = make_float2(l0, l1);
      }
    }
    __syncthreads();
  }
}

// ---- the GEMM ---------------------------------------------------------------------------
// first index > s (tile-relative) whose error set differs from es[s]; es has ni valid entries
__device__ __forceinline__ uint32_t tc_run_end(const uint32_t* es, uint32_t s, uint32_t ni) {
  const uint32_t e = es[s];
  if (es[ni - 1] == e) return ni;
  uint32_t lo = s + 1, hi = ni - 1;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (es[mid] != e) hi = mid; else lo = mid + 1;
  }
  return lo;
}

__global__ void __launch_bounds__(TC_THREADS, 1)
project_tc_kernel(const __grid_constant__ CUtensorMap tm_a, const __grid_constant__ CUtensorMap tm_bhi,
                  const __grid_constant__ CUtensorMap tm_blo, const TcProjectArgs a) {
  extern __shared__ unsigned char tc_raw[];
  // 128-byte swizzle wants 1024-byte aligned tiles
  unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(tc_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t N = a.N, KB = a.kb, S = a.stages;
  const uint32_t b_bytes = N * TC_BK * 4;
  const uint32_t stage_bytes = 2 * TC_A_BYTES + 2 * b_bytes;
  float* stg = reinterpret_cast<float*>(base + (size_t)S * stage_bytes);                // [4][32][33]
  uint64_t* bars = reinterpret_cast<uint64_t*>(stg + 4 * 32 * 33);
  uint64_t* full = bars;                     // [S]  TMA landed
  uint64_t* conv = bars + TC_MAX_STAGES;     // [S]  A split done
  uint64_t* empty = bars + 2 * TC_MAX_STAGES;  // [S]  MMAs of the stage retired
  uint64_t* tfull = bars + 3 * TC_MAX_STAGES;  // [2]  accumulator complete
  uint64_t* tempty = tfull + 2;                // [2]  accumulator drained
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (uint32_t s = 0; s < S; ++s) {
      mbar_init(tc_smem(full + s), 1);
      mbar_init(tc_smem(conv + s), 128);
      mbar_init(tc_smem(empty + s), 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(tc_smem(tfull + i), 1);
      mbar_init(tc_smem(tempty + i), 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tc_smem(tmem_slot)),
                 "r"(a.tmem_cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const uint32_t n_tiles = (a.n_items + TC_BM - 1) / TC_BM;
  const uint32_t* ES = a.eset + a.first_item;

  if (warp == 0) {
    // ===== TMA producer =====
    if (lane == 0) {
      uint32_t st = 0, ph = 0;
      for (uint32_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
        const uint32_t it0 = tile * TC_BM, ni = min((uint32_t)TC_BM, a.n_items - it0);
        for (uint32_t s = 0; s < ni;) {
          const uint32_t e = ES[it0 + s], s_end = tc_run_end(ES + it0, s, ni);
          for (uint32_t kb = 0; kb < KB; ++kb) {
            mbar_wait(tc_smem(empty + st), ph ^ 1);
            const uint32_t sb = tc_smem(base + (size_t)st * stage_bytes), fb = tc_smem(full + st);
            mbar_expect_tx(fb, TC_A_BYTES + 2 * b_bytes);
            tma_load_2d(sb, &tm_a, fb, (int)(kb * TC_BK), (int)it0);
            tma_load_2d(sb + 2 * TC_A_BYTES, &tm_bhi, fb, (int)(kb * TC_BK), (int)(e * N));
            tma_load_2d(sb + 2 * TC_A_BYTES + b_bytes, &tm_blo, fb, (int)(kb * TC_BK), (int)(e * N));
            if (++st == S) { st = 0; ph ^= 1; }
          }
          s = s_end;
        }
      }
    }
  } else if (warp == 1) {
    // ===== MMA issuer =====
    if (lane == 0) {
      // instruction descriptor (cute::UMMA::InstrDescriptor): D = F32 at [4,6), A = B = TF32 at
      // [7,10) / [10,13), both K-major, N >> 3 at [17,23), M >> 4 at [24,29)
      const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((N >> 3) << 17) | ((TC_BM >> 4) << 24);
      uint32_t st = 0, ph = 0, acc = 0, aph = 0;
      for (uint32_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
        const uint32_t it0 = tile * TC_BM, ni = min((uint32_t)TC_BM, a.n_items - it0);
        for (uint32_t s = 0; s < ni;) {
          const uint32_t s_end = tc_run_end(ES + it0, s, ni);
          mbar_wait(tc_smem(tempty + acc), aph ^ 1);
          tc_fence_after();
          const uint32_t d_tmem = tmem_base + acc * N;
          for (uint32_t kb = 0; kb < KB; ++kb) {
            mbar_wait(tc_smem(full + st), ph);
            mbar_wait(tc_smem(conv + st), ph);
            tc_fence_after();
            const uint32_t sb = tc_smem(base + (size_t)st * stage_bytes);
            const uint32_t a_hi = sb, a_lo = sb + TC_A_BYTES, b_hi = sb + 2 * TC_A_BYTES, b_lo = b_hi + b_bytes;
#pragma unroll
            for (uint32_t k = 0; k < TC_BK / 8; ++k) {  // UMMA K = 8 TF32 = 32 bytes inside the swizzle atom
              const uint32_t off = k * 32;
              tc_mma_tf32(d_tmem, tc_desc(a_hi + off), tc_desc(b_hi + off), idesc, (kb | k) ? 1u : 0u);
              tc_mma_tf32(d_tmem, tc_desc(a_lo + off), tc_desc(b_hi + off), idesc, 1u);
              tc_mma_tf32(d_tmem, tc_desc(a_hi + off), tc_desc(b_lo + off), idesc, 1u);
            }
            tc_commit(tc_smem(empty + st));  // stage reusable once these MMAs have read it
            if (++st == S) { st = 0; ph ^= 1; }
          }
          tc_commit(tc_smem(tfull + acc));   // accumulator complete
          if (++acc == 2) { acc = 0; aph ^= 1; }
          s = s_end;
        }
      }
    }
  } else if (warp < 6) {
    // ===== A split: hi in place, lo beside it =====
    const uint32_t t = threadIdx.x - 64;  // 0..127
    uint32_t st = 0, ph = 0;
    for (uint32_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
      const uint32_t it0 = tile * TC_BM, ni = min((uint32_t)TC_BM, a.n_items - it0);
      uint32_t jobs = 0;
      if (lane == 0)
        for (uint32_t s = 0; s < ni; s = tc_run_end(ES + it0, s, ni)) ++jobs;
      jobs = __shfl_sync(0xffffffffu, jobs, 0);
      for (uint32_t q = 0; q < jobs * KB; ++q) {
        mbar_wait(tc_smem(full + st), ph);
        float4* hi = reinterpret_cast<float4*>(base + (size_t)st * stage_bytes);
        float4* lo = reinterpret_cast<float4*>(base + (size_t)st * stage_bytes + TC_A_BYTES);
#pragma unroll
        for (int i = 0; i < (int)(TC_A_BYTES / 16 / 128); ++i) {
          const float4 x = hi[t + 128 * i];
          float4 h, l;
          tc_split(x.x, h.x, l.x); tc_split(x.y, h.y, l.y); tc_split(x.z, h.z, l.z); tc_split(x.w, h.w, l.w);
          hi[t + 128 * i] = h;
          lo[t + 128 * i] = l;
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> tensor-core reads
        mbar_arrive(tc_smem(conv + st));
        if (++st == S) { st = 0; ph ^= 1; }
      }
    }
  } else {
    // ===== epilogue: TMEM -> registers -> shared (transpose) -> global =====
    const uint32_t quad = warp & 3;              // TMEM lanes [32 quad, 32 quad + 32)
    float* my = stg + (size_t)quad * 32 * 33;
    uint32_t acc = 0, aph = 0;
    for (uint32_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
      const uint32_t it0 = tile * TC_BM, ni = min((uint32_t)TC_BM, a.n_items - it0);
      uint32_t s = 0;
      while (s < ni) {
        uint32_t s_end = 0;
        if (lane == 0) s_end = tc_run_end(ES + it0, s, ni);
        s_end = __shfl_sync(0xffffffffu, s_end, 0);
        mbar_wait(tc_smem(tfull + acc), aph);
        tc_fence_after();
        const uint32_t r_lo = quad * 32, r_hi = r_lo + 32;
        const bool any = s < r_hi && s_end > r_lo;  // warp-uniform: some of this warp's rows are in the run
        if (any) {
          for (uint32_t c0 = 0; c0 < N; c0 += 32) {
            uint32_t r[32];
            tc_ld32(tmem_base + ((quad * 32) << 16) + acc * N + c0, r);
#pragma unroll
            for (int j = 0; j < 32; ++j) my[lane * 33 + j] = __uint_as_float(r[j]);
            __syncwarp();
            for (uint32_t row = max(s, r_lo); row < min(s_end, r_hi); ++row)
              a.out[(size_t)(it0 + row) * N + c0 + lane] = my[(row - r_lo) * 33 + lane];
            __syncwarp();
          }
        }
        tc_fence_before();
        mbar_arrive(tc_smem(tempty + acc));
        if (++acc == 2) { acc = 0; aph ^= 1; }
        s = s_end;
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(a.tmem_cols) : "memory");
  }
}

}  // namespace ptsbe
