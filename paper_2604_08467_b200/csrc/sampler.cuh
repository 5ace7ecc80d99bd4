// Non-degenerate batched sampler (north-star subsystem 3).
//
// For every unique (error set, prefix) work item of a stage: turn the
// unnormalised marginal into an exact fixed-point CDF, draw the item's shot
// multiplicity from counter-based Philox uniforms, and emit the non-empty
// outcomes in ascending order.  The next stage's work list is then built by an
// order-preserving compaction (scan.cuh), so children of one error set stay in
// lexicographic prefix order -- the same order the reference iterates in
// (engine.py:513-523 `for prefix in sorted(groups)`), which is what makes the
// RNG stream of a work item (error-set id, stage, rank) reproducible on any
// number of GPUs.
//
// Replaces rng.multinomial + flatnonzero + dict insert (engine.py:519-522).
// Every operation that decides a count is integer arithmetic, so the CPU oracle
// (oracle/ptsbe_oracle.py: fixed_point_weights / multinomial_counts) reproduces
// the counts bit for bit from the same float64 marginals.
#pragma once
#include "common.cuh"
#include "scan.cuh"

namespace ptsbe {

// ---- Philox-4x32-10 (Salmon et al. 2011), counter = (c0,c1,c2,c3), key = (k0,k1) ----
struct Philox4 { uint32_t v[4]; };

__host__ __device__ __forceinline__ Philox4 philox4x32_10(uint32_t c0, uint32_t c1, uint32_t c2,
                                                          uint32_t c3, uint32_t k0, uint32_t k1) {
  const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u, W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint64_t p0 = (uint64_t)M0 * c0, p1 = (uint64_t)M1 * c2;
    const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0;
    const uint32_t n1 = (uint32_t)p1;
    const uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1;
    const uint32_t n3 = (uint32_t)p0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    k0 += W0; k1 += W1;
  }
  Philox4 o; o.v[0] = c0; o.v[1] = c1; o.v[2] = c2; o.v[3] = c3;
  return o;
}

struct SampleArgs {
  const void* probs;        // [items][nb] real, float (is_f32) or double
  const uint32_t* mult;     // [items] shots to split
  const uint32_t* slot_off; // [items] first output slot of the item (exclusive scan of mult)
  const uint32_t* eset_id;  // [items] GLOBAL error-set id (RNG stream)
  const uint32_t* rank;     // [items] rank of the prefix inside its error set (sorted order)
  const double* mass;       // [items] or null: then sum / minimum are taken from the raw row here
  const double* minv;       // [items] or null
  uint32_t* slot_index;     // [total shots] outcome index of each non-empty child
  uint32_t* slot_count;     // [total shots] its count
  uint32_t* nnz;            // [items] number of non-empty children
  unsigned long long* flag; // [1] min over flagged items of (eset id << 16 | stage << 8 | kind)
  uint32_t* flag_count;     // [1]
  uint64_t n_items;
  uint32_t first_item;      // probs/mass/minv are indexed by (item - first_item)
  uint32_t b;               // nb = 2^b
  uint32_t stage;
  uint32_t k0, k1;          // Philox key = seed
  uint32_t is_f32;
  double vanish;            // engine.py:54 VANISHING_MASS
  double neg_abs, neg_rel;  // engine.py:53 NEGATIVE_DIAG_TOLERANCE (+ relative term for c64)
  // Non-unitary Kraus operators (amplitude damping) give a trajectory a weight < 1, and every
  // unnormalised mass of that error set carries it.  The vanishing-mass guard is therefore
  // taken relative to the error set's stage-1 mass (== 1 for the reference's unitary errors, so
  // the reference behaviour is unchanged): stage 1 records it, later stages compare against it.
  double* set_mass;         // [error-set rows] or null (absolute guard)
  const uint32_t* eset_row; // [items] row of the item's error set in set_mass
  double vanish_stage1;     // absolute floor for the stage-1 mass itself
  // non-proportional sampler (nonprop_kernel; reference engine.py:527-576)
  uint32_t np_mode;         // 1: weighted choice of mult[item] distinct outcomes, 2: exhaustive harvest
  uint32_t child_mult;      // multiplicity handed to every emitted child (slot_count)
  double threshold;         // harvest: conditional probability an outcome must reach
  double* slot_prob;        // harvest: conditional probability of each emitted outcome
  uint32_t np_floor_bits;   // choice: weights below max >> np_floor_bits count as zero probability
};

constexpr int SAMPLE_THREADS = 128;

// One CTA per work item.  Shared memory: u64 cdf[nb] + u32 cnt[nb] + scan scratch.
__global__ void __launch_bounds__(SAMPLE_THREADS) sample_kernel(const SampleArgs a) {
  extern __shared__ __align__(16) unsigned char sm[];
  const uint32_t nb = 1u << a.b;
  uint64_t* cdf = reinterpret_cast<uint64_t*>(sm);
  uint32_t* cnt = reinterpret_cast<uint32_t*>(cdf + nb);
  __shared__ uint64_t ws64[33];
  __shared__ uint32_t ws32[33];
  __shared__ double redmax[SAMPLE_THREADS / 32], redmin[SAMPLE_THREADS / 32], redsum[SAMPLE_THREADS / 32];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const uint32_t per = (nb + SAMPLE_THREADS - 1) / SAMPLE_THREADS;

  for (uint64_t it = blockIdx.x; it < a.n_items; it += gridDim.x) {
    const uint64_t item = a.first_item + it;
    const uint32_t m = a.mult[item];
    // ---- load (coalesced), clamp, max ----
    double* pd = reinterpret_cast<double*>(cdf);
    double mx = 0.0, rawmin = 1e300, csum = 0.0;
    if (a.is_f32) {
      const float* p = reinterpret_cast<const float*>(a.probs) + it * nb;
      for (uint32_t k = tid; k < nb; k += SAMPLE_THREADS) {
        double v = (double)p[k]; rawmin = fmin(rawmin, v);
        v = v > 0.0 ? v : 0.0; pd[k] = v; mx = fmax(mx, v); csum += v;
      }
    } else {
      const double* p = reinterpret_cast<const double*>(a.probs) + it * nb;
      for (uint32_t k = tid; k < nb; k += SAMPLE_THREADS) {
        double v = p[k]; rawmin = fmin(rawmin, v);
        v = v > 0.0 ? v : 0.0; pd[k] = v; mx = fmax(mx, v); csum += v;
      }
    }
    for (uint32_t k = tid; k < nb; k += SAMPLE_THREADS) cnt[k] = 0;
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
      mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, d));
      rawmin = fmin(rawmin, __shfl_xor_sync(0xffffffffu, rawmin, d));
      csum += __shfl_xor_sync(0xffffffffu, csum, d);
    }
    if (lane == 0) { redmax[wid] = mx; redmin[wid] = rawmin; redsum[wid] = csum; }
    __syncthreads();
    mx = redmax[0]; rawmin = redmin[0]; csum = redsum[0];
#pragma unroll
    for (int w = 1; w < SAMPLE_THREADS / 32; ++w) {
      mx = fmax(mx, redmax[w]); rawmin = fmin(rawmin, redmin[w]); csum += redsum[w];
    }

    // ---- guards (engine.py:447-448, 475-476, 484-485) ----
    uint32_t bad = 0;
    {
      const double ms = a.mass ? a.mass[it] : csum, mn = a.minv ? a.minv[it] : rawmin;
      double floor_mass = a.vanish;
      if (a.set_mass) {
        if (a.stage == 1) { floor_mass = a.vanish_stage1; if (tid == 0) a.set_mass[a.eset_row[item]] = ms; }
        else floor_mass = a.vanish * a.set_mass[a.eset_row[item]];
      }
      if (mn < a.neg_abs - a.neg_rel * ms) bad = PTSBE_ENUMERIC;
      else if (ms < floor_mass) bad = PTSBE_EIMPOSSIBLE;
    }
    if (!bad && !(mx > 0.0)) bad = PTSBE_EIMPOSSIBLE;
    if (bad) {
      if (tid == 0) {
        a.nnz[item] = 0;
        atomicMin(a.flag, ((unsigned long long)a.eset_id[item] << 16) |
                              ((unsigned long long)(a.stage & 0xff) << 8) | bad);
        atomicAdd(a.flag_count, 1u);
      }
      __syncthreads();
      continue;
    }

    // ---- exact fixed-point weights: w_k = floor(p_k * 2^shift), shift from max only ----
    int ex;
    frexp(mx, &ex);                       // mx = f * 2^ex, f in [0.5, 1)
    const int shift = (62 - (int)a.b) - ex;  // p_k * 2^shift < 2^(62-b)
    const uint32_t k0 = tid * per;
    uint64_t local = 0;
    for (uint32_t k = k0; k < k0 + per && k < nb; ++k) {
      const uint64_t w = (uint64_t)ldexp(pd[k], shift);
      local += w;
      cdf[k] = w;  // same 8-byte slot as pd[k]; only this thread touches it
    }
    uint64_t total;
    uint64_t run = block_exclusive<uint64_t>(local, ws64, &total);
    for (uint32_t k = k0; k < k0 + per && k < nb; ++k) {
      run += cdf[k];
      cdf[k] = run;  // inclusive
    }
    __syncthreads();

    // ---- draws: outcome = #{k : cdf[k] <= r}, r = floor(x * W / 2^64) ----
    const uint32_t rk = a.rank[item], es = a.eset_id[item];
    for (uint32_t t = tid; t < m; t += SAMPLE_THREADS) {
      const Philox4 x = philox4x32_10(t, rk, a.stage, es, a.k0, a.k1);
      const uint64_t x64 = ((uint64_t)x.v[1] << 32) | x.v[0];
      const uint64_t r = __umul64hi(x64, total);
      uint32_t lo = 0, hi = nb;  // first index with cdf > r
      while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (cdf[mid] <= r) lo = mid + 1; else hi = mid;
      }
      atomicAdd(&cnt[lo], 1u);
    }
    __syncthreads();

    // ---- ordered emission of non-empty outcomes ----
    uint32_t mine = 0;
    for (uint32_t k = k0; k < k0 + per && k < nb; ++k) mine += cnt[k] != 0;
    uint32_t tot32;
    uint32_t pos = block_exclusive<uint32_t>(mine, ws32, &tot32);
    const uint32_t base = a.slot_off[item];
    for (uint32_t k = k0; k < k0 + per && k < nb; ++k) {
      const uint32_t c = cnt[k];
      if (c) { a.slot_index[base + pos] = k; a.slot_count[base + pos] = c; ++pos; }
    }
    if (tid == 0) a.nnz[item] = tot32;
    __syncthreads();
  }
}

// Non-proportional sampler (reference engine.py:527-576), one CTA per work item.
//   np_mode 1 (non-final stages): mult[item] DISTINCT outcomes, weighted, without replacement --
//     the distribution of rng.choice(positive, size, replace=False, p) (engine.py:555) as successive
//     draws from the remaining integer weights: draw t lands at r = floor(x_t * W_t / 2^64) in the
//     inclusive CDF, the chosen outcome's weight is then removed from the CDF tail.  Same fixed-point
//     weights and Philox counters as sample_kernel, so the oracle (wor_choice) reproduces the choice
//     bit for bit from the same float64 marginals.
//   np_mode 2 (final stage, exhaustive): every outcome whose conditional probability
//     clamp(P_k) / mass reaches `threshold`, tagged with it (engine.py:562-568).
// Children are emitted in ascending outcome order with slot_count = child_mult.
__global__ void __launch_bounds__(SAMPLE_THREADS) nonprop_kernel(const SampleArgs a) {
  extern __shared__ __align__(16) unsigned char sm[];
  const uint32_t nb = 1u << a.b;
  uint64_t* cdf = reinterpret_cast<uint64_t*>(sm);
  uint32_t* cnt = reinterpret_cast<uint32_t*>(cdf + nb);
  __shared__ uint64_t ws64[33];
  __shared__ uint32_t ws32[33];
  __shared__ double redmax[SAMPLE_THREADS / 32], redmin[SAMPLE_THREADS / 32], redsum[SAMPLE_THREADS / 32];
  __shared__ uint32_t s_pick;
  __shared__ uint64_t s_total;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const uint32_t per = (nb + SAMPLE_THREADS - 1) / SAMPLE_THREADS;

  for (uint64_t it = blockIdx.x; it < a.n_items; it += gridDim.x) {
    const uint64_t item = a.first_item + it;
    const uint32_t m = a.mult[item];
    double* pd = reinterpret_cast<double*>(cdf);
    double mx = 0.0, rawmin = 1e300, csum = 0.0;
    for (uint32_t k = tid; k < nb; k += SAMPLE_THREADS) {
      double v = a.is_f32 ? (double)(reinterpret_cast<const float*>(a.probs) + it * nb)[k]
                          : (reinterpret_cast<const double*>(a.probs) + it * nb)[k];
      rawmin = fmin(rawmin, v);
      v = v > 0.0 ? v : 0.0; pd[k] = v; mx = fmax(mx, v); csum += v;
      cnt[k] = 0;
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
      mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, d));
      rawmin = fmin(rawmin, __shfl_xor_sync(0xffffffffu, rawmin, d));
      csum += __shfl_xor_sync(0xffffffffu, csum, d);
    }
    if (lane == 0) { redmax[wid] = mx; redmin[wid] = rawmin; redsum[wid] = csum; }
    __syncthreads();
    mx = redmax[0]; rawmin = redmin[0]; csum = redsum[0];
#pragma unroll
    for (int w = 1; w < SAMPLE_THREADS / 32; ++w) {
      mx = fmax(mx, redmax[w]); rawmin = fmin(rawmin, redmin[w]); csum += redsum[w];
    }
    // ---- guards (engine.py:447-448, 475-476, 484-485), as sample_kernel ----
    uint32_t bad = 0;
    {
      const double ms = a.mass ? a.mass[it] : csum, mn = a.minv ? a.minv[it] : rawmin;
      double floor_mass = a.vanish;
      if (a.set_mass) {
        if (a.stage == 1) { floor_mass = a.vanish_stage1; if (tid == 0) a.set_mass[a.eset_row[item]] = ms; }
        else floor_mass = a.vanish * a.set_mass[a.eset_row[item]];
      }
      if (mn < a.neg_abs - a.neg_rel * ms) bad = PTSBE_ENUMERIC;
      else if (ms < floor_mass) bad = PTSBE_EIMPOSSIBLE;
    }
    if (!bad && !(mx > 0.0)) bad = PTSBE_EIMPOSSIBLE;
    if (bad) {
      if (tid == 0) {
        a.nnz[item] = 0;
        atomicMin(a.flag, ((unsigned long long)a.eset_id[item] << 16) |
                              ((unsigned long long)(a.stage & 0xff) << 8) | bad);
        atomicAdd(a.flag_count, 1u);
      }
      __syncthreads();
      continue;
    }
    const uint32_t k0 = tid * per;
    const uint32_t base = a.slot_off[item];
    if (a.np_mode == 2) {
      // ---- exhaustive harvest: p_k = clamp(P_k) / mass >= threshold, ascending k ----
      const double ms = a.mass ? a.mass[it] : csum;
      uint32_t mine = 0;
      for (uint32_t k = k0; k < k0 + per && k < nb; ++k) mine += (pd[k] / ms) >= a.threshold;
      uint32_t tot32;
      uint32_t pos = block_exclusive<uint32_t>(mine, ws32, &tot32);
      for (uint32_t k = k0; k < k0 + per && k < nb; ++k) {
        const double pk = pd[k] / ms;
        if (pk >= a.threshold) {
          a.slot_index[base + pos] = k;
          a.slot_count[base + pos] = a.child_mult;
          a.slot_prob[base + pos] = pk;
          ++pos;
        }
      }
      if (tid == 0) a.nnz[item] = tot32;
      __syncthreads();
      continue;
    }
    // ---- exact fixed-point weights and inclusive CDF, as sample_kernel ----
    int ex;
    frexp(mx, &ex);
    const int shift = (62 - (int)a.b) - ex;
    // Outcomes whose weight is below 2^-np_floor_bits of the row maximum are rounding noise of an
    // exactly-zero probability (the reference tests probs > 0.0, engine.py:550, and then fails on the
    // noise child with a vanishing-mass error at the next stage -- a rounding-dependent accident):
    // they are not eligible.  40 bits for complex128, 17 for complex64.
    const uint64_t wfloor = ((uint64_t)ldexp(mx, shift)) >> a.np_floor_bits;
    uint64_t local = 0;
    for (uint32_t k = k0; k < k0 + per && k < nb; ++k) {
      uint64_t w = (uint64_t)ldexp(pd[k], shift);
      if (w < wfloor) w = 0;
      local += w;
      cdf[k] = w;
    }
    uint64_t total;
    uint64_t run = block_exclusive<uint64_t>(local, ws64, &total);
    for (uint32_t k = k0; k < k0 + per && k < nb; ++k) {
      run += cdf[k];
      cdf[k] = run;
    }
    if (tid == 0) s_total = total;
    __syncthreads();
    // ---- successive draws without replacement ----
    const uint32_t rk = a.rank[item], es = a.eset_id[item];
    uint32_t taken = 0;
    for (uint32_t t = 0; t < m; ++t) {
      const uint64_t tot = s_total;
      if (tot == 0) break;  // fewer positive outcomes than requested (engine.py:551)
      if (tid == 0) {
        const Philox4 x = philox4x32_10(t, rk, a.stage, es, a.k0, a.k1);
        const uint64_t x64 = ((uint64_t)x.v[1] << 32) | x.v[0];
        const uint64_t r = __umul64hi(x64, tot);
        uint32_t lo = 0, hi = nb;  // first index with cdf > r
        while (lo < hi) {
          const uint32_t mid = (lo + hi) >> 1;
          if (cdf[mid] <= r) lo = mid + 1; else hi = mid;
        }
        s_pick = lo;
      }
      __syncthreads();
      const uint32_t pick = s_pick;
      const uint64_t w = cdf[pick] - (pick ? cdf[pick - 1] : 0ull);
      __syncthreads();  // everyone has read the weight before the tail moves
      for (uint32_t k = pick + tid; k < nb; k += SAMPLE_THREADS) cdf[k] -= w;
      if (tid == 0) { cnt[pick] = 1; s_total = tot - w; }
      ++taken;
      __syncthreads();
    }
    // ---- ordered emission of the chosen outcomes ----
    uint32_t mine = 0;
    for (uint32_t k = k0; k < k0 + per && k < nb; ++k) mine += cnt[k] != 0;
    uint32_t tot32;
    uint32_t pos = block_exclusive<uint32_t>(mine, ws32, &tot32);
    for (uint32_t k = k0; k < k0 + per && k < nb; ++k)
      if (cnt[k]) { a.slot_index[base + pos] = k; a.slot_count[base + pos] = a.child_mult; ++pos; }
    if (tid == 0) a.nnz[item] = tot32;
    (void)taken;
    __syncthreads();
  }
}

// Exhaustive harvest over a population vector that does not fit shared memory (final batches of
// 14-26 qubits: the data-harvesting regime of the paper).  One CTA per work item
// streams the 2^b reals twice: mass / minimum, then ordered threshold compaction in tiles of
// HB_TILE entries (each thread owns HB_PER consecutive entries of a tile, a block scan gives its
// output position).  Purely bandwidth-bound: 2 x 2^b x sizeof(real) read, 16 B per harvested record.
constexpr int HB_THREADS = 1024;  // one big CTA per item: 32 warps of loads in flight on its SM
constexpr int HB_PER = 8;
constexpr int HB_TILE = HB_THREADS * HB_PER;

__global__ void __launch_bounds__(HB_THREADS) harvest_big_kernel(const SampleArgs a) {
  const uint64_t nb = 1ull << a.b;
  __shared__ uint32_t ws32[33];
  __shared__ double redmin[HB_THREADS / 32], redsum[HB_THREADS / 32];
  __shared__ uint32_t s_base;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  for (uint64_t it = blockIdx.x; it < a.n_items; it += gridDim.x) {
    const uint64_t item = a.first_item + it;
    const float* pf = reinterpret_cast<const float*>(a.probs) + it * nb;
    const double* pdb = reinterpret_cast<const double*>(a.probs) + it * nb;
    auto at = [&](uint64_t k) -> double { return a.is_f32 ? (double)pf[k] : pdb[k]; };
    double rawmin = 1e300, csum = 0.0;
    for (uint64_t k = tid; k < nb; k += HB_THREADS) {
      double v = at(k);
      rawmin = fmin(rawmin, v);
      csum += v > 0.0 ? v : 0.0;
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
      rawmin = fmin(rawmin, __shfl_xor_sync(0xffffffffu, rawmin, d));
      csum += __shfl_xor_sync(0xffffffffu, csum, d);
    }
    if (lane == 0) { redmin[wid] = rawmin; redsum[wid] = csum; }
    __syncthreads();
    rawmin = redmin[0]; csum = redsum[0];
#pragma unroll
    for (int w = 1; w < HB_THREADS / 32; ++w) { rawmin = fmin(rawmin, redmin[w]); csum += redsum[w]; }
    const double ms = a.mass ? a.mass[it] : csum, mn = a.minv ? a.minv[it] : rawmin;
    uint32_t bad = 0;
    {
      double floor_mass = a.vanish;
      if (a.set_mass) {
        if (a.stage == 1) { floor_mass = a.vanish_stage1; if (tid == 0) a.set_mass[a.eset_row[item]] = ms; }
        else floor_mass = a.vanish * a.set_mass[a.eset_row[item]];
      }
      if (mn < a.neg_abs - a.neg_rel * ms) bad = PTSBE_ENUMERIC;
      else if (ms < floor_mass || !(ms > 0.0)) bad = PTSBE_EIMPOSSIBLE;
    }
    if (bad) {
      if (tid == 0) {
        a.nnz[item] = 0;
        atomicMin(a.flag, ((unsigned long long)a.eset_id[item] << 16) |
                              ((unsigned long long)(a.stage & 0xff) << 8) | bad);
        atomicAdd(a.flag_count, 1u);
      }
      __syncthreads();
      continue;
    }
    if (tid == 0) s_base = 0;
    __syncthreads();
    const uint32_t base = a.slot_off[item];
    for (uint64_t t0 = 0; t0 < nb; t0 += HB_TILE) {
      const uint64_t k0 = t0 + (uint64_t)tid * HB_PER;
      double pk[HB_PER];
      uint32_t mine = 0;
#pragma unroll
      for (int i = 0; i < HB_PER; ++i) {
        const uint64_t k = k0 + i;
        double v = k < nb ? at(k) : 0.0;
        v = v > 0.0 ? v / ms : 0.0;
        pk[i] = v;
        mine += (k < nb && v >= a.threshold);
      }
      uint32_t tot32;
      uint32_t pos = s_base + block_exclusive<uint32_t>(mine, ws32, &tot32);
#pragma unroll
      for (int i = 0; i < HB_PER; ++i) {
        if (k0 + i < nb && pk[i] >= a.threshold) {
          a.slot_index[base + pos] = (uint32_t)(k0 + i);
          a.slot_count[base + pos] = a.child_mult;
          a.slot_prob[base + pos] = pk[i];
          ++pos;
        }
      }
      __syncthreads();
      if (tid == 0) s_base += tot32;
      __syncthreads();
    }
    if (tid == 0) a.nnz[item] = s_base;
    __syncthreads();
  }
}

// Group-per-item variant for nb <= 2048 (b <= 11): same arithmetic, same results as
// sample_kernel, but no block-wide barriers.  GS lanes (8, 16 or 32) serve one item, 32 / GS
// items per warp in lockstep.  Each lane owns the nb/GS CONSECUTIVE outcomes
// [lane*per, lane*per+per); the row is staged through shared memory (padded by one slot per
// 32 so the strided per-lane reads are conflict-free), scanned serially in registers, and the
// lane totals are combined with one shuffle scan.  Most work items of the late stages draw one
// or two shots, so issue slots and latency per item -- not throughput of the draws -- matter.
constexpr int SG_THREADS = 256;

__device__ __forceinline__ uint32_t sw_pad(uint32_t k) { return k + (k >> 5); }

template <int GS>
__global__ void __launch_bounds__(SG_THREADS) sample_group_kernel(const SampleArgs a) {
  extern __shared__ __align__(16) unsigned char sm[];
  constexpr int GROUPS = SG_THREADS / GS;
  const uint32_t nb = 1u << a.b;
  const uint32_t padded = nb + (nb >> 5) + 1;
  const int lane = threadIdx.x & (GS - 1), grp = threadIdx.x / GS;
  uint64_t* cdf = reinterpret_cast<uint64_t*>(sm) + (size_t)grp * padded;
  uint32_t* cnt = reinterpret_cast<uint32_t*>(reinterpret_cast<uint64_t*>(sm) + (size_t)GROUPS * padded) +
                  (size_t)grp * padded;
  double* pd = reinterpret_cast<double*>(cdf);
  const uint32_t per = nb >= GS ? nb / GS : 1;           // outcomes per lane
  const int lanes_used = nb >= GS ? GS : (int)nb;
  const uint64_t n_groups = (uint64_t)gridDim.x * GROUPS;
  const uint64_t rounds = (a.n_items + n_groups - 1) / n_groups;

  // all groups of a warp run the same number of rounds (lockstep __syncwarp); a group past the
  // end redoes the last item with every global store masked off
  for (uint64_t r = 0; r < rounds; ++r) {
    uint64_t it = r * n_groups + (uint64_t)blockIdx.x * GROUPS + grp;
    const bool live = it < a.n_items;
    if (!live) it = a.n_items - 1;
    const uint64_t item = a.first_item + it;
    uint32_t m = a.mult[item];
    // ---- load, clamp, max / min / sum ----
    double mx = 0.0, rawmin = 1e300, csum = 0.0;
    if (a.is_f32) {
      const float* p = reinterpret_cast<const float*>(a.probs) + it * nb;
      for (uint32_t k = lane; k < nb; k += GS) {
        double v = (double)p[k]; rawmin = fmin(rawmin, v);
        v = v > 0.0 ? v : 0.0; pd[sw_pad(k)] = v; mx = fmax(mx, v); csum += v;
        cnt[sw_pad(k)] = 0;
      }
    } else {
      const double* p = reinterpret_cast<const double*>(a.probs) + it * nb;
      for (uint32_t k = lane; k < nb; k += GS) {
        double v = p[k]; rawmin = fmin(rawmin, v);
        v = v > 0.0 ? v : 0.0; pd[sw_pad(k)] = v; mx = fmax(mx, v); csum += v;
        cnt[sw_pad(k)] = 0;
      }
    }
#pragma unroll
    for (int d = GS / 2; d > 0; d >>= 1) {
      mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, d));
      rawmin = fmin(rawmin, __shfl_xor_sync(0xffffffffu, rawmin, d));
      csum += __shfl_xor_sync(0xffffffffu, csum, d);
    }
    // ---- guards (engine.py:447-448, 475-476, 484-485) ----
    uint32_t bad = 0;
    {
      const double ms = a.mass ? a.mass[it] : csum, mn = a.minv ? a.minv[it] : rawmin;
      double floor_mass = a.vanish;
      if (a.set_mass) {
        if (a.stage == 1) { floor_mass = a.vanish_stage1; if (lane == 0 && live) a.set_mass[a.eset_row[item]] = ms; }
        else floor_mass = a.vanish * a.set_mass[a.eset_row[item]];
      }
      if (mn < a.neg_abs - a.neg_rel * ms) bad = PTSBE_ENUMERIC;
      else if (ms < floor_mass) bad = PTSBE_EIMPOSSIBLE;
    }
    if (!bad && !(mx > 0.0)) bad = PTSBE_EIMPOSSIBLE;
    if (bad) {
      if (lane == 0 && live) {
        atomicMin(a.flag, ((unsigned long long)a.eset_id[item] << 16) |
                              ((unsigned long long)(a.stage & 0xff) << 8) | bad);
        atomicAdd(a.flag_count, 1u);
      }
      m = 0;      // no draws, no children; the group keeps in step with its warp
      mx = 1.0;
    }
    __syncwarp();
    // ---- exact fixed-point weights and their inclusive scan ----
    int ex;
    frexp(mx, &ex);
    const int shift = (62 - (int)a.b) - ex;
    const uint32_t k0 = lane * per;
    uint64_t run = 0;
    if (lane < lanes_used)
      for (uint32_t k = k0; k < k0 + per; ++k) {
        run += (uint64_t)ldexp(pd[sw_pad(k)], shift);
        cdf[sw_pad(k)] = run;  // same 8-byte slot as pd: lane-local inclusive sums
      }
    uint64_t incl = run;
#pragma unroll
    for (int d = 1; d < GS; d <<= 1) {
      const uint64_t o = __shfl_up_sync(0xffffffffu, incl, d, GS);
      if (lane >= d) incl += o;
    }
    const uint64_t total = __shfl_sync(0xffffffffu, incl, GS - 1, GS);
    const uint64_t base = incl - run;
    if (lane < lanes_used)
      for (uint32_t k = k0; k < k0 + per; ++k) cdf[sw_pad(k)] += base;
    __syncwarp();
    // ---- draws: outcome = #{k : cdf[k] <= r}, r = floor(x * W / 2^64) ----
    const uint32_t rk = a.rank[item], es = a.eset_id[item];
    for (uint32_t t = lane; t < m; t += GS) {
      const Philox4 x = philox4x32_10(t, rk, a.stage, es, a.k0, a.k1);
      const uint64_t x64 = ((uint64_t)x.v[1] << 32) | x.v[0];
      const uint64_t rr = __umul64hi(x64, total);
      uint32_t lo = 0, hi = nb;
      while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (cdf[sw_pad(mid)] <= rr) lo = mid + 1; else hi = mid;
      }
      atomicAdd(&cnt[sw_pad(lo)], 1u);
    }
    __syncwarp();
    // ---- ordered emission of the non-empty outcomes ----
    uint32_t mine = 0;
    if (lane < lanes_used && m)
      for (uint32_t k = k0; k < k0 + per; ++k) mine += cnt[sw_pad(k)] != 0;
    uint32_t pos = mine;
#pragma unroll
    for (int d = 1; d < GS; d <<= 1) {
      const uint32_t o = __shfl_up_sync(0xffffffffu, pos, d, GS);
      if (lane >= d) pos += o;
    }
    const uint32_t tot32 = __shfl_sync(0xffffffffu, pos, GS - 1, GS);
    pos -= mine;
    const uint32_t slot0 = a.slot_off[item];
    if (mine && live)
      for (uint32_t k = k0; k < k0 + per; ++k) {
        const uint32_t c = cnt[sw_pad(k)];
        if (c) { a.slot_index[slot0 + pos] = k; a.slot_count[slot0 + pos] = c; ++pos; }
      }
    if (lane == 0 && live) a.nnz[item] = tot32;
    __syncwarp();
  }
}

// ---- next-level construction ----------------------------------------------

struct ExpandArgs {
  // parent level
  const uint32_t* p_eset; const uint64_t* p_prefix; uint32_t p_n;
  const uint32_t* p_slot_off; const uint32_t* child_base;  // [p_n] exclusive scan of nnz
  const uint32_t* slot_index; const uint32_t* slot_count;
  // child level
  uint32_t* c_eset; uint32_t* c_parent; uint64_t* c_prefix; uint32_t* c_mult; uint32_t c_n;
  uint32_t words, offset, b;  // child prefix = parent prefix with b bits appended at qubit `offset`
  // Philox counters of the children (null at the final stage): rank = position inside the error set's run of
  // items, gid = global error-set id.  Items of one error set are contiguous at every level, so parent w's first
  // sibling is w - p_rank[w] and the error set's first child is child_base[w - p_rank[w]].
  const uint32_t* p_rank; const uint32_t* p_gid; uint32_t* c_rank; uint32_t* c_gid;
};

__global__ void expand_kernel(const ExpandArgs a) {
  const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= a.c_n) return;
  uint32_t lo = 0, hi = a.p_n;  // last parent with child_base <= c
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (a.child_base[mid] <= c) lo = mid; else hi = mid;
  }
  const uint32_t w = lo, pos = c - a.child_base[w];
  const uint32_t slot = a.p_slot_off[w] + pos;
  const uint32_t idx = a.slot_index[slot];
  a.c_eset[c] = a.p_eset[w];
  a.c_parent[c] = w;
  a.c_mult[c] = a.slot_count[slot];
  if (a.c_rank) {
    a.c_rank[c] = c - a.child_base[w - a.p_rank[w]];
    a.c_gid[c] = a.p_gid[w];
  }
  // qubit q -> word q/64, bit 63-(q%64); first batch qubit = MSB of idx (engine.py:489-490)
  for (uint32_t wd = 0; wd < a.words; ++wd) {
    uint64_t v = a.p_prefix[(size_t)wd * a.p_n + w];
    const int q0 = (int)wd * 64, q1 = q0 + 64;
    const int s = max(q0, (int)a.offset), e = min(q1, (int)(a.offset + a.b));
    for (int q = s; q < e; ++q) {
      const uint64_t bit = (idx >> (a.b - 1 - (q - a.offset))) & 1u;
      v |= bit << (63 - (q - q0));
    }
    a.c_prefix[(size_t)wd * a.c_n + c] = v;
  }
}

// Same result as expand_kernel, driven from the parent side: one thread per parent writes its
// (few) children.  Late stages have 1-2 children per parent, where the per-child binary search over
// tens of millions of scan entries (24 dependent loads) costs more than everything else in the
// compaction; early stages (hundreds of children per parent) keep the child-side kernel.
__global__ void expand_scatter_kernel(const ExpandArgs a, const uint32_t* __restrict__ nnz) {
  const uint32_t w = blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= a.p_n) return;
  const uint32_t n = nnz[w];
  if (n == 0) return;
  const uint32_t base = a.child_base[w], slot0 = a.p_slot_off[w], es = a.p_eset[w];
  uint64_t pv[4];
  const uint32_t words = min(a.words, 4u);
  for (uint32_t wd = 0; wd < words; ++wd) pv[wd] = a.p_prefix[(size_t)wd * a.p_n + w];
  uint32_t rank0 = 0, gid = 0;
  if (a.c_rank) {
    rank0 = base - a.child_base[w - a.p_rank[w]];
    gid = a.p_gid[w];
  }
  for (uint32_t k = 0; k < n; ++k) {
    const uint32_t c = base + k;
    const uint32_t idx = a.slot_index[slot0 + k];
    a.c_eset[c] = es;
    a.c_parent[c] = w;
    a.c_mult[c] = a.slot_count[slot0 + k];
    if (a.c_rank) {
      a.c_rank[c] = rank0 + k;
      a.c_gid[c] = gid;
    }
    for (uint32_t wd = 0; wd < words; ++wd) {
      uint64_t v = pv[wd];
      const int q0 = (int)wd * 64, q1 = q0 + 64;
      const int s = max(q0, (int)a.offset), e = min(q1, (int)(a.offset + a.b));
      for (int q = s; q < e; ++q) {
        const uint64_t bit = (idx >> (a.b - 1 - (q - a.offset))) & 1u;
        v |= bit << (63 - (q - q0));
      }
      a.c_prefix[(size_t)wd * a.c_n + c] = v;
    }
  }
}


__global__ void iota_kernel(uint32_t* p, uint32_t n, uint32_t add) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = i + add;
}

// Pre-trajectory sampling on the device (reference draw_realization / presample_errors,
// engine.py:232-281): one Kraus/Pauli index per (error set, gate site), drawn from the
// site's outcome distribution with a counter-based uniform -- Philox counter
// (site, GLOBAL error-set id, 'PRES', 0), key = seed -- so an error set's realisation does not
// depend on the batch, the rank or the order it is generated in.  site_cdf holds, per site, the
// inclusive cumulative probabilities of its outcomes (index 0 = no error).
constexpr uint32_t PRESAMPLE_TAG = 0x50524553u;  // "PRES"

__global__ void presample_kernel(const double* __restrict__ site_cdf, const uint32_t* __restrict__ site_off,
                                 uint32_t g, uint64_t n_sets, uint32_t first_id, uint32_t k0, uint32_t k1,
                                 uint8_t* __restrict__ out) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_sets * g) return;
  const uint32_t e = (uint32_t)(i / g), s = (uint32_t)(i - (uint64_t)e * g);
  const uint32_t a = site_off[s], b = site_off[s + 1];
  uint32_t idx = 0;
  if (b - a > 1) {
    const Philox4 x = philox4x32_10(s, first_id + e, PRESAMPLE_TAG, 0u, k0, k1);
    const uint64_t x64 = ((uint64_t)x.v[1] << 32) | x.v[0];
    const double u = (double)(x64 >> 11) * (1.0 / 9007199254740992.0);
    while (idx + 1 < b - a && site_cdf[a + idx] <= u) ++idx;
  }
  out[i] = (uint8_t)idx;
}

}  // namespace ptsbe
