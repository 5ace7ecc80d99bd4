// Fused per-item steps + per-qubit descent, ONE LANE PER DRAW (complex64, Hermitian cut).
//
// lane_descent_kernel (lane.cuh) serves a draw with a 4-lane group: the item's projection vector v is
// rebuilt per draw through the generic gather tables of the program's last step (32 shared-memory
// loads per lane), every tree level costs 4 chunk loads, 16 FMAs and 2 shuffles per lane, and a warp has 8
// draws in flight.  When the cut vector is x (x) conj(x) with x of DX complex entries (the ket and bra
// halves of the cut are mirror images: every projection-form stage of cfg2), the probability of a tree
// node is the Hermitian form  p = x^H H_node x  and needs, in packed real form (lane.cuh HERM),
//     w = { |x_p|^2 ; Re(x_p conj x_q), Im(x_p conj x_q)  for p < q }      (DX^2 reals, this order)
// Here one lane owns one (item, draw): it loads x (DX shared-memory loads), forms w in REGISTERS with
// compile-time indices, and walks the tree with DX^2 / 4 16-byte row loads and DX^2 FMAs per level -- no
// gather tables, no shuffles, 32 draws in flight per warp.  The tree columns are packed in the canonical
// order above by herm_pack_kernel (Program::herm_canon gives position and sign of every packed slot).
// Same Philox counters, guards, slot layout and dedup as lane_descent_kernel; replaces, like it,
// rng.multinomial of reference engine.py:519 plus the marginal contraction of engine.py:417-450 for the
// stage's per-item steps.
//
// CHAIN: the per-item steps before the outer product are a chain of vector-matrix products
//     x_1 = r . T_1[bits],  x_2 = x_1 . T_2[bits],  ...      (r: record of an earlier pass, T_s: transfer
// matrices sliced out of the error set's class-0 record by prefix bits -- the matrix-product-state form the
// cut planner produces).  A lane that owns an item would read its own DX x DX matrix: 32 lanes, 32 different
// matrices, every load instruction touching 32 cache lines.  Here a group of DX lanes serves one item, lane c
// computes component c of the product from rows that the group reads as contiguous blocks (the compiler stores
// records in consumer order: [slicing bits][contracted][surviving]), the intermediate vectors stay in registers
// and only x is handed to the draw phase through shared memory.  Same multiply-add order as lane_run.
#pragma once
#include "lane.cuh"

namespace ptsbe {

constexpr int LN_CHAIN_MAX = 4;  // vector-matrix steps a CHAIN kernel accepts

template <int DX, bool CHAIN>
__global__ void __launch_bounds__(LN_THREADS, 2) lane_descent_x_kernel(const LaneDescentArgs a) {
  using R = float;
  using C = float2;
  constexpr int D = DX * DX;                       // reals per packed column
  constexpr int NQ = D / 4 > 0 ? D / 4 : 1;        // 16-byte chunks per column
  constexpr uint32_t PITCH = NQ + 1;               // one chunk of padding staggers the rows over the banks
  extern __shared__ __align__(16) unsigned char ln_smem[];
  const ExecArgs& e = a.l.e;
  const DescentArgs& d = a.d;
  const LaneLayout L = lane_layout(e.n_steps, a.l.n_leaves, a.l.n_table_words, a.l.n_levels, e.arena_fast, e.words,
                                   (uint32_t)sizeof(C), a.l.ast ? a.l.ast : (uint32_t)LN_AST);
  const LaneCtx<R> cx = lane_setup<R>(a.l, ln_smem, L);
  const uint32_t N = 1u << d.b;
  double* mass_s = reinterpret_cast<double*>(ln_smem + L.end);                 // [LN_THREADS]
  uint32_t* cum_s = reinterpret_cast<uint32_t*>(mass_s + LN_THREADS);          // [LN_THREADS]
  uint32_t* slot0_s = cum_s + LN_THREADS;
  uint32_t* eset_s = slot0_s + LN_THREADS;
  uint32_t* bad_s = eset_s + LN_THREADS;
  uint32_t* rank_s = bad_s + LN_THREADS;
  uint32_t* gid_s = rank_s + LN_THREADS;
  uint32_t* dyn_s = gid_s + LN_THREADS;                                        // CHAIN: [LN_CHAIN_MAX][LN_THREADS]
  const int tid = threadIdx.x, lane32 = tid & 31, warp = tid >> 5;
  const bool WR = a.warp_runs != 0;  // every warp walks its own runs with a private table (lane.cuh)
  float4* table = reinterpret_cast<float4*>(dyn_s + (CHAIN ? LN_CHAIN_MAX * LN_THREADS : 0)) +
                  (WR ? (size_t)warp * N * PITCH : 0);  // [N][PITCH]
  __shared__ uint32_t s_end;
  const uint32_t wbase = warp * 32;
  const float4* TREE = reinterpret_cast<const float4*>(d.tree);
  uint32_t loaded = 0xffffffffu;
  __syncthreads();  // program image complete
  const LaneStep last = lane_decode(cx.steps, cx.tables, e.n_steps - 1);

  // packed Hermitian vector of the item in warp slot i, in registers
  auto load_w = [&](uint32_t i, float (&w)[D < 4 ? 4 : D]) {
    const uint32_t slot = wbase + i;
    LaneOp<C> A, B;
    if constexpr (CHAIN) {
      A.p = cx.arena_w + i;  // x of the item in warp slot i: element p at [p * ast + i]
      A.stride = cx.ast;
    } else {
      lane_operands<R>(cx, last, slot, eset_s[slot], A, B);
    }
    float xr[DX], xi[DX];
#pragma unroll
    for (int p = 0; p < DX; ++p) {
      const C x = A.p[p * A.stride];
      xr[p] = x.x;
      xi[p] = x.y;
    }
#pragma unroll
    for (int p = 0; p < DX; ++p) w[p] = fmaf(xr[p], xr[p], xi[p] * xi[p]);
    int k = DX;
#pragma unroll
    for (int p = 0; p < DX; ++p)
#pragma unroll
      for (int q = p + 1; q < DX; ++q) {
        w[k++] = fmaf(xr[p], xr[q], xi[p] * xi[q]);    // Re(x_p conj x_q)
        w[k++] = fmaf(xi[p], xr[q], -xr[p] * xi[q]);   // Im(x_p conj x_q)
      }
#pragma unroll
    for (int z = D; z < 4; ++z) w[z] = 0.f;
  };
  // four independent accumulators, added in a fixed order: the value does not depend on the lane
  auto dot = [&](const float (&w)[D < 4 ? 4 : D], const float4* row) -> R {
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const float4 m = row[q];
      float s = acc[q & 3];
      s = fmaf(w[4 * q], m.x, s);
      s = fmaf(w[4 * q + 1], m.y, s);
      s = fmaf(w[4 * q + 2], m.z, s);
      s = fmaf(w[4 * q + 3], m.w, s);
      acc[q & 3] = s;
    }
    return (acc[0] + acc[1]) + (acc[2] + acc[3]);
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
          const float4* src = TREE + (size_t)er * N * NQ;
          for (uint32_t x = lane32; x < N * NQ; x += 32) table[(x / NQ) * PITCH + (x % NQ)] = __ldg(src + x);
          loaded = er;
        }
        __syncwarp();
      } else {
        if (tid == 0) s_end = t1;
        __syncthreads();
        for (uint32_t i = pos + 1 + tid; i < t1; i += LN_THREADS)
          if (d.eset[d.first_item + i] != er) { atomicMin(&s_end, i); break; }
        if (er != loaded) {
          const float4* src = TREE + (size_t)er * N * NQ;
          for (uint32_t x = tid; x < N * NQ; x += LN_THREADS) table[(x / NQ) * PITCH + (x % NQ)] = __ldg(src + x);
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
        if constexpr (CHAIN) {
          // per item: offset of its transfer matrix inside the record, step by step (prefix-bit slicing)
          for (uint32_t s = 0; s + 1 < e.n_steps; ++s) {
            const LaneStep t = lane_decode(cx.steps, cx.tables, s);
            uint32_t add_a = 0, add_b = 0;
            if (t.flags & 8u) {
              const uint32_t* dt = t.dyn;
              const uint32_t na = dt[0];
              for (uint32_t z = 0; z < na; ++z)
                if (cx.bit(dt[1 + 2 * z], tid)) add_a += dt[2 + 2 * z];
              dt += 1 + 2 * na;
              const uint32_t nb = dt[0];
              for (uint32_t z = 0; z < nb; ++z)
                if (cx.bit(dt[1 + 2 * z], tid)) add_b += dt[2 + 2 * z];
            }
            dyn_s[s * LN_THREADS + tid] = (t.flags & 32u) ? add_b : add_a;
          }
          __syncwarp();
          // DX lanes per item, 32 / DX items per round: lane c owns component c
          constexpr int G = 32 / DX;
          const uint32_t grp = lane32 / DX, c = lane32 % DX;
          for (uint32_t sub = 0; sub < (uint32_t)DX; ++sub) {
            const uint32_t i = sub * G + grp, slot = wbase + i;
            C vec[8], acc;
            acc.x = acc.y = 0.f;
            for (uint32_t s = 0; s + 1 < e.n_steps; ++s) {
              const LaneStep t = lane_decode(cx.steps, cx.tables, s);
              const bool vec_a = (t.flags & 32u) != 0;  // which operand is the vector
              const uint32_t mk = vec_a ? t.s0.z : t.s0.x, mr = vec_a ? t.s0.w : t.s0.y;
              const uint32_t* lo_m = vec_a ? t.loB : t.loA;
              const uint32_t* k_m = vec_a ? t.kB : t.kA;
              const bool cj_v = vec_a ? (t.flags & 1u) : (t.flags & 2u);
              const bool cj_m = vec_a ? (t.flags & 2u) : (t.flags & 1u);
              if (s == 0) {
                const uint32_t vk = vec_a ? t.s0.x : t.s0.z, vr = vec_a ? t.s0.y : t.s0.w;
                const LevelDev& lv = cx.levels[vk - 1];
                const C* vp = reinterpret_cast<const C*>(lv.ext) + (size_t)cx.anc[(vk - 1) * LN_THREADS + slot] * lv.ext_rec + vr;
                if (!((vr | lv.ext_rec) & 1u)) {
                  const float4* vp4 = reinterpret_cast<const float4*>(vp);
#pragma unroll
                  for (int k = 0; k < 4; ++k)
                    if (2 * k < (int)t.kn) {
                      const float4 q = __ldg(vp4 + k);
                      vec[2 * k].x = q.x; vec[2 * k].y = q.y; vec[2 * k + 1].x = q.z; vec[2 * k + 1].y = q.w;
                    }
                } else {
#pragma unroll
                  for (int k = 0; k < 8; ++k)
                    if (k < (int)t.kn) vec[k] = __ldg(vp + k);
                }
              } else {
                // the previous product, gathered from the group's lanes
#pragma unroll
                for (int k = 0; k < DX; ++k) {
                  vec[k].x = __shfl_sync(0xffffffffu, acc.x, grp * DX + k);
                  vec[k].y = __shfl_sync(0xffffffffu, acc.y, grp * DX + k);
                }
              }
              const LevelDev& lm = cx.levels[mk - 1];
              const C* mp = reinterpret_cast<const C*>(lm.ext) + (size_t)cx.anc[(mk - 1) * LN_THREADS + slot] * lm.ext_rec +
                            mr + dyn_s[s * LN_THREADS + slot] + lo_m[c];
              acc.x = acc.y = 0.f;
#pragma unroll
              for (int k = 0; k < 8; ++k)
                if (k < (int)t.kn) {
                  C m = __ldg(mp + k_m[k]);
                  C v = vec[k];
                  if (cj_m) m.y = -m.y;
                  if (cj_v) v.y = -v.y;
                  if (vec_a) cmac_s<false, false>(acc, v, m);
                  else cmac_s<false, false>(acc, m, v);
                }
            }
            cx.arena_w[c * cx.ast + i] = acc;
          }
          __syncwarp();
        } else {
          __syncwarp();
          lane_run<R>(cx, 0, e.n_steps - 1, es_row, nullptr, false);
        }
        const uint32_t m = live ? d.mult[item] : 0u;
        slot0_s[tid] = d.slot_off[item];
        rank_s[tid] = d.rank[item];
        gid_s[tid] = d.eset_id[item];
        bad_s[tid] = 0;
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
        // ---- phase B: one (item, draw) per lane and round.  Round 0: the warp's items, mass (guards of
        // reference engine.py:445-450, 475-476) and draw 0; later rounds: 32 of the remaining draws each ----
        const uint32_t n_live = min(32u, end - w0);
        const uint32_t rounds = 1 + (total + 31) / 32;
        for (uint32_t rd = 0; rd < rounds; ++rd) {
          const bool first = rd == 0;  // warp-uniform
          bool active;
          uint32_t i, t;
          if (first) {
            active = (uint32_t)lane32 < n_live;
            i = active ? (uint32_t)lane32 : n_live - 1;
            t = 0;
          } else {
            const uint32_t d0 = (rd - 1) * 32 + lane32;
            active = d0 < total;
            const uint32_t dr = active ? d0 : total - 1;
            uint32_t lo = 0, hi = 31;  // smallest i with cum[i] > dr
            while (lo < hi) {
              const uint32_t mid = (lo + hi) >> 1;
              if (cum_s[wbase + mid] > dr) hi = mid; else lo = mid + 1;
            }
            i = lo;
            t = 1 + dr - (i ? cum_s[wbase + i - 1] : 0u);
          }
          float w[D < 4 ? 4 : D];
          load_w(i, w);
          uint32_t bad = 0;
          R mass;
          if (first) {
            mass = dot(w, table);
            if (!((double)mass >= floor_mass) || !(mass > R(0))) bad = PTSBE_EIMPOSSIBLE;
          } else {
            mass = (R)mass_s[wbase + i];
            bad = bad_s[wbase + i] == PTSBE_EIMPOSSIBLE ? PTSBE_EIMPOSSIBLE : 0u;
          }
          uint32_t node = 0;
          if (!bad) {
            // inverse-CDF walk down the tree of conditional marginals: same uniform, same decisions as
            // lane_descent_kernel
            const R tol = (R)(d.neg_abs - d.neg_rel * (double)mass);
            const Philox4 x = philox4x32_10(t, rank_s[wbase + i], d.stage, gid_s[wbase + i], d.k0, d.k1);
            const uint64_t x64 = ((uint64_t)x.v[1] << 32) | x.v[0];
            R p = mass;
            R r = (R)((double)(x64 >> 11) * (1.0 / 9007199254740992.0)) * mass;  // u in [0, 1)
            if (!(r < mass)) r = nextafterf(mass, 0.0f);                          // u rounded up to 1.0f
            for (uint32_t lvl = 1; lvl <= d.b; ++lvl) {
              R pl = dot(w, table + (size_t)((1u << (lvl - 1)) + node) * PITCH);
              if (pl < tol || p - pl < tol) bad = PTSBE_ENUMERIC;
              pl = fminf(fmaxf(pl, R(0)), p);
              if (r < pl) { node = 2 * node; p = pl; }
              else { node = 2 * node + 1; r -= pl; p -= pl; }
            }
          }
          if (active) {
            if (first) mass_s[wbase + i] = (double)mass;
            if (bad) {
              bad_s[wbase + i] = bad;
            } else {
              const uint32_t sl = slot0_s[wbase + i] + t;
              d.slot_index[sl] = node;
              d.slot_count[sl] = 1;
            }
          }
          if (first) __syncwarp();  // masses and flags visible to the later rounds
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

}  // namespace ptsbe
