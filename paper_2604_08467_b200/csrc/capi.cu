// C-ABI of libptsbe_b200.so (include/ptsbe_b200.h) and the host-side run
// driver: per-stage hoist passes, marginal pass, sampler, order-preserving
// compaction into the next stage's work list, final histogram.
//
// Replaces the fan-out loop of run_ptsbe (engine.py:885-906) and
// sample_proportional (engine.py:493-524): the loop over error sets and the
// loop over sorted prefixes become the batch axis of every launch.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <map>
#include <memory>
#include <mutex>
#include <set>
#include <tuple>

#include "common.cuh"
#include "descent.cuh"
#include "executor.cuh"
#include "histogram.cuh"
#include "lane.cuh"
#include "lane_x.cuh"
#include "project.cuh"
#include "project_tc.cuh"
#include "sampler.cuh"
#include "scan.cuh"

namespace ptsbe {

thread_local std::string g_last_error;
thread_local uint64_t g_launches = 0;
thread_local Workspace* g_ws = nullptr;

struct Program {
  ptsbe_program_desc d;
  DevBuf leaves, steps, tables;
  DevBuf memo_ptr, memo_idx, memo;  // variant-0 memo (class-0 programs): site -> steps CSR, values
  bool memo_ready = false;
  int blocks_per_sm = 0;  // resolved lazily per (program, item_bytes)
  // lane-per-item interpreter (lane.cuh): program small enough to run one thread per work item;
  // lane_fused: additionally its last step alone produces the projection vector
  bool lane_ok = false, lane_fused = false;
  int lane_blocks_per_sm = 0;
  // class-0 hoist program that can run one thread per error set with a global-memory arena (lane.cuh BIG)
  bool lane_big_ok = false;
  int lane_big_blocks_per_sm = 0;
  double macs = 0;  // complex multiply-adds of one execution (sum over steps of outputs x contracted entries)
  bool tiled = false;  // most multiply-adds sit in large separable steps: register-tiled kernel variant
  // projection vector is x (x) conj(x): Hermitian-packed tree columns (lane.cuh HERM)
  bool herm = false;
  std::vector<uint32_t> herm_map_host;
  DevBuf herm_map;
  // ... with x of herm_dx in {2, 4, 8} complex entries: lane-per-draw kernel (lane_x.cuh) over tree columns in
  // canonical order; herm_canon[s] = position | sign << 31 of packed slot s
  uint32_t herm_dx = 0;
  std::vector<uint32_t> herm_canon_host;
  DevBuf herm_canon;
  // ... and every step before the outer product is a vector-matrix product over a record (lane_x.cuh CHAIN)
  bool lane_chain = false;
};

}  // namespace ptsbe

using namespace ptsbe;

struct ptsbe_plan {
  int device = 0;
  uint32_t dtype = 0, n = 0, g = 0, f = 0, words = 1;
  std::vector<uint32_t> sizes, offsets;        // offsets[j] = qubits measured before stage j+1
  std::vector<std::vector<Program>> programs;  // [stage-1][pass]
  DevBuf pool;
  cudaStream_t stream = nullptr;
  int sm_count = 148;
  size_t elem = 8;
  std::mutex mu;
  // tunables (environment overrides for experiments)
  size_t probs_budget = 256ull << 20;  // bytes of marginal buffer per sub-batch
  size_t vec_budget = 512ull << 20;    // bytes of per-item vectors per sub-batch (descent stages)
  uint32_t lane = 1;                   // lane-per-item interpreter / fused descent (lane.cuh)
  uint32_t tc_project = 1;             // complex64 projection on tcgen05 tensor cores (project_tc.cuh)
  uint32_t lane_x = 1;                 // lane-per-draw fused descent for Hermitian cuts (lane_x.cuh)
  uint32_t lane_chain = 0;             // ... with the vector-matrix chain served by lane groups (lane_x.cuh CHAIN);
                                       // pays only with PTSBE_RECORD_LAYOUT=1
  uint32_t tile_min = 128;             // CTA-per-item programs: 4 x 4 register tiles for separable steps with at
                                       // least this many tiles, 2 x 2 below (keeps the CTA busy on mid-size steps)
  uint32_t lane_tiny = 16;             // lane interpreter: steps of <= this many multiply-adds use the generic loop
  uint32_t descent_tile_max = 2048;    // fused descent: most consecutive work items a CTA takes at a time
  uint32_t tree_herm = 1;              // small descent tables: trees + Hermitian packing in one kernel
  uint32_t tc_steps = 0;               // opt-in (slower): large separable steps of CTA-per-item programs on tcgen05
                                       // tensor cores (executor.cuh tc_step, TF32 x3)
  uint32_t tiled_plain = 1;            // CTA-per-item programs without a memo (per-prefix passes of the dense
                                       // regime, cfg3r1) also run their large steps with register tiles
  uint32_t warp_runs = 1;              // fused descent: a private tree table per warp when error sets bring ...
  uint32_t warp_run_len = 512;         // ... fewer than this many work items each on average (lane.cuh warp_runs)
  uint32_t stage_image = 1;            // lane-group class-0 programs keep their image in shared memory ...
  uint32_t stage_image_max = 4096;     // ... for batches of at most this many error sets (executor.cuh STAGED)
  bool raw_final = true;               // PTSBE_RAW_FINAL=0: per-item merge of the final stage's draws even for merged output
  uint32_t lane_big_min = 3072;        // class-0 hoists over at least this many error sets run one thread per
                                       // error set with a global-memory arena (lane.cuh BIG).  With the passes of all
                                       // stages concurrent on side streams the crossover against the lane-group
                                       // kernel sits near 3000 error sets on cfg5 (16384 when they ran one by one)
  uint32_t descent = 1;                // per-qubit descent sampler for low-multiplicity stages
  double descent_mult = 4.0;           // ... used when shots / unique prefixes of the stage <= this
  // per stage: 1 descent, 0 flat, -1 decide per chunk (ptsbe_plan_set_stage_samplers)
  std::vector<int> stage_descent;
  DevBuf site_variants;                // [g] u8 variants per site, or empty (no index validation)
  // the class-0 passes of stages 2..f depend on the error sets only, so they are launched up front on side
  // streams and overlap each other and stage 1; see run_chunk (measured a gain at every batch size: the passes
  // are latency-bound, small batches because they do not fill the GPU, large ones because they wait on L2)
  uint32_t prelaunch = 1, prelaunch_max = 0xffffffffu;
  uint32_t side_priority = 1;
  double eager_work_max = 8e9;         // complex multiply-adds per launch above which a hoist pass is not run early
  std::vector<cudaStream_t> side;
  uint64_t chunk_shots = 1ull << 26;
  size_t ext_budget = 48ull << 30;
  double vanish = 1e-12, neg_abs = -1e-12, neg_rel = 0.0, vanish_stage1 = 1e-30;
  // workspaces of destroyed batches: ptsbe_sample() creates a batch per call, and re-creating
  // multi-GB slabs (cudaMalloc / cudaFree) per call would dominate its wall time
  std::vector<std::unique_ptr<Workspace>> ws_cache;
  std::unique_ptr<Workspace> take_workspace() {
    if (ws_cache.empty()) return std::unique_ptr<Workspace>(new Workspace);
    // hand out the largest first: ws_tmp is requested before ws_out and needs more
    size_t best = 0;
    for (size_t i = 1; i < ws_cache.size(); ++i)
      if (ws_cache[i]->reserved() > ws_cache[best]->reserved()) best = i;
    std::unique_ptr<Workspace> w = std::move(ws_cache[best]);
    ws_cache.erase(ws_cache.begin() + best);
    w->reset();
    return w;
  }
  void give_workspace(std::unique_ptr<Workspace> w) {
    if (!w) return;
    if (ws_cache.size() < 4) ws_cache.push_back(std::move(w));
  }
};

namespace ptsbe {

// Host buffers handed to the caller (histograms).  Large ones are page-locked, so the
// device->host copy runs at PCIe rate instead of through the driver's bounce buffers, and
// are recycled between calls (pinning hundreds of MB costs as much as the copy): ptsbe_free()
// puts them back here.  Small ones are plain malloc.
struct HostPool {
  struct Ent { void* p; size_t cap; bool busy; };
  std::mutex mu;
  std::vector<Ent> ents;
  static constexpr size_t kMinPinned = 1ull << 20, kKeepBytes = 8ull << 30;
  void* get(size_t bytes) {
    if (bytes < kMinPinned) return malloc(std::max<size_t>(bytes, 8));
    std::lock_guard<std::mutex> lock(mu);
    int best = -1;
    for (size_t i = 0; i < ents.size(); ++i)
      if (!ents[i].busy && ents[i].cap >= bytes && (best < 0 || ents[i].cap < ents[best].cap)) best = (int)i;
    if (best >= 0) { ents[best].busy = true; return ents[best].p; }
    const size_t cap = (bytes + bytes / 8 + (1ull << 21) - 1) & ~((1ull << 21) - 1);
    void* p = nullptr;
    if (cudaHostAlloc(&p, cap, cudaHostAllocDefault) != cudaSuccess) {
      cudaGetLastError();
      return malloc(bytes);  // not pinned: slower copy, same result
    }
    ents.push_back(Ent{p, cap, true});
    return p;
  }
  bool put(void* p) {  // false: not one of ours
    std::lock_guard<std::mutex> lock(mu);
    size_t idle = 0;
    int hit = -1;
    for (size_t i = 0; i < ents.size(); ++i) {
      if (ents[i].p == p) hit = (int)i;
      else if (!ents[i].busy) idle += ents[i].cap;
    }
    if (hit < 0) return false;
    if (idle + ents[hit].cap > kKeepBytes) {
      cudaFreeHost(p);
      ents.erase(ents.begin() + hit);
    } else {
      ents[hit].busy = false;
    }
    return true;
  }
};
static HostPool g_host_pool;

// cudaFuncSetAttribute and occupancy are PER DEVICE: plans may live on several GPUs of one process,
// so the opt-in to > 48 KB of dynamic shared memory and the occupancy figures are remembered per
// (device, kernel[, shared-memory size]) under a lock, never in a process-wide flag.
static void opt_in_smem(const void* fn, int bytes) {
  static std::mutex mu;
  static std::set<std::pair<int, const void*>> done;
  int dev = 0;
  CK(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  if (done.count({dev, fn})) return;
  CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  done.insert({dev, fn});
}

static int cached_occupancy(const void* fn, int threads, size_t smem) {
  static std::mutex mu;
  static std::map<std::tuple<int, const void*, size_t>, int> memo;
  int dev = 0;
  CK(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  auto key = std::make_tuple(dev, fn, smem);
  auto it = memo.find(key);
  if (it != memo.end()) return it->second;
  int nb = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, threads, smem));
  nb = std::max(nb, 1);
  memo[key] = nb;
  return nb;
}

static size_t env_size(const char* name, size_t dflt) {
  const char* v = getenv(name);
  if (!v || !*v) return dflt;
  return (size_t)strtoull(v, nullptr, 10);
}

struct ExecLaunch {
  uint32_t desc_off, desc_cap = 0;
  unsigned grid, block;
  size_t smem;
  uint32_t item_bytes;
  uint32_t groups_per_block;
  bool staged = false;  // lane-group program with its image in shared memory (executor.cuh STAGED)
  bool tc = false;      // large separable steps on the tensor cores (executor.cuh TC)
  uint32_t tc_off = 0;
  void (*kern)(ExecArgs) = nullptr;
};

template <typename R>
static void (*pick_exec_kernel(uint32_t gs, bool memo, bool tiled, bool staged, bool tc))(ExecArgs) {
  if (gs == 8) return staged ? exec_kernel<R, 8, false, false, true> : exec_kernel<R, 8, false>;
  if (gs == 16) return staged ? exec_kernel<R, 16, false, false, true> : exec_kernel<R, 16, false>;
  if (gs == 32) return staged ? exec_kernel<R, 32, false, false, true> : exec_kernel<R, 32, false>;
  if constexpr (sizeof(R) == 4) {
    if (tc && tiled) return memo ? exec_kernel<R, 0, true, true, false, true> : exec_kernel<R, 0, false, true, false, true>;
  }
  if (memo) return tiled ? exec_kernel<R, 0, true, true> : exec_kernel<R, 0, true>;
  return tiled ? exec_kernel<R, 0, false, true> : exec_kernel<R, 0, false>;
}

template <typename R>
static ExecLaunch configure_exec(ptsbe_plan* pl, Program& pr, uint32_t n_items) {
  using C = typename CxT<R>::type;
  ExecLaunch L;
  const ptsbe_program_desc& d = pr.d;
  size_t ib = (size_t)d.arena_fast_elems * sizeof(C) + (size_t)pl->words * 8 + 4ull * (d.level + 1);
  ib = (ib + 15) & ~size_t(15);
  L.item_bytes = (uint32_t)ib;
  const uint32_t gs = d.threads_per_item;  // 8 / 16 / 32: sub-warp groups; larger: one CTA per item
  const bool warp = gs <= 32;
  // class-0 lane-group programs over small batches are bound by the latency of their dependent
  // program reads: keep the image in shared memory when it fits beside the groups' arenas
  const size_t image = (((size_t)d.n_steps * STEP_WORDS + (size_t)d.n_leaves * LEAF_WORDS + d.n_table_words) * 4 + 15) & ~size_t(15);
  L.staged = warp && pl->stage_image && d.level == 1 && d.n_steps >= 32 && image <= 120 * 1024 &&
             n_items <= pl->stage_image_max && ib * (32 / gs) + 1024 + image <= 200 * 1024;
  if (warp) {
    uint32_t block = 256;
    const size_t extra = L.staged ? image : 0;
    while (block > 32 && ib * (block / gs) + 1024 + extra > 200 * 1024) block >>= 1;
    L.groups_per_block = block / gs;
    L.block = block;
  } else {
    L.groups_per_block = 1;
    L.block = gs;
  }
  L.smem = ib * L.groups_per_block + 1024;
  const bool memo = !warp && d.memo_elems;
  if (memo) L.smem += memo_smem_bytes(d.n_steps);
  L.desc_off = 0;
  if (!warp) {  // staged step descriptors
    L.desc_off = (uint32_t)L.smem;
    L.desc_cap = std::min<uint32_t>(d.n_steps, (uint32_t)env_size("PTSBE_DESC_CAP", DESC_CAP));
    L.smem += (size_t)L.desc_cap * STEP_WORDS * 4;
    if (memo) L.smem += (size_t)L.desc_cap * 2 * sizeof(void*);  // pre-resolved leaf operands
  }
  if (L.staged) {  // the image follows the groups and the reduction scratch
    L.desc_off = (uint32_t)L.smem;
    L.smem += image;
  }
  const bool tiled = pr.tiled && (memo || pl->tiled_plain);
  L.tc = !warp && tiled && pl->tc_steps && sizeof(R) == 4;
  if (L.tc) {  // operand tiles, mbarrier and TMEM slot of the tensor-core steps
    L.tc_off = (uint32_t)L.smem;
    L.smem += TCS_BYTES;
  }
  if (L.smem > 227 * 1024)
    throw Failure(PTSBE_ERESOURCE, "stage program needs more shared memory than one SM has");
  void (*kern)(ExecArgs) = pick_exec_kernel<R>(gs, memo, tiled, L.staged, L.tc);
  L.kern = kern;
  int per_sm;
  if (L.staged) {
    opt_in_smem((const void*)kern, 227 * 1024);
    per_sm = cached_occupancy((const void*)kern, (int)L.block, L.smem);
  } else {
    if (pr.blocks_per_sm == 0) {
      CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
      int nb = 0;
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, (int)L.block, L.smem));
      pr.blocks_per_sm = std::max(nb, 1);
    }
    per_sm = pr.blocks_per_sm;
  }
  const uint64_t need = (n_items + L.groups_per_block - 1) / L.groups_per_block;
  const uint64_t cap = (uint64_t)pl->sm_count * per_sm;
  L.grid = (unsigned)std::max<uint64_t>(1, std::min(need, cap));
  return L;
}

template <typename R>
static void launch_exec(ptsbe_plan* pl, Program& pr, uint32_t mode, const LevelDev* levels_dev,
                        const uint8_t* kraus_dev, uint32_t first, uint32_t n_items, void* out,
                        double* mass, double* minv, uint32_t vec_stride, uint32_t vec_row);

// Variant-0 memo of a class-0 program: one pass of the interpreter over a single pseudo work
// item whose Kraus-index row is all zeros, every step writing its value to the memo.
template <typename R>
static void build_memo(ptsbe_plan* pl, Program& pr) {
  cudaStream_t st = pl->stream;
  WorkspaceScope persistent(nullptr);  // the memo outlives the run whose workspace is installed
  pr.memo.alloc((size_t)pr.d.memo_elems * pl->elem + 64, st);
  const size_t pfx_at = 64 + (((size_t)pl->g + 7) & ~size_t(7));
  DevBuf zeros(pfx_at + 8 * pl->words, st), lvl(2 * sizeof(LevelDev), st);
  CK(cudaMemsetAsync(zeros.p, 0, zeros.bytes, st));
  LevelDev table[2];
  memset(table, 0, sizeof table);
  table[1].eset = zeros.as<uint32_t>();
  table[1].parent = zeros.as<uint32_t>();
  table[1].prefix = reinterpret_cast<const uint64_t*>(zeros.as<char>() + pfx_at);
  table[1].n = 1;
  CK(cudaMemcpyAsync(lvl.p, table, sizeof table, cudaMemcpyHostToDevice, st));
  CK(cudaStreamSynchronize(st));  // `table` is a stack object
  launch_exec<R>(pl, pr, EXEC_MEMO_BUILD, lvl.as<LevelDev>(), zeros.as<uint8_t>() + 64, 0, 1, nullptr,
                 nullptr, nullptr, 0, 0);
  CK(cudaStreamSynchronize(st));
  pr.memo_ready = true;
}

template <typename R>
static void launch_exec(ptsbe_plan* pl, Program& pr, uint32_t mode, const LevelDev* levels_dev,
                        const uint8_t* kraus_dev, uint32_t first, uint32_t n_items, void* out,
                        double* mass, double* minv, uint32_t vec_stride, uint32_t vec_row) {
  using C = typename CxT<R>::type;
  if (n_items == 0) return;
  const bool memo = pr.d.memo_elems && pr.d.threads_per_item > 32;
  if (memo && !pr.memo_ready && mode != EXEC_MEMO_BUILD) build_memo<R>(pl, pr);
  ExecLaunch L = configure_exec<R>(pl, pr, n_items);
  DevBuf spill;
  if (pr.d.arena_spill_elems)
    spill.alloc((size_t)L.grid * L.groups_per_block * pr.d.arena_spill_elems * sizeof(C),
                pl->stream);
  ExecArgs a;
  a.leaves = pr.leaves.as<uint32_t>();
  a.steps = pr.steps.as<uint32_t>();
  a.tables = pr.tables.as<uint32_t>();
  a.pool = pl->pool.p;
  a.kraus = kraus_dev;
  a.levels = levels_dev;
  a.spill = spill.p;
  a.out = out;
  a.out_mass = mass;
  a.out_min = minv;
  a.n_steps = pr.d.n_steps;
  a.arena_fast = pr.d.arena_fast_elems;
  a.arena_spill = pr.d.arena_spill_elems;
  a.out_elems = mode == EXEC_VECTOR ? pr.d.proj_d : pr.d.out_elems;
  a.result_kind = pr.d.result_kind;
  a.result_ref = pr.d.result_ref;
  a.level = pr.d.level;
  a.first_item = first;
  a.n_items = n_items;
  a.g = pl->g;
  a.words = pl->words;
  a.item_bytes = L.item_bytes;
  a.mode = mode;
  a.vec_stride = vec_stride;
  a.vec_row = vec_row;
  a.desc_off = L.desc_off;
  a.desc_cap = L.desc_cap;
  a.memo = memo ? pr.memo.p : nullptr;
  a.memo_ptr = pr.memo_ptr.as<uint32_t>();
  a.memo_idx = pr.memo_idx.as<uint32_t>();
  a.n_memo_sites = pr.d.n_memo_sites;
  a.n_leaves = pr.d.n_leaves;
  a.n_table_words = pr.d.n_table_words;
  a.tc_off = L.tc_off;
  a.tile_min = pl->tile_min;
  L.kern<<<L.grid, L.block, L.smem, pl->stream>>>(a);
  g_launches++;
  CK(cudaGetLastError());
}

static void launch_exec_any(ptsbe_plan* pl, Program& pr, uint32_t mode, const LevelDev* lv,
                            const uint8_t* kraus, uint32_t first, uint32_t n, void* out,
                            double* mass, double* minv, uint32_t vec_stride = 0,
                            uint32_t vec_row = 0) {
  if (pl->dtype == PTSBE_C64)
    launch_exec<float>(pl, pr, mode, lv, kraus, first, n, out, mass, minv, vec_stride, vec_row);
  else
    launch_exec<double>(pl, pr, mode, lv, kraus, first, n, out, mass, minv, vec_stride, vec_row);
}

// ---- lane-per-item interpreter (lane.cuh) ----
static void classify_lane(const ptsbe_plan* pl, Program& pr) {
  const ptsbe_program_desc& d = pr.d;
  pr.lane_ok = pr.lane_fused = false;
  pr.lane_big_ok = false;
  if (d.n_steps && d.steps && d.level == 1 && d.threads_per_item <= 32 && !d.arena_spill_elems && !d.memo_elems &&
      !d.proj_d && d.arena_fast_elems > 48 && pl->f + 2 <= (uint32_t)LN_MAX_LEVELS) {
    const LaneLayout Lb = lane_layout(d.n_steps, d.n_leaves, 0, pl->f + 2, 0, pl->words, (uint32_t)pl->elem);
    uint64_t serial = 0;
    for (uint32_t s = 0; s < d.n_steps; ++s) {
      const uint32_t* st = d.steps + (size_t)s * STEP_WORDS;
      serial += (uint64_t)st[6] * std::max<uint32_t>(st[7], 1);
    }
    pr.lane_big_ok = Lb.end <= 100 * 1024 && serial <= (1u << 18);
  }
  if (!d.n_steps || !d.steps || d.threads_per_item > 32 || d.arena_spill_elems || d.arena_fast_elems > 48 ||
      d.memo_elems || d.level + 1 > (uint32_t)LN_MAX_LEVELS || pl->f + 2 > (uint32_t)LN_MAX_LEVELS)
    return;
  const size_t image = ((size_t)d.n_steps * STEP_WORDS + (size_t)d.n_leaves * LEAF_WORDS + d.n_table_words) * 4;
  if (image > 24 * 1024) return;
  const LaneLayout L = lane_layout(d.n_steps, d.n_leaves, d.n_table_words, pl->f + 2, d.arena_fast_elems,
                                   pl->words, (uint32_t)pl->elem);
  if (L.end > 72 * 1024) return;  // keeps at least three CTAs per SM
  uint64_t serial = 0;
  bool inner_to_arena = true;
  for (uint32_t s = 0; s < d.n_steps; ++s) {
    const uint32_t* st = d.steps + (size_t)s * STEP_WORDS;
    serial += (uint64_t)st[6] * std::max<uint32_t>(st[7], 1);
    if (s + 1 < d.n_steps && st[4] != 0) inner_to_arena = false;
  }
  if (serial > 16384) return;  // one thread would run too long; the group mapping is better
  pr.lane_ok = true;
  const uint32_t* last = d.steps + (size_t)(d.n_steps - 1) * STEP_WORDS;
  pr.lane_fused = d.proj_d && d.result_kind == 3 && inner_to_arena && last[4] == 1 && last[5] == 0 &&
                  last[6] == d.proj_d;
  // Hermitian form: last step = outer product of one arena tensor with its own conjugate
  pr.herm = false;
  pr.herm_map_host.clear();
  const uint32_t D = d.proj_d, flags = last[11];
  if (pr.lane_fused && D <= 4096 && last[7] == 1 && last[9] == 1 && !(flags & (4u | 8u)) &&
      last[0] == 0 && last[2] == 0 && last[1] == last[3] && ((flags & 3u) == 1u || (flags & 3u) == 2u) && d.tables) {
    const uint32_t* t = d.tables + last[10];
    const uint32_t lo_n = last[8];
    const uint32_t *loA = t, *loB = t + lo_n, *kA = t + 2 * lo_n + 2, *kB = kA + 1;
    std::vector<std::pair<uint32_t, uint32_t>> ab(D);
    bool ok = lo_n == D;
    for (uint32_t c = 0; ok && c < D; ++c) ab[c] = {loA[c] + kA[0], loB[c] + kB[0]};
    std::vector<uint32_t> partner(D, 0xffffffffu);
    for (uint32_t c = 0; ok && c < D; ++c) {
      for (uint32_t c2 = 0; c2 < D; ++c2)
        if (ab[c2].first == ab[c].second && ab[c2].second == ab[c].first) { partner[c] = c2; break; }
      if (partner[c] == 0xffffffffu) ok = false;
    }
    if (ok) {
      // slots: diagonal elements first come as they appear, pairs as (Re, Im) of the smaller index
      for (uint32_t c = 0; c < D; ++c) {
        const uint32_t c2 = partner[c];
        if (c2 == c) pr.herm_map_host.push_back(c | (c << 12) | (0u << 24));
        else if (c < c2) {
          pr.herm_map_host.push_back(c | (c2 << 12) | (0u << 24));
          pr.herm_map_host.push_back(c | (c2 << 12) | (1u << 24));
        }
      }
      pr.herm = pr.herm_map_host.size() == D;
      if (!pr.herm) pr.herm_map_host.clear();
    }
    // canonical order of lane_x.cuh: x has DX entries at element offsets 0 .. DX-1 of the operand
    pr.herm_dx = 0;
    pr.herm_canon_host.clear();
    uint32_t dx = 0;
    for (uint32_t k : {4u, 8u}) if (k * k == D) dx = k;  // packed rows of exactly D reals (herm_shape pads below 16)
    if (pr.herm && dx && pl->dtype == PTSBE_C64) {
      bool fine = true;
      std::vector<uint32_t> canon(D, 0), hit(D, 0);
      for (uint32_t s2 = 0; fine && s2 < D; ++s2) {
        const uint32_t m = pr.herm_map_host[s2];
        const uint32_t c = m & 0xfffu, c2 = (m >> 12) & 0xfffu, kind = m >> 24;
        uint32_t p = ab[c].first, q = ab[c].second;
        if ((flags & 3u) == 1u) std::swap(p, q);  // v_c = conj(x_a) x_b = x_b conj(x_a)
        if (p >= dx || q >= dx || (c == c2) != (p == q)) { fine = false; break; }
        uint32_t pos, neg = 0;
        if (p == q) {
          pos = p;
        } else {
          const uint32_t lo = std::min(p, q), hi = std::max(p, q);
          uint32_t idx = 0;
          for (uint32_t z = 0; z < lo; ++z) idx += dx - 1 - z;
          idx += hi - lo - 1;
          pos = dx + 2 * idx + (kind ? 1u : 0u);
          neg = (kind == 1 && p > q) ? 1u : 0u;
        }
        if (pos >= D || hit[pos]++) { fine = false; break; }
        canon[s2] = pos | (neg << 31);
      }
      if (fine) {
        pr.herm_dx = dx;
        pr.herm_canon_host = canon;
      }
    }
  }
  // chain form (lane_x.cuh CHAIN): steps 0 .. n-2 are x_s = x_{s-1} . T_s with T_s a block of a record
  // (an earlier pass of this stage) sliced by prefix bits, x_0 a record of an earlier pass
  pr.lane_chain = false;
  if (pr.herm_dx && d.n_steps >= 2 && d.n_steps - 1 <= (uint32_t)LN_CHAIN_MAX && d.tables) {
    const uint32_t dx = pr.herm_dx;
    bool ok = last[0] == 0;
    uint32_t prev_out = 0;
    for (uint32_t s = 0; ok && s + 1 < d.n_steps; ++s) {
      const uint32_t* st = d.steps + (size_t)s * STEP_WORDS;
      const uint32_t fl = st[11], kn = st[7], lo_n = st[8], hi_n = st[9];
      const bool vec_a = (fl & 32u) != 0, vec_b = (fl & 64u) != 0;
      if (vec_a == vec_b || (fl & 4u) || st[4] != 0 || st[6] != dx || lo_n != dx || hi_n != 1 || kn < 1 || kn > 8) { ok = false; break; }
      const uint32_t* t = d.tables + st[10];
      const uint32_t *kA = t + 2 * lo_n + 2 * hi_n, *kB = kA + kn, *dyn = kB + kn;
      const uint32_t vk = vec_a ? st[0] : st[2], vr = vec_a ? st[1] : st[3], mk = vec_a ? st[2] : st[0];
      const uint32_t* kV = vec_a ? kA : kB;
      for (uint32_t k = 0; k < kn; ++k) if (kV[k] != k) ok = false;
      if (fl & 8u) {  // no prefix-bit slicing on the vector side
        const uint32_t na = dyn[0], nb = dyn[1 + 2 * na];
        if ((vec_a ? na : nb) != 0) ok = false;
      }
      if (mk < 2 || mk - 1 > d.level) ok = false;   // the matrix comes from a record
      if (s == 0) { if (vk < 2 || vk - 1 > d.level) ok = false; }
      else if (vk != 0 || vr != prev_out || kn != dx) ok = false;
      prev_out = st[5];
    }
    if (ok && last[1] != prev_out) ok = false;  // the outer product is taken of the chain's result
    pr.lane_chain = ok;
  }
}

template <typename R>
static LaneArgs lane_args(ptsbe_plan* pl, Program& pr, uint32_t mode, const LevelDev* levels_dev,
                          const uint8_t* kraus_dev, uint32_t first, uint32_t n_items, void* out,
                          uint32_t vec_row) {
  LaneArgs a;
  memset(&a, 0, sizeof a);
  a.e.leaves = pr.leaves.as<uint32_t>();
  a.e.steps = pr.steps.as<uint32_t>();
  a.e.tables = pr.tables.as<uint32_t>();
  a.e.pool = pl->pool.p;
  a.e.kraus = kraus_dev;
  a.e.levels = levels_dev;
  a.e.out = out;
  a.e.n_steps = pr.d.n_steps;
  a.e.arena_fast = pr.d.arena_fast_elems;
  a.e.out_elems = pr.d.out_elems;
  a.e.level = pr.d.level;
  a.e.first_item = first;
  a.e.n_items = n_items;
  a.e.g = pl->g;
  a.e.words = pl->words;
  a.e.mode = mode;
  a.e.vec_row = vec_row;
  a.n_leaves = pr.d.n_leaves;
  a.n_table_words = pr.d.n_table_words;
  a.n_levels = pl->f + 2;
  a.tiny = pl->lane_tiny;
  return a;
}

template <typename R>
static void launch_lane(ptsbe_plan* pl, Program& pr, uint32_t mode, const LevelDev* levels_dev,
                        const uint8_t* kraus_dev, uint32_t first, uint32_t n_items, void* out,
                        uint32_t vec_row) {
  using C = typename CxT<R>::type;
  if (n_items == 0) return;
  const LaneArgs a = lane_args<R>(pl, pr, mode, levels_dev, kraus_dev, first, n_items, out, vec_row);
  const LaneLayout L = lane_layout(a.e.n_steps, a.n_leaves, a.n_table_words, a.n_levels, a.e.arena_fast,
                                   a.e.words, (uint32_t)sizeof(C));
  if (pr.lane_blocks_per_sm == 0) {
    CK(cudaFuncSetAttribute(exec_lane_kernel<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    int nb = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, exec_lane_kernel<R>, LN_THREADS, L.end));
    pr.lane_blocks_per_sm = std::max(nb, 1);
  }
  const uint64_t need = cdiv(n_items, LN_THREADS);
  const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(need, (uint64_t)pl->sm_count * pr.lane_blocks_per_sm));
  exec_lane_kernel<R><<<grid, LN_THREADS, L.end, pl->stream>>>(a);
  g_launches++;
  CK(cudaGetLastError());
}

// class-0 hoist over a large batch of error sets: one thread per error set, arena in global memory
template <typename R>
static void launch_lane_big(ptsbe_plan* pl, Program& pr, uint32_t mode, const LevelDev* levels_dev,
                            const uint8_t* kraus_dev, uint32_t first, uint32_t n_items, void* out,
                            double* mass = nullptr, double* minv = nullptr) {
  using C = typename CxT<R>::type;
  if (n_items == 0) return;
  LaneArgs a = lane_args<R>(pl, pr, mode, levels_dev, kraus_dev, first, n_items, out, 0);
  a.e.out_mass = mass;
  a.e.out_min = minv;
  a.e.result_kind = pr.d.result_kind;
  a.e.result_ref = pr.d.result_ref;
  a.e.item_bytes = pr.d.threads_per_item;  // MARGINAL: the mass is folded the way that many lanes would (lane.cuh)
  a.tiny = 0;  // hundreds of steps per item: the unrolled variants pay here (measured: 20.5 against 22.6 ms on cfg5)
  const LaneLayout L = lane_layout(a.e.n_steps, a.n_leaves, 0, a.n_levels, 0, a.e.words, (uint32_t)sizeof(C));
  opt_in_smem((const void*)exec_lane_kernel<R, true>, 200 * 1024);
  if (pr.lane_big_blocks_per_sm == 0)
    pr.lane_big_blocks_per_sm = cached_occupancy((const void*)exec_lane_kernel<R, true>, LN_THREADS, L.end);
  const uint64_t need = cdiv(n_items, LN_THREADS);
  const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(need, (uint64_t)pl->sm_count * pr.lane_big_blocks_per_sm));
  DevBuf arena((size_t)grid * LN_WARPS * pr.d.arena_fast_elems * 32 * sizeof(C), pl->stream);
  a.e.spill = arena.p;
  exec_lane_kernel<R, true><<<grid, LN_THREADS, L.end, pl->stream>>>(a);
  g_launches++;
  CK(cudaGetLastError());
}

// hoist pass of a per-prefix program: lane-per-item when the program qualifies
static void launch_hoist(ptsbe_plan* pl, Program& pr, const LevelDev* lv, const uint8_t* kraus,
                         uint32_t n, void* out) {
  if (pr.lane_big_ok && pl->lane && n >= pl->lane_big_min) {
    if (pl->dtype == PTSBE_C64) launch_lane_big<float>(pl, pr, EXEC_HOIST, lv, kraus, 0, n, out);
    else launch_lane_big<double>(pl, pr, EXEC_HOIST, lv, kraus, 0, n, out);
    return;
  }
  if (pr.lane_ok && pl->lane) {
    if (pl->dtype == PTSBE_C64) launch_lane<float>(pl, pr, EXEC_HOIST, lv, kraus, 0, n, out, 0);
    else launch_lane<double>(pl, pr, EXEC_HOIST, lv, kraus, 0, n, out, 0);
  } else {
    launch_exec_any(pl, pr, EXEC_HOIST, lv, kraus, 0, n, out, nullptr, nullptr);
  }
}

// ---- per-qubit descent sampler (descent.cuh) ----
struct DescentShape { uint32_t nch = 0, dpad = 0; size_t smem = 0; bool fits = false; };

static DescentShape descent_shape(const ptsbe_plan* pl, uint32_t D, uint32_t b) {
  DescentShape s;
  const uint32_t cpc = pl->dtype == PTSBE_C64 ? 2 : 1;
  for (uint32_t nch = 1; nch <= 8; nch <<= 1)
    if (DS_GS * nch * cpc >= D) { s.nch = nch; break; }
  if (!s.nch || b > 12) { s.nch = 0; return s; }
  s.dpad = DS_GS * s.nch * cpc;
  s.smem = ((size_t)s.dpad * pl->elem + (size_t)DS_GROUPS * 4) << b;
  s.fits = s.smem <= 160 * 1024;  // the stand-alone kernel's table; the fused Hermitian kernel packs it in half
  return s;
}

template <typename R, int NCH>
static void launch_descent_t(ptsbe_plan* pl, const DescentArgs& a, size_t smem) {
  opt_in_smem((const void*)descent_kernel<R, NCH>, 200 * 1024);
  const int per_sm = cached_occupancy((const void*)descent_kernel<R, NCH>, DS_THREADS, smem);
  const uint64_t tiles = cdiv(a.n_items, DS_TILE);
  const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(tiles, (uint64_t)pl->sm_count * per_sm));
  descent_kernel<R, NCH><<<grid, DS_THREADS, smem, pl->stream>>>(a);
  g_launches++;
  CK(cudaGetLastError());
}

static void launch_descent(ptsbe_plan* pl, const DescentArgs& a, const DescentShape& sh) {
  if (a.n_items == 0) return;
  const bool f32 = pl->dtype == PTSBE_C64;
  switch (sh.nch) {
    case 1: f32 ? launch_descent_t<float, 1>(pl, a, sh.smem) : launch_descent_t<double, 1>(pl, a, sh.smem); break;
    case 2: f32 ? launch_descent_t<float, 2>(pl, a, sh.smem) : launch_descent_t<double, 2>(pl, a, sh.smem); break;
    case 4: f32 ? launch_descent_t<float, 4>(pl, a, sh.smem) : launch_descent_t<double, 4>(pl, a, sh.smem); break;
    case 8: f32 ? launch_descent_t<float, 8>(pl, a, sh.smem) : launch_descent_t<double, 8>(pl, a, sh.smem); break;
    default: throw Failure(PTSBE_EINVAL, "descent sampler: unsupported vector length");
  }
}

template <typename R, int NCH, bool HERM>
static void launch_lane_descent_t(ptsbe_plan* pl, Program& pr, LaneDescentArgs& a, uint32_t n_sets) {
  using C = typename CxT<R>::type;
  using CH = typename DsChunk<R>::type;
  const LaneLayout L = lane_layout(a.l.e.n_steps, a.l.n_leaves, a.l.n_table_words, a.l.n_levels,
                                   a.l.e.arena_fast, a.l.e.words, (uint32_t)sizeof(C));
  const size_t table = ((size_t)(LN_GS * NCH + (NCH >= 2 ? 0 : 1)) * sizeof(CH)) << a.d.b;
  const size_t fixed = (size_t)L.end + (size_t)LN_THREADS * (8 + 6 * 4);
  // short runs of items per error set: a private table per warp, no CTA barriers (lane.cuh warp_runs)
  a.warp_runs = pl->warp_runs && a.d.n_items < (uint64_t)pl->warp_run_len * n_sets &&
                fixed + table * LN_WARPS <= 110 * 1024;
  const size_t smem = fixed + table * (a.warp_runs ? LN_WARPS : 1);
  if (smem > 200 * 1024) throw Failure(PTSBE_ERESOURCE, "fused descent needs more shared memory than one SM has");
  opt_in_smem((const void*)lane_descent_kernel<R, NCH, HERM>, 200 * 1024);
  const int per_sm = cached_occupancy((const void*)lane_descent_kernel<R, NCH, HERM>, LN_THREADS, smem);
  // tiles: long enough to amortise the CTA barriers around an error-set run, short enough that
  // every resident CTA gets several
  const uint64_t ctas = (uint64_t)pl->sm_count * per_sm;
  uint64_t tile = a.d.n_items / (ctas * 4) / LN_THREADS * LN_THREADS;
  tile = std::min<uint64_t>(pl->descent_tile_max, std::max<uint64_t>(LN_THREADS, tile));
  a.tile = (uint32_t)tile;
  const uint64_t tiles = cdiv(a.d.n_items, tile);
  const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(tiles, ctas));
  lane_descent_kernel<R, NCH, HERM><<<grid, LN_THREADS, smem, pl->stream>>>(a);
  g_launches++;
  CK(cudaGetLastError());
}

template <int DX, bool CHAIN>
static void launch_lane_descent_x(ptsbe_plan* pl, Program& pr, LaneDescentArgs& a, uint32_t n_sets) {
  // CHAIN keeps the intermediate vectors in registers: the arena holds only x (DX entries per item)
  if (CHAIN) a.l.e.arena_fast = DX;
  a.l.ast = 32;  // one lane per item and per draw: every lane stays inside its own arena slice
  const LaneLayout L = lane_layout(a.l.e.n_steps, a.l.n_leaves, a.l.n_table_words, a.l.n_levels,
                                   a.l.e.arena_fast, a.l.e.words, (uint32_t)sizeof(float2), a.l.ast);
  constexpr size_t NQ = DX * DX / 4 > 0 ? DX * DX / 4 : 1;
  const size_t table = ((NQ + 1) * 16) << a.d.b;
  const size_t fixed = (size_t)L.end + (size_t)LN_THREADS * (8 + 6 * 4 + (CHAIN ? LN_CHAIN_MAX * 4 : 0));
  a.warp_runs = pl->warp_runs && a.d.n_items < (uint64_t)pl->warp_run_len * n_sets &&
                fixed + table * LN_WARPS <= 110 * 1024;
  const size_t smem = fixed + table * (a.warp_runs ? LN_WARPS : 1);
  if (smem > 200 * 1024) throw Failure(PTSBE_ERESOURCE, "fused descent needs more shared memory than one SM has");
  opt_in_smem((const void*)lane_descent_x_kernel<DX, CHAIN>, 200 * 1024);
  const int per_sm = cached_occupancy((const void*)lane_descent_x_kernel<DX, CHAIN>, LN_THREADS, smem);
  const uint64_t ctas = (uint64_t)pl->sm_count * per_sm;
  uint64_t tile = a.d.n_items / (ctas * 4) / LN_THREADS * LN_THREADS;
  tile = std::min<uint64_t>(pl->descent_tile_max, std::max<uint64_t>(LN_THREADS, tile));
  a.tile = (uint32_t)tile;
  const uint64_t tiles = cdiv(a.d.n_items, tile);
  const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(tiles, ctas));
  lane_descent_x_kernel<DX, CHAIN><<<grid, LN_THREADS, smem, pl->stream>>>(a);
  g_launches++;
  CK(cudaGetLastError());
}

static bool lane_descent_fits(const ptsbe_plan* pl, const Program& pr, const DescentShape& sh, uint32_t b) {
  const uint32_t elem = (uint32_t)pl->elem;
  const LaneLayout L = lane_layout(pr.d.n_steps, pr.d.n_leaves, pr.d.n_table_words, pl->f + 2,
                                   pr.d.arena_fast_elems, pl->words, elem);
  // sh is the 8-lane shape of descent.cuh; the fused kernel spreads the same padded column over LN_GS lanes
  const uint32_t nch_f = sh.nch * (DS_GS / LN_GS);
  const size_t smem = (size_t)L.end + (size_t)LN_THREADS * (8 + 6 * 4) + (((size_t)(LN_GS * nch_f + (nch_f >= 2 ? 0 : 1)) * 16) << b);
  return nch_f <= 8 && smem <= 200 * 1024;
}

// descent shape of the Hermitian-packed form: D reals per column
static DescentShape herm_shape(const ptsbe_plan* pl, uint32_t D);

// the fused kernel over Hermitian-packed columns (table of D reals per node)
static bool lane_descent_fits_packed(const ptsbe_plan* pl, const Program& pr, const DescentShape& hsh, uint32_t b) {
  if (!hsh.nch) return false;
  const LaneLayout L = lane_layout(pr.d.n_steps, pr.d.n_leaves, pr.d.n_table_words, pl->f + 2,
                                   pr.d.arena_fast_elems, pl->words, (uint32_t)pl->elem);
  const size_t smem = (size_t)L.end + (size_t)LN_THREADS * (8 + 6 * 4) +
                      (((size_t)(LN_GS * hsh.nch + (hsh.nch >= 2 ? 0 : 1)) * 16) << b);
  return smem <= 200 * 1024;
}

// How a projection-form stage is sampled by descent: fused per-item steps + descent (packed table when the cut
// vector is Hermitian, which also fits where the unpacked table does not: complex128 at D = 64, b = 8), the
// stand-alone kernel, or not at all (ok == false: project + flat sampler).
struct DescentChoice { DescentShape dsh, hsh; bool fused = false, ok = false; };
static DescentChoice choose_descent(const ptsbe_plan* pl, const Program& prj, uint32_t b) {
  DescentChoice c;
  c.dsh = descent_shape(pl, prj.d.proj_d, b);
  if (!c.dsh.nch) return c;
  if (pl->lane && prj.lane_fused) {
    if (prj.herm) {
      c.hsh = herm_shape(pl, prj.d.proj_d);
      c.fused = lane_descent_fits_packed(pl, prj, c.hsh, b);
      if (!c.fused) c.hsh = DescentShape();
    }
    if (!c.fused) c.fused = lane_descent_fits(pl, prj, c.dsh, b);
  }
  c.ok = c.fused || c.dsh.fits;
  return c;
}

static void launch_lane_descent(ptsbe_plan* pl, Program& pr, LaneDescentArgs& a, const DescentShape& sh,
                                uint32_t n_sets) {
  if (a.d.n_items == 0) return;
  const bool f32 = pl->dtype == PTSBE_C64;
  if (a.herm_map && f32 && pr.herm_dx && pl->lane_x) {
    // x (x) conj(x) with a small x: one lane per draw over canonically packed columns (lane_x.cuh)
    const bool chain = pr.lane_chain && pl->lane_chain;
    switch (pr.herm_dx) {
      case 4: chain ? launch_lane_descent_x<4, true>(pl, pr, a, n_sets) : launch_lane_descent_x<4, false>(pl, pr, a, n_sets); return;
      case 8: chain ? launch_lane_descent_x<8, true>(pl, pr, a, n_sets) : launch_lane_descent_x<8, false>(pl, pr, a, n_sets); return;
      default: break;
    }
  }
  if (a.herm_map) {
    switch (sh.nch) {
      case 1: f32 ? launch_lane_descent_t<float, 1, true>(pl, pr, a, n_sets) : launch_lane_descent_t<double, 1, true>(pl, pr, a, n_sets); break;
      case 2: f32 ? launch_lane_descent_t<float, 2, true>(pl, pr, a, n_sets) : launch_lane_descent_t<double, 2, true>(pl, pr, a, n_sets); break;
      case 4: f32 ? launch_lane_descent_t<float, 4, true>(pl, pr, a, n_sets) : launch_lane_descent_t<double, 4, true>(pl, pr, a, n_sets); break;
      case 8: f32 ? launch_lane_descent_t<float, 8, true>(pl, pr, a, n_sets) : launch_lane_descent_t<double, 8, true>(pl, pr, a, n_sets); break;
      default: throw Failure(PTSBE_EINVAL, "descent sampler: unsupported vector length");
    }
    return;
  }
  switch (sh.nch) {
    case 1: f32 ? launch_lane_descent_t<float, 1, false>(pl, pr, a, n_sets) : launch_lane_descent_t<double, 1, false>(pl, pr, a, n_sets); break;
    case 2: f32 ? launch_lane_descent_t<float, 2, false>(pl, pr, a, n_sets) : launch_lane_descent_t<double, 2, false>(pl, pr, a, n_sets); break;
    case 4: f32 ? launch_lane_descent_t<float, 4, false>(pl, pr, a, n_sets) : launch_lane_descent_t<double, 4, false>(pl, pr, a, n_sets); break;
    case 8: f32 ? launch_lane_descent_t<float, 8, false>(pl, pr, a, n_sets) : launch_lane_descent_t<double, 8, false>(pl, pr, a, n_sets); break;
    default: throw Failure(PTSBE_EINVAL, "descent sampler: unsupported vector length");
  }
}

// descent shape of the Hermitian-packed form: D reals per column
static DescentShape herm_shape(const ptsbe_plan* pl, uint32_t D) {
  DescentShape s;
  const uint32_t epc = pl->dtype == PTSBE_C64 ? 4 : 2;  // reals per 16-byte chunk
  for (uint32_t nch = 1; nch <= 8; nch <<= 1)
    if (LN_GS * nch * epc >= D) { s.nch = nch; break; }
  s.dpad = LN_GS * s.nch * epc;
  return s;
}

static void launch_tree_build(ptsbe_plan* pl, const Program& pr, const void* rec0, uint32_t rec_stride,
                              uint32_t n_sets, uint32_t b, uint32_t dpad, void* tree) {
  TreeArgs t;
  t.rec0 = rec0;
  t.tree = tree;
  t.rec_stride = rec_stride;
  t.m_off = pr.d.result_ref;
  t.D = pr.d.proj_d;
  t.b = b;
  t.dpad = dpad;
  t.n_sets = n_sets;
  static const bool reduce_tree = env_size("PTSBE_TREE_REDUCE", 1) != 0;
  if (b <= (uint32_t)TB_MAX_B && reduce_tree) {
    const dim3 grid(n_sets, cdiv(dpad, (uint32_t)TB_ROWS));
    if (pl->dtype == PTSBE_C64) tree_reduce_kernel<float><<<grid, TB_ROWS * 32, 0, pl->stream>>>(t);
    else tree_reduce_kernel<double><<<grid, TB_ROWS * 32, 0, pl->stream>>>(t);
  } else {
    const dim3 grid(n_sets, cdiv(((uint64_t)dpad) << b, 256));  // error sets on x: up to 2^31 - 1
    if (pl->dtype == PTSBE_C64) tree_build_kernel<float><<<grid, 256, 0, pl->stream>>>(t);
    else tree_build_kernel<double><<<grid, 256, 0, pl->stream>>>(t);
  }
  g_launches++;
  CK(cudaGetLastError());
}

static inline uint32_t vec_pitch(uint32_t n) { return (n + PJ_TI - 1) / PJ_TI * PJ_TI; }

// P = Re(V . M) for the work items [first, first + n) of a level (project.cuh)
static void launch_project(ptsbe_plan* pl, const Program& pr, const void* v, uint32_t v_stride,
                           const void* rec0, uint32_t rec_stride, const uint32_t* eset,
                           uint32_t first, uint32_t n, void* out) {
  if (n == 0) return;
  ProjectArgs a;
  a.vt = v;
  a.v_stride = v_stride;
  a.rec0 = rec0;
  a.eset = eset;
  a.out = out;
  a.first_item = first;
  a.n_items = n;
  a.D = pr.d.proj_d;
  a.N = pr.d.out_elems;
  a.rec_stride = rec_stride;
  a.m_off = pr.d.result_ref;
  // column tile: 64 when the whole row fits (no dead columns), else 128
  const int narrow = a.N <= 64;
  const uint32_t tn = narrow ? 64 : PJ_TN;
  const uint64_t tiles = (uint64_t)cdiv(n, PJ_TI) * cdiv(a.N, tn);
  const bool f32 = pl->dtype == PTSBE_C64;
  const size_t smem = f32 ? 2 * (size_t)ProjK<float>::KC * (PJ_TI + tn) * sizeof(float2)    // two-deep ring
                          : 2 * (size_t)ProjK<double>::KC * (PJ_TI + tn) * sizeof(double2);
  using Kern = void (*)(const ProjectArgs);
  static const Kern kern[2][2] = {{project_kernel<double, PJ_TN>, project_kernel<double, 64>},
                                  {project_kernel<float, PJ_TN>, project_kernel<float, 64>}};
  const Kern k = kern[f32][narrow];
  opt_in_smem((const void*)k, 110 * 1024);
  const int occ = cached_occupancy((const void*)k, PJ_THREADS, smem);
  const unsigned grid = (unsigned)std::min<uint64_t>(tiles, (uint64_t)pl->sm_count * occ);
  k<<<grid, PJ_THREADS, smem, pl->stream>>>(a);
  g_launches++;
  CK(cudaGetLastError());
}

// ---- tensor-core projection (project_tc.cuh) ----
// cuTensorMapEncodeTiled through the runtime's driver entry point (no link against libcuda)
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeTiledFn encode_tiled_fn() {
  static EncodeTiledFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return (EncodeTiledFn)p;
  }();
  if (!fn) throw Failure(PTSBE_EDEVICE, "cuTensorMapEncodeTiled is not available from this driver");
  return fn;
}

// fp32 matrix [rows][k_floats] with row pitch `pitch_bytes`, tiles of box_rows x 32 floats, 128-byte swizzle
static CUtensorMap tc_map_2d(const void* ptr, uint64_t k_floats, uint64_t rows, uint64_t pitch_bytes, uint32_t box_rows) {
  CUtensorMap m;
  const cuuint64_t dims[2] = {k_floats, rows};
  const cuuint64_t strides[1] = {pitch_bytes};
  const cuuint32_t box[2] = {(cuuint32_t)TC_BK, box_rows};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult rc = encode_tiled_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(ptr), dims, strides, box,
                                        estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                        CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (rc != CUDA_SUCCESS) throw Failure(PTSBE_EDEVICE, "cuTensorMapEncodeTiled failed (" + std::to_string((int)rc) + ")");
  return m;
}

struct TcShape {
  uint32_t K = 0, kb = 0, stages = 0, tmem_cols = 0;
  size_t smem = 0;
  bool ok = false;
};

// K = 2 D padded to a multiple of 32 floats; ring depth from the shared memory one SM has
static TcShape tc_shape(uint32_t D, uint32_t N) {
  TcShape t;
  if (N < 32 || N > 256 || (N & (N - 1)) || D < 1) return t;
  t.K = (2 * D + TC_BK - 1) / TC_BK * TC_BK;
  t.kb = t.K / TC_BK;
  const size_t stage = 2 * (size_t)TC_A_BYTES + 2 * (size_t)N * TC_BK * 4;
  const size_t fixed = 1024 + 4 * 32 * 33 * 4 + (3 * TC_MAX_STAGES + 4) * 8 + 16;
  t.stages = (uint32_t)std::min<size_t>(TC_MAX_STAGES, (220 * 1024 - fixed) / stage);
  if (t.stages < 2) return t;
  t.smem = fixed + t.stages * stage;
  t.tmem_cols = 32;
  while (t.tmem_cols < 2 * N) t.tmem_cols <<= 1;
  t.ok = true;
  return t;
}

// hi / lo K-major images of B_e for every error set of the chunk (once per stage)
static void launch_tc_prep(ptsbe_plan* pl, const void* rec0, uint32_t rec_stride, uint32_t m_off, uint32_t n_sets,
                           uint32_t D, uint32_t N, const TcShape& t, float* b_hi, float* b_lo) {
  TcPrepArgs a;
  a.rec0 = reinterpret_cast<const float2*>(rec0);
  a.b_hi = b_hi;
  a.b_lo = b_lo;
  a.n_sets = n_sets; a.D = D; a.N = N; a.K = t.K; a.rec_stride = rec_stride; a.m_off = m_off;
  tc_prep_b_kernel<<<dim3(n_sets, cdiv(N, 32)), 256, 0, pl->stream>>>(a);
  g_launches++;
  CK(cudaGetLastError());
}

// P = A . B_e on the tensor cores for the work items [first, first + n) of a level; vrows: one row of
// t.K / 2 complex64 per item (zero padded), out [n][N] fp32
static void launch_project_tc(ptsbe_plan* pl, const TcShape& t, const void* vrows, const float* b_hi, const float* b_lo,
                              uint32_t n_sets, const uint32_t* eset, uint32_t first, uint32_t n, uint32_t N, void* out) {
  if (n == 0) return;
  const CUtensorMap ma = tc_map_2d(vrows, t.K, n, (uint64_t)t.K * 4, TC_BM);
  const CUtensorMap mh = tc_map_2d(b_hi, t.K, (uint64_t)n_sets * N, (uint64_t)t.K * 4, N);
  const CUtensorMap ml = tc_map_2d(b_lo, t.K, (uint64_t)n_sets * N, (uint64_t)t.K * 4, N);
  TcProjectArgs a;
  a.eset = eset;
  a.out = reinterpret_cast<float*>(out);
  a.first_item = first;
  a.n_items = n;
  a.N = N;
  a.kb = t.kb;
  a.stages = t.stages;
  a.tmem_cols = t.tmem_cols;
  opt_in_smem((const void*)project_tc_kernel, 227 * 1024);
  const unsigned grid = (unsigned)std::min<uint64_t>(cdiv(n, TC_BM), (uint64_t)pl->sm_count);
  project_tc_kernel<<<grid, TC_THREADS, t.smem, pl->stream>>>(ma, mh, ml, a);
  g_launches++;
  CK(cudaGetLastError());
}

static void launch_sampler(cudaStream_t st, SampleArgs& a, int sm_count) {
  if (a.n_items == 0) return;
  const size_t nb = 1ull << a.b;
  if (a.np_mode == 2 && nb * 12 > 160 * 1024) {
    // exhaustive harvest of a population vector beyond shared memory: streamed from global memory
    if (a.b > 30) throw Failure(PTSBE_ECAPACITY, "exhaustive harvest supports final batches of at most 30 qubits");
    const unsigned grid = (unsigned)std::min<uint64_t>(a.n_items, (uint64_t)sm_count * 2);
    harvest_big_kernel<<<grid, HB_THREADS, 0, st>>>(a);
    g_launches++;
    CK(cudaGetLastError());
    return;
  }
  if (a.b > 14) throw Failure(PTSBE_ECAPACITY, "sampler supports stage batches of at most 14 qubits");
  opt_in_smem((const void*)sample_kernel, 200 * 1024);
  opt_in_smem((const void*)sample_group_kernel<8>, 200 * 1024);
  opt_in_smem((const void*)sample_group_kernel<16>, 200 * 1024);
  opt_in_smem((const void*)sample_group_kernel<32>, 200 * 1024);
  if (a.np_mode) {
    opt_in_smem((const void*)nonprop_kernel, 200 * 1024);
    const unsigned grid = (unsigned)std::min<uint64_t>(a.n_items, (uint64_t)sm_count * 16);
    nonprop_kernel<<<grid, SAMPLE_THREADS, nb * 12, st>>>(a);
    g_launches++;
    CK(cudaGetLastError());
    return;
  }
  // Many items with few shots each: a group of 8/16/32 lanes per item.  Few items with many
  // shots (stage 1): one CTA per item so the draws spread over 128 threads.
  if (a.b <= 11 && a.n_items >= (uint64_t)sm_count * 16) {
    const int gs = nb <= 128 ? 8 : (nb <= 256 ? 16 : 32);  // ~50 KB of staging per block
    const size_t padded = nb + (nb >> 5) + 1;
    const size_t smem = (size_t)(SG_THREADS / gs) * padded * 12;
    const uint64_t per_sm = std::max<size_t>(1, std::min<size_t>(8, (200 * 1024) / smem));
    const uint64_t groups = SG_THREADS / gs;
    const unsigned grid = (unsigned)std::min<uint64_t>((a.n_items + groups - 1) / groups, (uint64_t)sm_count * per_sm);
    if (gs == 8) sample_group_kernel<8><<<grid, SG_THREADS, smem, st>>>(a);
    else if (gs == 16) sample_group_kernel<16><<<grid, SG_THREADS, smem, st>>>(a);
    else sample_group_kernel<32><<<grid, SG_THREADS, smem, st>>>(a);
  } else {
    const size_t smem = nb * 12;
    const uint64_t cap = (uint64_t)sm_count * 16;
    const unsigned grid = (unsigned)std::min<uint64_t>(a.n_items, cap);
    sample_kernel<<<grid, SAMPLE_THREADS, smem, st>>>(a);
  }
  g_launches++;
  CK(cudaGetLastError());
}

// Work-item list of one level, device resident.
struct Level {
  uint32_t n = 0;
  DevBuf eset, parent, prefix, mult, slot_off, rank, gid;
};

// non-proportional sampling (reference engine.py:527-576): per-stage multiplicities are not shot
// counts but branching factors
struct NonpropParams {
  uint32_t nonfinal_shots;  // children per prefix in every non-final stage (distinct, weighted)
  uint32_t final_mode;      // 0: exhaustive harvest (threshold), 1: direct multinomial of direct_count
  uint32_t direct_count;
  double threshold;
};

struct RunOutput {
  DevBuf probs;  // non-proportional exhaustive mode: conditional probability tag of every record
  // final records of one chunk, device resident (level f+1): eset rows, keys, counts
  DevBuf eset, keys, counts;
  uint64_t n = 0;
  bool unit_counts = false;  // every record is one raw draw (count 1): the merge may sort keys alone
};

// Runs error sets [e0, e0+ne) of a resident batch through all stages.
// A chunk is "dense" when some hoist pass has enough work to fill the GPU by itself (see run_chunk)
static bool chunk_is_dense(const ptsbe_plan* pl, uint64_t n_sets, uint64_t shots) {
  for (uint32_t j = 2; j <= pl->f; ++j)
    for (uint32_t p = 0; p + 1 < j; ++p) {
      const double items = std::min<double>((double)shots, (double)n_sets * std::pow(2.0, std::min<uint32_t>(pl->offsets[p], 60)));
      if (items * pl->programs[j - 1][p].macs > pl->eager_work_max) return true;
    }
  return false;
}

// Per-error-set tables of the descent sampler for one stage: column sums over the binary tree of the batch
// qubits (tree), Hermitian-packed (htree) when the fused kernel takes them that way.  Depends on the class-0
// records only.
static void build_descent_tables(ptsbe_plan* pl, Program& prj, const void* rec0, uint32_t rec_stride, uint32_t ne,
                                 uint32_t b, const DescentShape& dsh, const DescentShape& hsh, bool fused,
                                 DevBuf& tree, DevBuf& htree) {
  cudaStream_t st = pl->stream;
  const uint32_t nb = 1u << b;
  // small tables: trees and packing in one kernel, a warp per error set (lane.cuh tree_herm_kernel)
  const size_t th_warp = (size_t)2 * nb * sizeof(double2) + (size_t)prj.d.proj_d * nb * pl->elem;
  const bool tree_herm = fused && prj.herm && hsh.nch && pl->tree_herm && b <= (uint32_t)TB_MAX_B &&
                         (size_t)prj.d.proj_d * nb * pl->elem <= 16 * 1024;
  if (tree_herm) {
    const size_t real = pl->elem / 2;
    htree.alloc(((size_t)ne * hsh.dpad * real) << b, st);
    TreeHermArgs th;
    th.rec0 = rec0;
    th.packed = htree.p;
    th.map = prj.herm_map.as<uint32_t>();
    th.canon = (prj.herm_dx && pl->lane_x) ? prj.herm_canon.as<uint32_t>() : nullptr;
    th.rec_stride = rec_stride;
    th.m_off = prj.d.result_ref;
    th.D = prj.d.proj_d;
    th.b = b;
    th.dpad_r = hsh.dpad;
    th.n_sets = ne;
    const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(cdiv(ne, (uint32_t)TH_WARPS), (uint64_t)pl->sm_count * 8));
    if (pl->dtype == PTSBE_C64) {
      opt_in_smem((const void*)tree_herm_kernel<float>, 200 * 1024);
      tree_herm_kernel<float><<<grid, TH_WARPS * 32, th_warp * TH_WARPS, st>>>(th);
    } else {
      opt_in_smem((const void*)tree_herm_kernel<double>, 200 * 1024);
      tree_herm_kernel<double><<<grid, TH_WARPS * 32, th_warp * TH_WARPS, st>>>(th);
    }
    g_launches++;
    CK(cudaGetLastError());
    return;
  }
  tree.alloc(((size_t)ne * dsh.dpad * pl->elem) << b, st);
  launch_tree_build(pl, prj, rec0, rec_stride, ne, b, dsh.dpad, tree.p);
  if (fused && prj.herm && hsh.nch) {
    const size_t real = pl->elem / 2;
    htree.alloc(((size_t)ne * hsh.dpad * real) << b, st);
    HermPackArgs hp;
    hp.tree = tree.p;
    hp.packed = htree.p;
    hp.map = prj.herm_map.as<uint32_t>();
    hp.canon = (prj.herm_dx && pl->lane_x) ? prj.herm_canon.as<uint32_t>() : nullptr;
    hp.D = prj.d.proj_d;
    hp.dpad_c = dsh.dpad;
    hp.dpad_r = hsh.dpad;
    hp.b = b;
    const dim3 grid(ne, cdiv(((uint64_t)hsh.dpad) << b, 256));
    if (pl->dtype == PTSBE_C64) herm_pack_kernel<float><<<grid, 256, 0, st>>>(hp);
    else herm_pack_kernel<double><<<grid, 256, 0, st>>>(hp);
    g_launches++;
    CK(cudaGetLastError());
  }
}

static void run_chunk(ptsbe_plan* pl, const uint8_t* kraus_dev, const uint32_t* shots_dev,
                      const uint32_t* ids_dev, uint32_t ne, uint64_t chunk_shots, uint64_t seed,
                      RunOutput& out, ptsbe_run_stats* stats, unsigned long long* flag_dev,
                      uint32_t* flag_count_dev, Workspace& ws_out, const NonpropParams* npp = nullptr,
                      bool merged_out = false) {
  cudaStream_t st = pl->stream;
  const uint32_t f = pl->f, words = pl->words;
  const bool np_exhaustive = npp && npp->final_mode == 0;
  // multiplicity of the items ENTERING stage j in non-proportional mode
  auto np_mult = [&](uint32_t j) -> uint32_t {
    if (j < f) return npp->nonfinal_shots;
    return np_exhaustive ? (1u << pl->sizes[f - 1]) : npp->direct_count;
  };
  DevBuf slot_prob;
  if (np_exhaustive) slot_prob.alloc(chunk_shots * 8, st);
  const unsigned T = 256;
  std::vector<Level> lv(f + 2);
  std::vector<LevelDev> table(f + 2);
  memset(table.data(), 0, sizeof(LevelDev) * table.size());
  DevBuf table_dev((f + 2) * sizeof(LevelDev), st);
  DevBuf slot_index(chunk_shots * 4, st), slot_count(chunk_shots * 4, st);
  DevBuf scal(16, st);
  DevBuf set_mass((size_t)ne * 8, st);  // stage-1 mass (trajectory weight) of every error set

  // level 1: one item per error set, empty prefix
  {
    Level& l = lv[1];
    l.n = ne;
    l.eset.alloc((size_t)ne * 4, st);
    l.parent.alloc((size_t)ne * 4, st);
    l.prefix.alloc((size_t)ne * 8 * words, st);
    l.mult.alloc((size_t)ne * 4, st);
    l.slot_off.alloc((size_t)ne * 4, st);
    l.rank.alloc((size_t)ne * 4, st);
    l.gid.alloc((size_t)ne * 4, st);
    iota_kernel<<<cdiv(ne, T), T, 0, st>>>(l.eset.as<uint32_t>(), ne, 0);
    g_launches++;
    CK(cudaMemsetAsync(l.parent.p, 0, (size_t)ne * 4, st));
    CK(cudaMemsetAsync(l.prefix.p, 0, (size_t)ne * 8 * words, st));
    CK(cudaMemsetAsync(l.rank.p, 0, (size_t)ne * 4, st));
    if (npp) {
      fill_u32_kernel<<<cdiv(ne, T), T, 0, st>>>(l.mult.as<uint32_t>(), ne, np_mult(1));
      g_launches++;
    } else {
      CK(cudaMemcpyAsync(l.mult.p, shots_dev, (size_t)ne * 4, cudaMemcpyDeviceToDevice, st));
    }
    CK(cudaMemcpyAsync(l.gid.p, ids_dev, (size_t)ne * 4, cudaMemcpyDeviceToDevice, st));
    exclusive_scan<uint32_t, uint32_t>(l.mult.as<uint32_t>(), l.slot_off.as<uint32_t>(), ne,
                                       nullptr, st);
  }

  std::vector<cudaEvent_t> ev(f + 1);
  for (auto& e : ev) CK(cudaEventCreate(&e));
  CK(cudaEventRecord(ev[0], st));
  EventLog log(st);

  // ---- hoist passes run as early as their inputs exist, on one side stream per stage ----
  // Pass p of stage j needs the level-(p+1) work list (complete when stage p has been sampled) and the records
  // of the passes below it of the same stage -- nothing of stages p+1 .. j-1.  So as soon as level L is
  // built, pass L-1 of EVERY later stage is launched on that stage's side stream (class-0 passes, L = 1, before
  // stage 1 starts, together with the stage's descent tables when the plan fixed the sampler), and the main
  // stream waits for a stage's side stream where the stage begins.  The passes are latency-bound -- small
  // batches because no pass fills the GPU (cfg5 at E = 100: 2.96 -> 1.3 ms per step), large ones because they
  // wait on L2 and barriers (cfg5 at 10^5 sets 52.7 -> 48 ms, cfg2 37.1 -> 35.9 ms) -- so they overlap well.
  struct EventBag {
    std::vector<cudaEvent_t> v;
    cudaEvent_t make() { cudaEvent_t e; CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming)); v.push_back(e); return e; }
    ~EventBag() { for (cudaEvent_t e : v) cudaEventDestroy(e); }
  } events;
  std::vector<std::vector<DevBuf>> sext(f + 1);           // [stage][pass] records of the hoist passes
  std::vector<std::vector<LevelDev>> stab(f + 1);         // [stage] level table as the stage's passes see it
  std::vector<DevBuf> stab_dev(f + 1);
  std::vector<cudaEvent_t> sev(f + 1, nullptr);           // last work queued on the stage's side stream
  std::vector<uint32_t> passes_done(f + 1, 0);            // leading passes of the stage already launched
  std::vector<char> eager_off(f + 1, 0);                  // the stage has a pass that fills the GPU by itself
  struct PreTab { DevBuf tree, htree; bool done = false; };
  std::vector<PreTab> pre_tab(f + 1);
  struct SideGuard {  // declared after the buffers, so destroyed before them: no side-stream work outlives the
    ptsbe_plan* pl; bool on = false;  // chunk's records, tables or workspace, on any exit path
    ~SideGuard() { if (on) for (cudaStream_t q : pl->side) cudaStreamSynchronize(q); }
  } side_guard{pl};
  for (uint32_t j = 1; j <= f; ++j) {
    sext[j].resize(j);
    stab[j].assign(f + 2, LevelDev{});
    memset(stab[j].data(), 0, sizeof(LevelDev) * (f + 2));
  }
  // Dense regime (cfg3r1: hoist passes of 10^6-10^7 multiply-adds per item): every pass fills the GPU by itself
  // and running light passes beside them only takes SMs away (7.8 s against 7.2 s per 10^5 error sets), so a
  // chunk with any such pass runs everything in order.  Items of pass p are bounded by the chunk's shots and by
  // error sets x 2^(qubits measured before stage p+1).
  const bool dense = chunk_is_dense(pl, ne, chunk_shots);
  const bool eager = pl->prelaunch && f >= 2 && ne <= pl->prelaunch_max && !dense;
  if (eager) {
    while (pl->side.size() < f) {
      // the side stream of an earlier stage outranks those of later stages (and the plan's own stream outranks
      // them all): what the pipeline needs next is scheduled first, the rest fills the gaps
      cudaStream_t q;
      int lo = 0, hi = 0;  // numerically lower = higher priority
      CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
      const int prio = pl->side_priority ? std::min(lo, hi + 1 + (int)pl->side.size()) : lo;
      CK(cudaStreamCreateWithPriority(&q, cudaStreamNonBlocking, prio));
      pl->side.push_back(q);
    }
    side_guard.on = true;
    for (uint32_t j = 2; j <= f; ++j) stab_dev[j].alloc((f + 2) * sizeof(LevelDev), st);
  }
  // level L is complete on the main stream: launch pass L-1 of the stages L+1 .. f
  auto eager_hoists = [&](uint32_t L) {
    if (!eager || L + 1 > f) return;
    const uint32_t p = L - 1;
    for (uint32_t j = L + 1; j <= f; ++j) {  // records and table rows first (allocations on the main stream)
      Program& pp = pl->programs[j - 1][p];
      // a pass with enough work to fill the GPU gains nothing from running beside others (dense regime, cfg3r1:
      // 808 ms with every pass early against 741 ms in order); it and the later passes of its stage stay in order
      if ((double)lv[L].n * pp.macs > pl->eager_work_max) eager_off[j] = 1;
      if (eager_off[j]) continue;
      LevelDev& row = stab[j][L];
      row.eset = lv[L].eset.as<uint32_t>();
      row.parent = lv[L].parent.as<uint32_t>();
      row.prefix = lv[L].prefix.as<uint64_t>();
      row.n = lv[L].n;
      if (pp.d.n_steps && pp.d.out_elems) {
        sext[j][p].alloc((size_t)lv[L].n * pp.d.out_elems * pl->elem, st);
        row.ext = sext[j][p].p;        // a step may read its OWN pass's record, so the row points at it already
        row.ext_rec = pp.d.out_elems;
        // the variant-0 memo is built once per plan, on the plan's own stream
        if (p == 0 && pp.d.memo_elems && pp.d.threads_per_item > 32 && !pp.memo_ready) {
          if (pl->dtype == PTSBE_C64) build_memo<float>(pl, pp); else build_memo<double>(pl, pp);
        }
      }
      passes_done[j] = L;
    }
    cudaEvent_t ready = events.make();
    CK(cudaEventRecord(ready, st));
    for (uint32_t j = L + 1; j <= f; ++j) {
      Program& pp = pl->programs[j - 1][p];
      if (eager_off[j] || !(pp.d.n_steps && pp.d.out_elems)) continue;
      struct Swap { ptsbe_plan* pl; cudaStream_t keep; ~Swap() { pl->stream = keep; } } swap{pl, pl->stream};
      pl->stream = pl->side[j - 1];
      CK(cudaStreamWaitEvent(pl->stream, ready, 0));
      CK(cudaMemcpyAsync(stab_dev[j].p, stab[j].data(), sizeof(LevelDev) * (f + 2), cudaMemcpyHostToDevice, pl->stream));
      launch_hoist(pl, pp, stab_dev[j].as<LevelDev>(), kraus_dev, lv[L].n, sext[j][p].p);
      // the descent tables of the stage depend on the class-0 records only: same side stream, when the plan
      // has fixed the stage's sampler (the per-chunk choice needs the stage's work-list size)
      Program& pj = pl->programs[j - 1][j - 1];
      if (p == 0 && pl->descent && pl->stage_descent[j - 1] == 1 && pj.d.result_kind == 3 &&
          (!npp || (j == f && !np_exhaustive))) {
        const uint32_t bj = pl->sizes[j - 1];
        const DescentChoice dc = choose_descent(pl, pj, bj);
        if (dc.ok) {
          build_descent_tables(pl, pj, sext[j][0].p, pp.d.out_elems, ne, bj, dc.dsh, dc.hsh, dc.fused, pre_tab[j].tree, pre_tab[j].htree);
          pre_tab[j].done = true;
        }
      }
      sev[j] = events.make();
      CK(cudaEventRecord(sev[j], pl->stream));
    }
  };
  CK(cudaStreamSynchronize(st));  // level 1 is complete
  eager_hoists(1);

  for (uint32_t j = 1; j <= f; ++j) {
    Level& cur = lv[j];
    const uint32_t U = cur.n, b = pl->sizes[j - 1], nb = 1u << b;
    stats->stage_events[j - 1] += U;
    auto& progs = pl->programs[j - 1];
    // level table for this stage
    std::vector<DevBuf>& ext = sext[j];
    for (uint32_t l = 1; l <= j; ++l) {
      table[l].eset = lv[l].eset.as<uint32_t>();
      table[l].parent = lv[l].parent.as<uint32_t>();
      table[l].prefix = lv[l].prefix.as<uint64_t>();
      table[l].n = lv[l].n;
      table[l].ext = nullptr;
      table[l].ext_rec = 0;
      if (l < j && progs[l - 1].d.out_elems && progs[l - 1].d.n_steps) {
        // passes below passes_done[j] were launched early on the stage's side stream, records included
        if (l - 1 >= passes_done[j]) ext[l - 1].alloc((size_t)lv[l].n * progs[l - 1].d.out_elems * pl->elem, st);
        table[l].ext = ext[l - 1].p;
        table[l].ext_rec = progs[l - 1].d.out_elems;
      }
    }
    CK(cudaMemcpyAsync(table_dev.p, table.data(), sizeof(LevelDev) * (f + 2),
                       cudaMemcpyHostToDevice, st));
    if (sev[j]) CK(cudaStreamWaitEvent(st, sev[j], 0));  // the stage's early passes (and descent tables)
    // hoist passes: everything that does not depend on the newest prefix bits
    for (uint32_t p = 0; p + 1 < j; ++p) {
      if (!progs[p].d.n_steps) continue;
      if (p < passes_done[j]) continue;  // launched early
      log.begin(&stats->hoist_ms[j - 1]);
      launch_hoist(pl, progs[p], table_dev.as<LevelDev>(), kraus_dev, lv[p + 1].n, ext[p].p);
      log.end();
    }
    // marginal pass + sampler, in sub-batches sized to the probs buffer
    const size_t real = pl->dtype == PTSBE_C64 ? 4 : 8;
    const bool proj = progs[j - 1].d.result_kind == 3;
    DevBuf nnz((size_t)U * 4, st);
    // Stages whose work items carry few shots each are sampled by per-qubit descent over the
    // error set's conditional-marginal tree (descent.cuh) instead of project + sample.
    DescentChoice dc;
    const int hint = pl->stage_descent[j - 1];
    const bool few_shots = hint >= 0 ? hint == 1 : (double)chunk_shots <= pl->descent_mult * (double)U;
    if (proj && pl->descent && j > 1 && U && few_shots &&
        (!npp || (j == f && !np_exhaustive)))  // choice without replacement / harvest need the full vector
      dc = choose_descent(pl, progs[j - 1], b);
    if (dc.ok) {
      const DescentShape& dsh = dc.dsh;
      const Program& pr = progs[j - 1];
      Program& prj = progs[j - 1];
      const bool fused = dc.fused;
      // tree of conditional marginals per error set (Hermitian-packed when v = x (x) conj(x)); built up front
      // on the stage's side stream when the plan fixed the sampler (pre_tab), here otherwise
      const DescentShape& hsh = dc.hsh;
      DevBuf htree, tree;
      if (pre_tab[j].done) {
        htree = std::move(pre_tab[j].htree);
        tree = std::move(pre_tab[j].tree);
      } else {
        log.begin(&stats->descent_ms[j - 1]);
        build_descent_tables(pl, prj, table[1].ext, table[1].ext_rec, ne, b, dsh, hsh, fused, tree, htree);
        log.end();
      }
      if (fused) {
        // per-item steps and descent in one kernel: v never leaves the SM; raw per-draw outcomes
        // are merged into ordered (outcome, count) pairs afterwards
        DevBuf big_list(((size_t)(chunk_shots / LN_DEDUP_SERIAL) + 1) * 4, st), big_count(16, st);
        CK(cudaMemsetAsync(big_count.p, 0, 16, st));
        LaneDescentArgs fa;
        memset(&fa, 0, sizeof fa);
        if (pl->dtype == PTSBE_C64)
          fa.l = lane_args<float>(pl, prj, EXEC_VECTOR, table_dev.as<LevelDev>(), kraus_dev, 0, U, nullptr, 0);
        else
          fa.l = lane_args<double>(pl, prj, EXEC_VECTOR, table_dev.as<LevelDev>(), kraus_dev, 0, U, nullptr, 0);
        DescentArgs& da = fa.d;
        da.tree = hsh.nch ? htree.p : tree.p;
        fa.herm_map = hsh.nch ? prj.herm_map.as<uint32_t>() : nullptr;
        da.eset = cur.eset.as<uint32_t>();
        da.mult = cur.mult.as<uint32_t>();
        da.slot_off = cur.slot_off.as<uint32_t>();
        da.eset_id = cur.gid.as<uint32_t>();
        da.rank = cur.rank.as<uint32_t>();
        da.slot_index = slot_index.as<uint32_t>();
        da.slot_count = slot_count.as<uint32_t>();
        da.nnz = nnz.as<uint32_t>();
        da.flag = flag_dev;
        da.flag_count = flag_count_dev;
        da.set_mass = set_mass.as<double>();
        da.first_item = 0;
        da.n_items = U;
        da.b = b;
        da.stage = j;
        da.k0 = (uint32_t)seed;
        da.k1 = (uint32_t)(seed >> 32);
        da.vanish = pl->vanish;
        da.neg_abs = pl->neg_abs;
        da.neg_rel = pl->neg_rel;
        fa.big_list = big_list.as<uint32_t>();
        fa.big_count = big_count.as<uint32_t>();
        log.begin(&stats->descent_ms[j - 1]);
        DescentShape fsh = dsh;  // chunks per lane of the fused kernel's LN_GS-lane groups
        fsh.nch = dsh.nch * (DS_GS / LN_GS);
        launch_lane_descent(pl, prj, fa, hsh.nch ? hsh : fsh, ne);
        // Final stage of a run whose records are merged over error sets anyway: the raw draws (count 1 each,
        // nnz = multiplicity) go to the histogram as they are -- the descent sampler is chosen for stages with
        // about one draw per item, so the per-item merge removes next to nothing and the sort can then move
        // keys alone (merge_records of reference engine.py:815-829 sums equal bitstrings either way).
        const bool raw_final = merged_out && j == f && !npp && pl->raw_final;
        if (raw_final) out.unit_counts = true;
        DedupArgs dd;
        dd.slot_off = da.slot_off;
        dd.slot_index = da.slot_index;
        dd.slot_count = da.slot_count;
        dd.nnz = da.nnz;
        dd.big_list = fa.big_list;
        dd.big_count = fa.big_count;
        dd.first_item = 0;
        dd.n_items = U;
        dd.b = b;
        if (!raw_final) {
          dedup_kernel<<<cdiv(U, 256), 256, 0, st>>>(dd);
          dedup_big_kernel<<<pl->sm_count, 256, sizeof(uint32_t) << b, st>>>(dd);
          g_launches += 2;
        }
        CK(cudaGetLastError());
        log.end();
        stats->marg_launches[j - 1]++;
        stats->descent_items[j - 1] += U;
      } else {
      const size_t row = (size_t)dsh.dpad * pl->elem;
      const uint32_t B = (uint32_t)std::max<size_t>(DS_TILE, std::min<size_t>(U, pl->vec_budget / row));
      DevBuf vbuf((size_t)B * row, st);
      if (dsh.dpad != pr.d.proj_d) CK(cudaMemsetAsync(vbuf.p, 0, (size_t)B * row, st));
      for (uint32_t s0 = 0; s0 < U; s0 += B) {
        const uint32_t nbatch = std::min(B, U - s0);
        log.begin(&stats->marg_ms[j - 1]);
        launch_exec_any(pl, progs[j - 1], EXEC_VECTOR, table_dev.as<LevelDev>(), kraus_dev, s0,
                        nbatch, vbuf.p, nullptr, nullptr, 0, dsh.dpad);
        log.end();
        stats->marg_launches[j - 1]++;
        DescentArgs da;
        da.v = vbuf.p;
        da.tree = tree.p;
        da.eset = cur.eset.as<uint32_t>();
        da.mult = cur.mult.as<uint32_t>();
        da.slot_off = cur.slot_off.as<uint32_t>();
        da.eset_id = cur.gid.as<uint32_t>();
        da.rank = cur.rank.as<uint32_t>();
        da.slot_index = slot_index.as<uint32_t>();
        da.slot_count = slot_count.as<uint32_t>();
        da.nnz = nnz.as<uint32_t>();
        da.flag = flag_dev;
        da.flag_count = flag_count_dev;
        da.set_mass = set_mass.as<double>();
        da.first_item = s0;
        da.n_items = nbatch;
        da.b = b;
        da.stage = j;
        da.k0 = (uint32_t)seed;
        da.k1 = (uint32_t)(seed >> 32);
        da.vanish = pl->vanish;
        da.neg_abs = pl->neg_abs;
        da.neg_rel = pl->neg_rel;
        log.begin(&stats->descent_ms[j - 1]);
        launch_descent(pl, da, dsh);
        log.end();
      }
      stats->descent_items[j - 1] += U;
      }
    } else {
    uint32_t B = (uint32_t)std::max<size_t>(1, std::min<size_t>(U, pl->probs_budget / (nb * real)));
    DevBuf probs((size_t)B * nb * real, st), mass((size_t)B * 8, st), minv((size_t)B * 8, st);
    DevBuf vbuf;
    // complex64 projections with long runs of items per error set go to the tensor cores
    // (project_tc.cuh): v as one row per item, B_e images built once per error set for this stage
    TcShape tcs;
    if (proj && pl->tc_project && pl->dtype == PTSBE_C64 && (uint64_t)U >= 64ull * ne)
      tcs = tc_shape(progs[j - 1].d.proj_d, nb);
    DevBuf tc_bhi, tc_blo;
    if (tcs.ok) {
      vbuf.alloc((size_t)B * tcs.K * 4, st);
      if (tcs.K != 2 * progs[j - 1].d.proj_d) CK(cudaMemsetAsync(vbuf.p, 0, (size_t)B * tcs.K * 4, st));
      tc_bhi.alloc((size_t)ne * nb * tcs.K * 4, st);
      tc_blo.alloc((size_t)ne * nb * tcs.K * 4, st);
      log.begin(&stats->project_ms[j - 1]);
      launch_tc_prep(pl, table[1].ext, table[1].ext_rec, progs[j - 1].d.result_ref, ne, progs[j - 1].d.proj_d, nb, tcs,
                     tc_bhi.as<float>(), tc_blo.as<float>());
      log.end();
    } else if (proj) {
      vbuf.alloc((size_t)vec_pitch(B) * progs[j - 1].d.proj_d * pl->elem, st);
    }
    for (uint32_t s0 = 0; s0 < U; s0 += B) {
      const uint32_t nbatch = std::min(B, U - s0);
      log.begin(&stats->marg_ms[j - 1]);
      if (tcs.ok) {
        launch_exec_any(pl, progs[j - 1], EXEC_VECTOR, table_dev.as<LevelDev>(), kraus_dev, s0,
                        nbatch, vbuf.p, nullptr, nullptr, 0, tcs.K / 2);
        log.end();
        log.begin(&stats->project_ms[j - 1]);
        launch_project_tc(pl, tcs, vbuf.p, tc_bhi.as<float>(), tc_blo.as<float>(), ne, cur.eset.as<uint32_t>(), s0,
                          nbatch, nb, probs.p);
      } else if (proj) {
        launch_exec_any(pl, progs[j - 1], EXEC_VECTOR, table_dev.as<LevelDev>(), kraus_dev, s0,
                        nbatch, vbuf.p, nullptr, nullptr, vec_pitch(nbatch));
        log.end();
        log.begin(&stats->project_ms[j - 1]);
        launch_project(pl, progs[j - 1], vbuf.p, vec_pitch(nbatch), table[1].ext, table[1].ext_rec,
                       cur.eset.as<uint32_t>(), s0, nbatch, probs.p);
      } else if (j == 1 && progs[0].lane_big_ok && progs[0].d.result_kind == 0 && pl->lane && U >= pl->lane_big_min) {
        // stage 1 over a large batch of error sets: one thread per error set (lane.cuh BIG)
        if (pl->dtype == PTSBE_C64)
          launch_lane_big<float>(pl, progs[0], EXEC_MARGINAL, table_dev.as<LevelDev>(), kraus_dev, s0, nbatch,
                                 probs.p, mass.as<double>(), minv.as<double>());
        else
          launch_lane_big<double>(pl, progs[0], EXEC_MARGINAL, table_dev.as<LevelDev>(), kraus_dev, s0, nbatch,
                                  probs.p, mass.as<double>(), minv.as<double>());
      } else {
        launch_exec_any(pl, progs[j - 1], EXEC_MARGINAL, table_dev.as<LevelDev>(), kraus_dev, s0,
                        nbatch, probs.p, mass.as<double>(), minv.as<double>());
      }
      log.end();
      stats->marg_launches[j - 1]++;
      SampleArgs sa;
      memset(&sa, 0, sizeof sa);
      sa.probs = probs.p;
      sa.mult = cur.mult.as<uint32_t>();
      sa.slot_off = cur.slot_off.as<uint32_t>();
      sa.eset_id = cur.gid.as<uint32_t>();
      sa.rank = cur.rank.as<uint32_t>();
      sa.mass = proj ? nullptr : mass.as<double>();
      sa.minv = proj ? nullptr : minv.as<double>();
      sa.slot_index = slot_index.as<uint32_t>();
      sa.slot_count = slot_count.as<uint32_t>();
      sa.nnz = nnz.as<uint32_t>();
      sa.flag = flag_dev;
      sa.flag_count = flag_count_dev;
      sa.n_items = nbatch;
      sa.first_item = s0;
      sa.b = b;
      sa.stage = j;
      sa.k0 = (uint32_t)seed;
      sa.k1 = (uint32_t)(seed >> 32);
      sa.is_f32 = pl->dtype == PTSBE_C64;
      sa.vanish = pl->vanish;
      sa.set_mass = set_mass.as<double>();
      sa.eset_row = cur.eset.as<uint32_t>();
      sa.vanish_stage1 = pl->vanish_stage1;
      sa.neg_abs = pl->neg_abs;
      sa.neg_rel = pl->neg_rel;
      sa.np_mode = 0;
      sa.np_floor_bits = pl->dtype == PTSBE_C64 ? 17 : 40;
      sa.child_mult = 0;
      sa.threshold = 0.0;
      sa.slot_prob = nullptr;
      if (npp && j < f) {
        sa.np_mode = 1;
        sa.child_mult = np_mult(j + 1);
      } else if (np_exhaustive && j == f) {
        sa.np_mode = 2;
        sa.child_mult = 1;
        sa.threshold = npp->threshold;
        sa.slot_prob = slot_prob.as<double>();
      }
      log.begin(&stats->sampler_ms[j - 1]);
      launch_sampler(st, sa, pl->sm_count);
      log.end();
    }
    }
    // compaction into level j+1
    log.begin(&stats->compact_ms[j - 1]);
    DevBuf child_base((size_t)U * 4, st);
    exclusive_scan<uint32_t, uint32_t>(nnz.as<uint32_t>(), child_base.as<uint32_t>(), U,
                                       scal.as<uint32_t>(), st);
    uint32_t Un = 0;
    CK(cudaMemcpyAsync(&Un, scal.p, 4, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    Level& nx = lv[j + 1];
    nx.n = Un;
    if (j == f) {  // the final level is the chunk's output: it outlives the chunk's temporaries
      nx.eset.alloc((size_t)Un * 4, ws_out);
      nx.prefix.alloc((size_t)Un * 8 * words, ws_out);
      nx.mult.alloc((size_t)Un * 4, ws_out);
    } else {
      nx.eset.alloc((size_t)Un * 4, st);
      nx.prefix.alloc((size_t)Un * 8 * words, st);
      nx.mult.alloc((size_t)Un * 4, st);
    }
    nx.parent.alloc((size_t)Un * 4, st);
    if (Un) {
      ExpandArgs ea;
      ea.p_eset = cur.eset.as<uint32_t>();
      ea.p_prefix = cur.prefix.as<uint64_t>();
      ea.p_n = U;
      ea.p_slot_off = cur.slot_off.as<uint32_t>();
      ea.child_base = child_base.as<uint32_t>();
      ea.slot_index = slot_index.as<uint32_t>();
      ea.slot_count = slot_count.as<uint32_t>();
      ea.c_eset = nx.eset.as<uint32_t>();
      ea.c_parent = nx.parent.as<uint32_t>();
      ea.c_prefix = nx.prefix.as<uint64_t>();
      ea.c_mult = nx.mult.as<uint32_t>();
      ea.c_n = Un;
      ea.words = words;
      ea.offset = pl->offsets[j - 1];
      ea.b = b;
      ea.p_rank = ea.p_gid = nullptr;
      ea.c_rank = ea.c_gid = nullptr;
      if (j < f) {  // rank and global id of the children, written by the expansion itself
        nx.rank.alloc((size_t)Un * 4, st);
        nx.gid.alloc((size_t)Un * 4, st);
        ea.p_rank = cur.rank.as<uint32_t>();
        ea.p_gid = cur.gid.as<uint32_t>();
        ea.c_rank = nx.rank.as<uint32_t>();
        ea.c_gid = nx.gid.as<uint32_t>();
      }
      // few children per parent (late stages): parent-side scatter; otherwise child-side binary search
      if (words <= 4 && (uint64_t)Un <= 4ull * U)
        expand_scatter_kernel<<<cdiv(U, T), T, 0, st>>>(ea, nnz.as<uint32_t>());
      else
        expand_kernel<<<cdiv(Un, T), T, 0, st>>>(ea);
      g_launches++;
      if (np_exhaustive && j == f) {
        out.probs.alloc((size_t)Un * 8, ws_out);
        gather_prob_kernel<<<cdiv(Un, T), T, 0, st>>>(nx.parent.as<uint32_t>(), child_base.as<uint32_t>(),
                                                      cur.slot_off.as<uint32_t>(), slot_prob.as<double>(),
                                                      out.probs.as<double>(), Un);
        g_launches++;
      }
      if (j < f) {
        nx.slot_off.alloc((size_t)Un * 4, st);
        exclusive_scan<uint32_t, uint32_t>(nx.mult.as<uint32_t>(), nx.slot_off.as<uint32_t>(), Un,
                                           nullptr, st);
      }
    }
    CK(cudaGetLastError());
    log.end();
    CK(cudaEventRecord(ev[j], st));
    eager_hoists(j + 1);  // level j+1 is complete: its hoist passes of all later stages can start
    for (auto& buf : sext[j]) buf.release();
    // parents' per-stage arrays are no longer needed (lists stay for ancestor lookups)
    cur.mult.release();
    cur.slot_off.release();
    cur.rank.release();
    cur.gid.release();
  }
  CK(cudaStreamSynchronize(st));
  log.flush();
  for (uint32_t j = 1; j <= f; ++j) {
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, ev[j - 1], ev[j]));
    stats->stage_ms[j - 1] += ms;
  }
  for (auto& e : ev) cudaEventDestroy(e);
  Level& fin = lv[f + 1];
  out.n = fin.n;
  out.eset = std::move(fin.eset);
  out.keys = std::move(fin.prefix);
  out.counts = std::move(fin.mult);
}

}  // namespace ptsbe

// ---------------------------------------------------------------------------
// resident batch
// ---------------------------------------------------------------------------
struct ptsbe_batch {
  ptsbe_plan* plan = nullptr;
  uint64_t n_sets = 0, total_shots = 0;
  std::vector<uint32_t> shots_host;
  DevBuf kraus, shots, ids;
  std::unique_ptr<Workspace> ws_tmp_own;  // temporaries of one chunk (rewound after every chunk)
  std::unique_ptr<Workspace> ws_out_own;  // chunk outputs and the merged histogram (reset at the start of a run)
  Workspace& ws_tmp() { return *ws_tmp_own; }
  Workspace& ws_out() { return *ws_out_own; }
  // last run
  Histogram merged;
  RunOutput per_set;  // when merged == 0 (single chunk only)
  bool have_per_set = false;
};

namespace ptsbe {

// Kraus indices must address a variant the plan's tables hold (reference merge_errors raises on an
// unknown label, engine.py:300-312; here an out-of-range index would gather outside the pool).
__global__ void check_kraus_kernel(const uint8_t* kraus, const uint8_t* variants, uint64_t n, uint32_t g,
                                   unsigned long long* first_bad) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    if (kraus[i] >= variants[i % g]) atomicMin(first_bad, (unsigned long long)i);
}

static void check_kraus(ptsbe_plan* pl, const uint8_t* kraus_dev, uint64_t n_sets) {
  if (!pl->site_variants.p || !pl->g || !n_sets) return;
  cudaStream_t st = pl->stream;
  DevBuf bad(8, st);
  CK(cudaMemsetAsync(bad.p, 0xff, 8, st));
  const uint64_t n = n_sets * pl->g;
  const unsigned grid = (unsigned)std::min<uint64_t>(cdiv(n, 256), (uint64_t)pl->sm_count * 8);
  check_kraus_kernel<<<grid, 256, 0, st>>>(kraus_dev, pl->site_variants.as<uint8_t>(), n, pl->g,
                                           bad.as<unsigned long long>());
  g_launches++;
  CK(cudaGetLastError());
  unsigned long long first = 0;
  CK(cudaMemcpyAsync(&first, bad.p, 8, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (first != ~0ull)
    throw Failure(PTSBE_EINVAL, "Kraus index out of range: error set row " + std::to_string(first / pl->g) +
                                    ", site " + std::to_string(first % pl->g) +
                                    " addresses a variant this plan's tables do not hold");
}

// Joins per-chunk record lists (level f+1 of run_chunk) into one: keys [words][n] SoA, counts,
// error-set rows offset by the chunk's first set, probability tags when every chunk carries them.
static void concat_outputs(std::vector<RunOutput>& outs, const std::vector<uint64_t>& first_set,
                           uint32_t words, RunOutput& all, cudaStream_t st) {
  uint64_t total = 0;
  bool tags = true;
  for (auto& o : outs) { total += o.n; tags = tags && (o.n == 0 || o.probs.p != nullptr); }
  all = RunOutput();
  all.n = total;
  if (!total) return;
  all.keys.alloc(total * 8 * words, st);
  all.counts.alloc(total * 4, st);
  all.eset.alloc(total * 4, st);
  if (tags) all.probs.alloc(total * 8, st);
  uint64_t off = 0;
  for (size_t c = 0; c < outs.size(); ++c) {
    RunOutput& o = outs[c];
    if (!o.n) continue;
    for (uint32_t w = 0; w < words; ++w)
      CK(cudaMemcpyAsync(all.keys.as<uint64_t>() + (uint64_t)w * total + off,
                         o.keys.as<uint64_t>() + (uint64_t)w * o.n, o.n * 8, cudaMemcpyDeviceToDevice, st));
    CK(cudaMemcpyAsync(all.counts.as<uint32_t>() + off, o.counts.p, o.n * 4, cudaMemcpyDeviceToDevice, st));
    add_offset_u32_kernel<<<cdiv(o.n, 256), 256, 0, st>>>(o.eset.as<uint32_t>(), all.eset.as<uint32_t>() + off,
                                                          o.n, (uint32_t)first_set[c]);
    g_launches++;
    CK(cudaGetLastError());
    if (tags) CK(cudaMemcpyAsync(all.probs.as<double>() + off, o.probs.p, o.n * 8, cudaMemcpyDeviceToDevice, st));
    off += o.n;
  }
}

static void run_batch(ptsbe_batch* bt, uint64_t seed, int merged, ptsbe_run_stats* stats) {
  ptsbe_plan* pl = bt->plan;
  cudaStream_t st = pl->stream;
  CK(cudaSetDevice(pl->device));
  memset(stats, 0, sizeof *stats);
  stats->first_flagged_id = -1;
  stats->total_shots = bt->total_shots;
  g_launches = 0;
  bt->ws_tmp().reset();
  bt->ws_out().reset();
  bt->merged = Histogram();
  bt->per_set = RunOutput();
  WorkspaceScope scope(&bt->ws_out());  // flags, concatenation and the histogram live in ws_out
  DevBuf flag(16, st);
  CK(cudaMemsetAsync(flag.p, 0xff, 8, st));
  CK(cudaMemsetAsync(flag.as<unsigned char>() + 8, 0, 8, st));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaEventRecord(e0, st));

  // chunk the error sets: bounded shots (slot arrays) and bounded hoist records
  std::vector<std::pair<uint64_t, uint64_t>> chunks;  // (first set, count)
  {
    // hoist-record bound of a chunk of `cnt` error sets with `sh` shots: records of pass p exist for
    // every level-(p+1) item
    std::vector<double> fan(pl->f + 1);
    for (uint32_t p = 0; p <= pl->f; ++p) fan[p] = std::pow(2.0, std::min<uint32_t>(pl->offsets[std::min(p, pl->f - 1)], 60));
    // early hoist passes keep the records of all stages alive at once (decided for the whole batch: the walk
    // below runs once per error set)
    const bool sum_stages = pl->prelaunch && !chunk_is_dense(pl, bt->n_sets, bt->total_shots);
    auto ext_bytes_of = [&](uint64_t sh, uint64_t cnt) {
      size_t worst = 0;
      for (uint32_t j = 1; j <= pl->f; ++j) {
        size_t here = 0;
        for (uint32_t p = 0; p + 1 < j; ++p) {
          const double cap_items = std::min<double>((double)sh, (double)cnt * fan[p]);
          here += (size_t)(cap_items * pl->programs[j - 1][p].d.out_elems * pl->elem);
        }
        // early hoist passes (run_chunk) keep the records of ALL stages alive at once
        worst = sum_stages ? worst + here : std::max(worst, here);
      }
      return worst;
    };
    uint64_t e = 0;
    // the whole batch fits one chunk (the usual case): no walk over the error sets, which costs
    // milliseconds of idle GPU at 10^5 sets
    if (bt->n_sets && bt->total_shots <= pl->chunk_shots && bt->total_shots < (1ull << 32) &&
        ext_bytes_of(bt->total_shots, bt->n_sets) <= pl->ext_budget) {
      chunks.push_back({0, bt->n_sets});
      e = bt->n_sets;
    }
    while (e < bt->n_sets) {
      uint64_t cnt = 0, sh = 0;
      while (e + cnt < bt->n_sets) {
        const uint64_t s = bt->shots_host[e + cnt];
        if (cnt && sh + s > pl->chunk_shots) break;
        if (cnt && ext_bytes_of(sh + s, cnt + 1) > pl->ext_budget) break;
        sh += s;
        ++cnt;
      }
      if (sh >= (1ull << 32)) throw Failure(PTSBE_ECAPACITY, "one error set with >= 2^32 shots");
      chunks.push_back({e, cnt});
      e += cnt;
    }
  }
  stats->n_chunks = (uint32_t)chunks.size();
  const uint32_t words = pl->words;
  std::vector<RunOutput> outs(chunks.size());
  uint64_t total_rec = 0;
  for (size_t c = 0; c < chunks.size(); ++c) {
    const uint64_t e = chunks[c].first, cnt = chunks[c].second;
    uint64_t sh = 0;
    for (uint64_t i = 0; i < cnt; ++i) sh += bt->shots_host[e + i];
    {
      WorkspaceScope chunk_scope(&bt->ws_tmp());
      const Workspace::Mark mark = bt->ws_tmp().mark();
      run_chunk(pl, bt->kraus.as<uint8_t>() + e * pl->g, bt->shots.as<uint32_t>() + e,
                bt->ids.as<uint32_t>() + e, (uint32_t)cnt, sh, seed, outs[c], stats,
                flag.as<unsigned long long>(), flag.as<uint32_t>() + 2, bt->ws_out(), nullptr, merged != 0);
      bt->ws_tmp().rewind(mark);  // run_chunk returns with the stream drained
    }
    total_rec += outs[c].n;
  }
  // flags
  struct { unsigned long long first; uint32_t count; uint32_t pad; } fl;
  CK(cudaMemcpyAsync(&fl, flag.p, 16, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  stats->flagged_sets = fl.count;
  if (fl.count) {
    stats->first_flag_kind = (uint32_t)(fl.first & 0xff);
    stats->first_flag_stage = (uint32_t)((fl.first >> 8) & 0xff);
    stats->first_flagged_id = (int64_t)(fl.first >> 16);
  }
  bt->have_per_set = false;
  EventLog hlog(st);
  hlog.begin(&stats->histogram_ms);
  WorkspaceScope hist_scope(&bt->ws_tmp());  // sort/scan temporaries and the histogram: until the next run
  if (merged) {
    if (chunks.size() == 1) {
      reduce_by_key(outs[0].keys.as<uint64_t>(), outs[0].n, words, outs[0].counts.as<uint32_t>(),
                    nullptr, outs[0].n, pl->n, bt->merged, st, outs[0].unit_counts);
    } else {
      // concatenate chunk records (SoA with common stride), then reduce
      DevBuf keys(total_rec * 8 * words, st), counts(total_rec * 4, st);
      uint64_t off = 0;
      for (auto& o : outs) {
        for (uint32_t w = 0; w < words; ++w)
          CK(cudaMemcpyAsync(keys.as<uint64_t>() + (uint64_t)w * total_rec + off,
                             o.keys.as<uint64_t>() + (uint64_t)w * o.n, o.n * 8,
                             cudaMemcpyDeviceToDevice, st));
        CK(cudaMemcpyAsync(counts.as<uint32_t>() + off, o.counts.p, o.n * 4,
                           cudaMemcpyDeviceToDevice, st));
        off += o.n;
      }
      reduce_by_key(keys.as<uint64_t>(), total_rec, words, counts.as<uint32_t>(), nullptr,
                    total_rec, pl->n, bt->merged, st);
    }
    stats->n_records = bt->merged.n;
  } else {
    if (chunks.size() == 1) {
      bt->per_set = std::move(outs[0]);
    } else {
      // concatenate the chunks' records: keys are SoA with the record count as stride, error-set rows
      // are relative to the chunk's first set (the reference's per-set API has no size limit,
      // engine.py:493-524)
      std::vector<uint64_t> first_set;
      for (auto& ch : chunks) first_set.push_back(ch.first);
      concat_outputs(outs, first_set, words, bt->per_set, st);
    }
    bt->have_per_set = true;
    stats->n_records = bt->per_set.n;
  }
  hlog.end();
  CK(cudaEventRecord(e1, st));
  CK(cudaStreamSynchronize(st));
  hlog.flush();
  CK(cudaEventElapsedTime(&stats->loop_ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  stats->gpu_launches = g_launches;
}

template <typename F>
static int guarded(F&& fn) {
  try {
    fn();
    return PTSBE_OK;
  } catch (const Failure& e) {
    g_last_error = e.what();
    return e.code;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return PTSBE_EDEVICE;
  }
}

}  // namespace ptsbe

namespace ptsbe {
template <typename T>
__global__ void fma_peak_kernel(T* out, int iters) {
  T a0 = threadIdx.x * T(1e-3), a1 = a0 + T(1), a2 = a0 + T(2), a3 = a0 + T(3);
  T a4 = a0 + T(4), a5 = a0 + T(5), a6 = a0 + T(6), a7 = a0 + T(7);
  const T m = T(0.999), c = T(1e-4);
  for (int i = 0; i < iters; ++i) {
    a0 = fma(a0, m, c); a1 = fma(a1, m, c); a2 = fma(a2, m, c); a3 = fma(a3, m, c);
    a4 = fma(a4, m, c); a5 = fma(a5, m, c); a6 = fma(a6, m, c); a7 = fma(a7, m, c);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}
template <typename T>
static double fma_peak(int sm_count, int iters) {
  const int blocks = sm_count * 8, threads = 256;
  DevBuf out((size_t)blocks * threads * sizeof(T), nullptr);
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  fma_peak_kernel<T><<<blocks, threads>>>(out.as<T>(), iters / 8);
  float best = 1e30f;
  for (int r = 0; r < 3; ++r) {
    CK(cudaEventRecord(a));
    fma_peak_kernel<T><<<blocks, threads>>>(out.as<T>(), iters);
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, a, b));
    best = std::min(best, ms);
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  CK(cudaDeviceSynchronize());
  return 2.0 * 8.0 * iters * (double)blocks * threads / (best * 1e-3) / 1e12;
}
}  // namespace ptsbe

extern "C" {

const char* ptsbe_last_error(void) { return g_last_error.c_str(); }
const char* ptsbe_version(void) { return "ptsbe_b200 0.1 (sm_100a)"; }

int ptsbe_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

void ptsbe_free(void* p) {
  if (p && !g_host_pool.put(p)) free(p);
}

int ptsbe_plan_create(const ptsbe_plan_desc* d, int device, ptsbe_plan** out) {
  return guarded([&] {
    if (!d || !out) throw Failure(PTSBE_EINVAL, "null plan descriptor");
    if (d->dtype > 1) throw Failure(PTSBE_EINVAL, "dtype must be PTSBE_C64 or PTSBE_C128");
    if (d->n_stages < 1 || d->n_stages > PTSBE_MAX_STAGES)
      throw Failure(PTSBE_ECAPACITY, "stage count outside 1..PTSBE_MAX_STAGES");
    if (ptsbe_device_count() <= device)
      throw Failure(PTSBE_EDEVICE, "no CUDA device: libptsbe_b200 has no CPU fallback");
    CK(cudaSetDevice(device));
    std::unique_ptr<ptsbe_plan> pl(new ptsbe_plan);
    pl->device = device;
    pl->dtype = d->dtype;
    pl->n = d->n_qubits;
    pl->g = d->n_sites;
    pl->f = d->n_stages;
    pl->words = std::max<uint32_t>(1, (d->n_qubits + 63) / 64);
    pl->elem = d->dtype == PTSBE_C64 ? 8 : 16;
    uint32_t off = 0;
    for (uint32_t j = 0; j < d->n_stages; ++j) {
      pl->sizes.push_back(d->stage_sizes[j]);
      pl->offsets.push_back(off);
      off += d->stage_sizes[j];
    }
    if (off != d->n_qubits) throw Failure(PTSBE_EINVAL, "stage sizes do not sum to n_qubits");
    if (d->dtype == PTSBE_C64) { pl->neg_abs = -1e-12; pl->neg_rel = 1e-4; }
    {
      int lo = 0, hi = 0;
      CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
      pl->side_priority = (uint32_t)env_size("PTSBE_SIDE_PRIORITY", 1);
      CK(cudaStreamCreateWithPriority(&pl->stream, cudaStreamNonBlocking, pl->side_priority ? hi : lo));
    }
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, device));
    pl->sm_count = prop.multiProcessorCount;
    cudaMemPool_t mp;
    CK(cudaDeviceGetDefaultMemPool(&mp, device));
    uint64_t thr = UINT64_MAX;
    CK(cudaMemPoolSetAttribute(mp, cudaMemPoolAttrReleaseThreshold, &thr));
    pl->probs_budget = env_size("PTSBE_PROBS_BYTES", pl->probs_budget);
    pl->vec_budget = env_size("PTSBE_VEC_BYTES", pl->vec_budget);
    pl->descent = (uint32_t)env_size("PTSBE_DESCENT", pl->descent);
    pl->tc_project = (uint32_t)env_size("PTSBE_TC_PROJECT", pl->tc_project);
    pl->lane_x = (uint32_t)env_size("PTSBE_LANE_X", pl->lane_x);
    pl->lane_chain = (uint32_t)env_size("PTSBE_LANE_CHAIN", pl->lane_chain);
    pl->lane_big_min = (uint32_t)env_size("PTSBE_LANE_BIG_MIN", pl->lane_big_min);
    pl->raw_final = env_size("PTSBE_RAW_FINAL", 1) != 0;
    pl->stage_image = (uint32_t)env_size("PTSBE_STAGE_IMAGE", pl->stage_image);
    pl->warp_runs = (uint32_t)env_size("PTSBE_WARP_RUNS", pl->warp_runs);
    pl->tiled_plain = (uint32_t)env_size("PTSBE_TILED_PLAIN", pl->tiled_plain);
    pl->tc_steps = (uint32_t)env_size("PTSBE_TC_STEPS", pl->tc_steps);
    pl->tree_herm = (uint32_t)env_size("PTSBE_TREE_HERM", pl->tree_herm);
    pl->lane_tiny = (uint32_t)env_size("PTSBE_LANE_TINY", pl->lane_tiny);
    pl->descent_tile_max = (uint32_t)env_size("PTSBE_DESCENT_TILE_MAX", pl->descent_tile_max);
    pl->tile_min = (uint32_t)env_size("PTSBE_TILE_MIN", pl->tile_min);
    pl->prelaunch = (uint32_t)env_size("PTSBE_PRELAUNCH", pl->prelaunch);
    pl->prelaunch_max = (uint32_t)env_size("PTSBE_PRELAUNCH_MAX", pl->prelaunch_max);
    if (const char* v = getenv("PTSBE_EAGER_WORK_MAX")) pl->eager_work_max = atof(v);
    pl->warp_run_len = (uint32_t)env_size("PTSBE_WARP_RUN_LEN", pl->warp_run_len);
    pl->stage_image_max = (uint32_t)env_size("PTSBE_STAGE_IMAGE_MAX", pl->stage_image_max);
    pl->lane = (uint32_t)env_size("PTSBE_LANE", pl->lane);
    if (const char* dm = getenv("PTSBE_DESCENT_MULT")) if (*dm) pl->descent_mult = atof(dm);
    pl->chunk_shots = env_size("PTSBE_CHUNK_SHOTS", pl->chunk_shots);
    pl->ext_budget = env_size("PTSBE_EXT_BYTES", pl->ext_budget);
    pl->stage_descent.assign(d->n_stages, -1);
    const bool use_memo = env_size("PTSBE_MEMO", 1) != 0;  // variant-0 memo of class-0 programs
    cudaStream_t st = pl->stream;
    pl->pool.alloc(std::max<size_t>(16, d->pool_elems * pl->elem), st);
    if (d->pool_elems)
      CK(cudaMemcpyAsync(pl->pool.p, d->pool, d->pool_elems * pl->elem, cudaMemcpyHostToDevice, st));
    if (d->site_variants && d->n_sites) {
      pl->site_variants.alloc(d->n_sites, st);
      CK(cudaMemcpyAsync(pl->site_variants.p, d->site_variants, d->n_sites, cudaMemcpyHostToDevice, st));
    }
    size_t k = 0;
    pl->programs.resize(d->n_stages);
    for (uint32_t j = 1; j <= d->n_stages; ++j) {
      pl->programs[j - 1].resize(j);
      for (uint32_t p = 0; p < j; ++p, ++k) {
        Program& pr = pl->programs[j - 1][p];
        pr.d = d->programs[k];
        if (!use_memo) pr.d.memo_elems = 0;
        if (pr.d.level != p + 1) throw Failure(PTSBE_EINVAL, "program level does not match its pass");
        if (pr.d.result_kind == 3 && (p + 1 != j || j < 2 || pr.d.proj_d < 1))
          throw Failure(PTSBE_EINVAL, "projection form is only valid for the marginal pass of a stage >= 2");
        if (pr.d.threads_per_item > 256 ||
            ((pr.d.threads_per_item & 31) && pr.d.threads_per_item != 8 && pr.d.threads_per_item != 16))
          throw Failure(PTSBE_EINVAL, "threads_per_item must be 8, 16 or a multiple of 32 up to 256");
        pr.leaves.alloc(std::max<size_t>(16, (size_t)pr.d.n_leaves * LEAF_WORDS * 4), st);
        pr.steps.alloc(std::max<size_t>(16, (size_t)pr.d.n_steps * STEP_WORDS * 4), st);
        pr.tables.alloc(std::max<size_t>(16, (size_t)pr.d.n_table_words * 4), st);
        if (pr.d.n_leaves)
          CK(cudaMemcpyAsync(pr.leaves.p, pr.d.leaves, (size_t)pr.d.n_leaves * LEAF_WORDS * 4,
                             cudaMemcpyHostToDevice, st));
        if (pr.d.n_steps)
          CK(cudaMemcpyAsync(pr.steps.p, pr.d.steps, (size_t)pr.d.n_steps * STEP_WORDS * 4,
                             cudaMemcpyHostToDevice, st));
        if (pr.d.n_table_words)
          CK(cudaMemcpyAsync(pr.tables.p, pr.d.tables, (size_t)pr.d.n_table_words * 4,
                             cudaMemcpyHostToDevice, st));
        classify_lane(pl.get(), pr);
        if (pr.herm && env_size("PTSBE_HERM", 1)) {
          if (pr.herm_dx) {
            pr.herm_canon.alloc(pr.herm_canon_host.size() * 4, st);
            CK(cudaMemcpyAsync(pr.herm_canon.p, pr.herm_canon_host.data(), pr.herm_canon_host.size() * 4,
                               cudaMemcpyHostToDevice, st));
          }
          pr.herm_map.alloc(pr.herm_map_host.size() * 4, st);
          CK(cudaMemcpyAsync(pr.herm_map.p, pr.herm_map_host.data(), pr.herm_map_host.size() * 4,
                             cudaMemcpyHostToDevice, st));
        } else {
          pr.herm = false;
        }
        {
          double big = 0, all = 0;
          for (uint32_t q = 0; q < pr.d.n_steps && pr.d.steps; ++q) {
            const uint32_t* stw = pr.d.steps + (size_t)q * STEP_WORDS;
            const double macs = (double)stw[6] * std::max<uint32_t>(stw[7], 1);
            all += macs;
            if (stw[17]) big += macs;
          }
          pr.tiled = big >= 1.5e5 && big >= 0.5 * all;
          pr.macs = all;
        }
        if (pr.d.memo_elems) {
          if (!pr.d.memo_ptr || !pr.d.memo_idx || pr.d.n_memo_sites > pl->g || pr.d.n_steps >= 0xFFFF)
            throw Failure(PTSBE_EINVAL, "memo program without its site -> steps table");
          const size_t np = (size_t)pr.d.n_memo_sites + 2;
          pr.memo_ptr.alloc(np * 4, st);
          pr.memo_idx.alloc(std::max<size_t>(16, (size_t)pr.d.n_memo_idx * 4), st);
          CK(cudaMemcpyAsync(pr.memo_ptr.p, pr.d.memo_ptr, np * 4, cudaMemcpyHostToDevice, st));
          if (pr.d.n_memo_idx)
            CK(cudaMemcpyAsync(pr.memo_idx.p, pr.d.memo_idx, (size_t)pr.d.n_memo_idx * 4,
                               cudaMemcpyHostToDevice, st));
        }
        pr.d.leaves = pr.d.steps = pr.d.tables = pr.d.memo_ptr = pr.d.memo_idx = nullptr;
      }
    }
    CK(cudaStreamSynchronize(st));
    *out = pl.release();
  });
}

void ptsbe_plan_destroy(ptsbe_plan* pl) {
  if (!pl) return;
  cudaSetDevice(pl->device);
  cudaStreamSynchronize(pl->stream);
  pl->ws_cache.clear();
  pl->pool.release();
  pl->site_variants.release();  // every stream-ordered buffer goes before its stream does
  for (auto& s : pl->programs)
    for (auto& p : s) {
      p.leaves.release(); p.steps.release(); p.tables.release();
      p.memo_ptr.release(); p.memo_idx.release(); p.memo.release(); p.herm_map.release(); p.herm_canon.release();
    }
  cudaStreamSynchronize(pl->stream);
  for (cudaStream_t q : pl->side) { cudaStreamSynchronize(q); cudaStreamDestroy(q); }
  cudaStreamDestroy(pl->stream);
  delete pl;
}

int ptsbe_plan_set_stage_samplers(ptsbe_plan* pl, const int32_t* kinds, uint32_t n_stages) {
  return guarded([&] {
    if (!pl || !kinds) throw Failure(PTSBE_EINVAL, "null argument");
    if (n_stages != pl->f) throw Failure(PTSBE_EINVAL, "one sampler kind per stage expected");
    std::lock_guard<std::mutex> lock(pl->mu);
    for (uint32_t j = 0; j < n_stages; ++j) {
      if (kinds[j] < -1 || kinds[j] > 1) throw Failure(PTSBE_EINVAL, "sampler kind must be -1 (auto), 0 (flat) or 1 (descent)");
      pl->stage_descent[j] = kinds[j];
    }
  });
}

int ptsbe_marginals(ptsbe_plan* pl, uint32_t stage, const uint8_t* kraus_idx,
                    const uint64_t* prefixes, uint64_t n_items, double* out_probs,
                    double* out_mass, double* out_min) {
  return guarded([&] {
    if (!pl) throw Failure(PTSBE_EINVAL, "null plan");
    if (stage < 1 || stage > pl->f) throw Failure(PTSBE_EINVAL, "stage outside 1..f");
    std::lock_guard<std::mutex> lock(pl->mu);
    CK(cudaSetDevice(pl->device));
    g_launches = 0;
    cudaStream_t st = pl->stream;
    const uint32_t j = stage, words = pl->words, f = pl->f;
    auto& progs = pl->programs[j - 1];
    const uint32_t nb = progs[j - 1].d.out_elems;
    const size_t real = pl->dtype == PTSBE_C64 ? 4 : 8;
    size_t per_item = (size_t)nb * real;
    for (uint32_t p = 0; p + 1 < j; ++p) per_item += (size_t)progs[p].d.out_elems * pl->elem;
    const uint64_t chunk = std::max<uint64_t>(1, std::min<uint64_t>(65536, (1ull << 30) / per_item));
    std::vector<LevelDev> table(f + 2);
    DevBuf table_dev((f + 2) * sizeof(LevelDev), st);
    std::vector<unsigned char> host(chunk * nb * real);
    for (uint64_t c0 = 0; c0 < n_items; c0 += chunk) {
      const uint32_t W = (uint32_t)std::min<uint64_t>(chunk, n_items - c0);
      DevBuf kraus((size_t)W * std::max<uint32_t>(pl->g, 1), st), ident((size_t)W * 4, st),
          pfx((size_t)W * 8 * words, st);
      if (pl->g)
        CK(cudaMemcpyAsync(kraus.p, kraus_idx + c0 * pl->g, (size_t)W * pl->g,
                           cudaMemcpyHostToDevice, st));
      check_kraus(pl, kraus.as<uint8_t>(), W);
      // prefixes arrive item-major [W][words]; the device wants [words][W]
      std::vector<uint64_t> soa((size_t)W * words);
      for (uint32_t i = 0; i < W; ++i)
        for (uint32_t w = 0; w < words; ++w)
          soa[(size_t)w * W + i] = prefixes ? prefixes[(c0 + i) * words + w] : 0;
      CK(cudaMemcpyAsync(pfx.p, soa.data(), soa.size() * 8, cudaMemcpyHostToDevice, st));
      iota_kernel<<<cdiv(W, 256), 256, 0, st>>>(ident.as<uint32_t>(), W, 0);
      g_launches++;
      memset(table.data(), 0, sizeof(LevelDev) * table.size());
      std::vector<DevBuf> ext(j);
      for (uint32_t l = 1; l <= j; ++l) {
        table[l].eset = ident.as<uint32_t>();
        table[l].parent = ident.as<uint32_t>();
        table[l].prefix = pfx.as<uint64_t>();
        table[l].n = W;
        if (l < j && progs[l - 1].d.out_elems && progs[l - 1].d.n_steps) {
          ext[l - 1].alloc((size_t)W * progs[l - 1].d.out_elems * pl->elem, st);
          table[l].ext = ext[l - 1].p;
          table[l].ext_rec = progs[l - 1].d.out_elems;
        }
      }
      CK(cudaMemcpyAsync(table_dev.p, table.data(), sizeof(LevelDev) * (f + 2),
                         cudaMemcpyHostToDevice, st));
      for (uint32_t p = 0; p + 1 < j; ++p)
        if (progs[p].d.n_steps)
          launch_exec_any(pl, progs[p], EXEC_HOIST, table_dev.as<LevelDev>(), kraus.as<uint8_t>(),
                          0, W, ext[p].p, nullptr, nullptr);
      DevBuf probs((size_t)W * nb * real, st), mass((size_t)W * 8, st), minv((size_t)W * 8, st);
      if (progs[j - 1].d.result_kind == 3) {
        DevBuf vbuf((size_t)vec_pitch(W) * progs[j - 1].d.proj_d * pl->elem, st);
        CK(cudaMemsetAsync(vbuf.p, 0, vbuf.bytes, st));
        launch_exec_any(pl, progs[j - 1], EXEC_VECTOR, table_dev.as<LevelDev>(), kraus.as<uint8_t>(),
                        0, W, vbuf.p, nullptr, nullptr, vec_pitch(W));
        launch_project(pl, progs[j - 1], vbuf.p, vec_pitch(W), table[1].ext, table[1].ext_rec,
                       ident.as<uint32_t>(), 0, W, probs.p);
        if (pl->dtype == PTSBE_C64)
          row_stats_kernel<float><<<cdiv((uint64_t)W * 32, 256), 256, 0, st>>>(
              probs.as<float>(), W, nb, mass.as<double>(), minv.as<double>());
        else
          row_stats_kernel<double><<<cdiv((uint64_t)W * 32, 256), 256, 0, st>>>(
              probs.as<double>(), W, nb, mass.as<double>(), minv.as<double>());
        g_launches++;
      } else {
        launch_exec_any(pl, progs[j - 1], EXEC_MARGINAL, table_dev.as<LevelDev>(),
                        kraus.as<uint8_t>(), 0, W, probs.p, mass.as<double>(), minv.as<double>());
      }
      CK(cudaMemcpyAsync(host.data(), probs.p, (size_t)W * nb * real, cudaMemcpyDeviceToHost, st));
      if (out_mass) CK(cudaMemcpyAsync(out_mass + c0, mass.p, (size_t)W * 8, cudaMemcpyDeviceToHost, st));
      if (out_min) CK(cudaMemcpyAsync(out_min + c0, minv.p, (size_t)W * 8, cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      double* o = out_probs + c0 * nb;
      if (pl->dtype == PTSBE_C64) {
        const float* h = reinterpret_cast<const float*>(host.data());
        for (size_t i = 0; i < (size_t)W * nb; ++i) o[i] = (double)h[i];
      } else {
        memcpy(o, host.data(), (size_t)W * nb * 8);
      }
    }
  });
}

// Runs pass 0 of stage 1 of a plan in RAW mode for one item: complex result of a
// constant network (tensor.py execute_path / contract_pair on the device).
int ptsbe_execute_raw(ptsbe_plan* pl, void* out_complex) {
  return guarded([&] {
    if (!pl) throw Failure(PTSBE_EINVAL, "null plan");
    std::lock_guard<std::mutex> lock(pl->mu);
    CK(cudaSetDevice(pl->device));
    cudaStream_t st = pl->stream;
    Program& pr = pl->programs[0][0];
    std::vector<LevelDev> table(pl->f + 2);
    memset(table.data(), 0, sizeof(LevelDev) * table.size());
    DevBuf table_dev(table.size() * sizeof(LevelDev), st), ident(16, st), pfx(8 * pl->words, st),
        kraus(16, st), res((size_t)pr.d.out_elems * pl->elem, st);
    CK(cudaMemsetAsync(ident.p, 0, 16, st));
    CK(cudaMemsetAsync(pfx.p, 0, 8 * pl->words, st));
    CK(cudaMemsetAsync(kraus.p, 0, 16, st));
    table[1].eset = ident.as<uint32_t>();
    table[1].parent = ident.as<uint32_t>();
    table[1].prefix = pfx.as<uint64_t>();
    table[1].n = 1;
    CK(cudaMemcpyAsync(table_dev.p, table.data(), table.size() * sizeof(LevelDev),
                       cudaMemcpyHostToDevice, st));
    launch_exec_any(pl, pr, EXEC_RAW, table_dev.as<LevelDev>(), kraus.as<uint8_t>(), 0, 1, res.p,
                    nullptr, nullptr);
    CK(cudaMemcpyAsync(out_complex, res.p, (size_t)pr.d.out_elems * pl->elem,
                       cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
  });
}

int ptsbe_sample_stage(uint32_t b, uint32_t stage, uint64_t seed, uint64_t n_items,
                       const double* probs, const uint32_t* mult, const uint32_t* eset_id,
                       const uint32_t* rank, uint32_t** child_item, uint32_t** child_index,
                       uint32_t** child_count, uint64_t* n_children, int device) {
  return guarded([&] {
    if (ptsbe_device_count() <= device)
      throw Failure(PTSBE_EDEVICE, "no CUDA device: libptsbe_b200 has no CPU fallback");
    if (b > 14) throw Failure(PTSBE_ECAPACITY, "sampler supports stage batches of at most 14 qubits");
    CK(cudaSetDevice(device));
    g_launches = 0;
    cudaStream_t st;
    CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    {
      const uint64_t nb = 1ull << b;
      uint64_t shots = 0;
      for (uint64_t i = 0; i < n_items; ++i) shots += mult[i];
      DevBuf dp(n_items * nb * 8, st), dm(n_items * 4, st), de(n_items * 4, st), dr(n_items * 4, st),
          so(n_items * 4, st), si(std::max<uint64_t>(shots, 1) * 4, st),
          sc(std::max<uint64_t>(shots, 1) * 4, st), nnz(n_items * 4, st), flag(16, st),
          base(n_items * 4, st);
      CK(cudaMemcpyAsync(dp.p, probs, n_items * nb * 8, cudaMemcpyHostToDevice, st));
      CK(cudaMemcpyAsync(dm.p, mult, n_items * 4, cudaMemcpyHostToDevice, st));
      CK(cudaMemcpyAsync(de.p, eset_id, n_items * 4, cudaMemcpyHostToDevice, st));
      CK(cudaMemcpyAsync(dr.p, rank, n_items * 4, cudaMemcpyHostToDevice, st));
      CK(cudaMemsetAsync(flag.p, 0xff, 8, st));
      CK(cudaMemsetAsync(flag.as<unsigned char>() + 8, 0, 8, st));
      exclusive_scan<uint32_t, uint32_t>(dm.as<uint32_t>(), so.as<uint32_t>(), n_items, nullptr, st);
      SampleArgs sa;
      memset(&sa, 0, sizeof sa);
      memset(&sa, 0, sizeof sa);
      sa.probs = dp.p;
      sa.mult = dm.as<uint32_t>();
      sa.slot_off = so.as<uint32_t>();
      sa.eset_id = de.as<uint32_t>();
      sa.rank = dr.as<uint32_t>();
      sa.slot_index = si.as<uint32_t>();
      sa.slot_count = sc.as<uint32_t>();
      sa.nnz = nnz.as<uint32_t>();
      sa.flag = flag.as<unsigned long long>();
      sa.flag_count = flag.as<uint32_t>() + 2;
      sa.n_items = n_items;
      sa.b = b;
      sa.stage = stage;
      sa.k0 = (uint32_t)seed;
      sa.k1 = (uint32_t)(seed >> 32);
      sa.is_f32 = 0;
      sa.neg_abs = -1e-12;
      cudaDeviceProp prop;
      CK(cudaGetDeviceProperties(&prop, device));
      launch_sampler(st, sa, prop.multiProcessorCount);
      std::vector<uint32_t> h_nnz(n_items), h_so(n_items), h_si(shots), h_sc(shots);
      CK(cudaMemcpyAsync(h_nnz.data(), nnz.p, n_items * 4, cudaMemcpyDeviceToHost, st));
      CK(cudaMemcpyAsync(h_so.data(), so.p, n_items * 4, cudaMemcpyDeviceToHost, st));
      if (shots) {
        CK(cudaMemcpyAsync(h_si.data(), si.p, shots * 4, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(h_sc.data(), sc.p, shots * 4, cudaMemcpyDeviceToHost, st));
      }
      CK(cudaStreamSynchronize(st));
      uint64_t total = 0;
      for (uint64_t i = 0; i < n_items; ++i) total += h_nnz[i];
      uint32_t* ci = (uint32_t*)malloc(std::max<uint64_t>(total, 1) * 4);
      uint32_t* cx = (uint32_t*)malloc(std::max<uint64_t>(total, 1) * 4);
      uint32_t* cc = (uint32_t*)malloc(std::max<uint64_t>(total, 1) * 4);
      uint64_t k = 0;
      for (uint64_t i = 0; i < n_items; ++i)
        for (uint32_t c = 0; c < h_nnz[i]; ++c, ++k) {
          ci[k] = (uint32_t)i;
          cx[k] = h_si[h_so[i] + c];
          cc[k] = h_sc[h_so[i] + c];
        }
      *child_item = ci;
      *child_index = cx;
      *child_count = cc;
      *n_children = total;
    }
    cudaStreamSynchronize(st);
    cudaStreamDestroy(st);
  });
}

int ptsbe_batch_upload(ptsbe_plan* pl, const uint8_t* kraus_idx, const uint32_t* shots,
                       const uint32_t* eset_ids, uint64_t n_sets, ptsbe_batch** out) {
  return guarded([&] {
    if (!pl || !out) throw Failure(PTSBE_EINVAL, "null plan");
    if (n_sets < 1) throw Failure(PTSBE_EINVAL, "need at least one error set");
    if (n_sets >= (1ull << 32)) throw Failure(PTSBE_ECAPACITY, "more than 2^32 error sets");
    CK(cudaSetDevice(pl->device));
    std::unique_ptr<ptsbe_batch> bt(new ptsbe_batch);
    bt->plan = pl;
    bt->n_sets = n_sets;
    {
      std::lock_guard<std::mutex> lock(pl->mu);
      bt->ws_tmp_own = pl->take_workspace();
      bt->ws_out_own = pl->take_workspace();
    }
    bt->shots_host.assign(shots, shots + n_sets);
    for (uint64_t i = 0; i < n_sets; ++i) {
      if (shots[i] < 1) throw Failure(PTSBE_EINVAL, "proportional sampling needs m >= 1");
      bt->total_shots += shots[i];
    }
    cudaStream_t st = pl->stream;
    bt->kraus.alloc(std::max<size_t>(16, n_sets * pl->g), st);
    bt->shots.alloc(n_sets * 4, st);
    bt->ids.alloc(n_sets * 4, st);
    if (pl->g) CK(cudaMemcpyAsync(bt->kraus.p, kraus_idx, n_sets * pl->g, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(bt->shots.p, shots, n_sets * 4, cudaMemcpyHostToDevice, st));
    if (eset_ids) {
      CK(cudaMemcpyAsync(bt->ids.p, eset_ids, n_sets * 4, cudaMemcpyHostToDevice, st));
    } else {
      iota_kernel<<<cdiv(n_sets, 256), 256, 0, st>>>(bt->ids.as<uint32_t>(), (uint32_t)n_sets, 0);
    }
    CK(cudaStreamSynchronize(st));
    {
      std::lock_guard<std::mutex> lock(pl->mu);
      check_kraus(pl, bt->kraus.as<uint8_t>(), n_sets);
    }
    *out = bt.release();
  });
}

int ptsbe_batch_presample(ptsbe_plan* pl, const double* site_cdf, const uint32_t* site_off,
                          uint64_t n_sets, uint32_t first_id, uint32_t shots_per_set, uint64_t seed,
                          ptsbe_batch** out) {
  return guarded([&] {
    if (!pl || !out || !site_cdf || !site_off) throw Failure(PTSBE_EINVAL, "null argument");
    if (n_sets < 1 || n_sets >= (1ull << 32)) throw Failure(PTSBE_EINVAL, "need 1 .. 2^32 error sets");
    if (shots_per_set < 1) throw Failure(PTSBE_EINVAL, "proportional sampling needs m >= 1");
    if (site_off[0] != 0) throw Failure(PTSBE_EINVAL, "site_off must start at 0");
    for (uint32_t s = 0; s < pl->g; ++s)
      if (site_off[s + 1] <= site_off[s] || site_off[s + 1] - site_off[s] > 255)
        throw Failure(PTSBE_EINVAL, "every site needs 1 .. 255 outcomes");
    CK(cudaSetDevice(pl->device));
    std::unique_ptr<ptsbe_batch> bt(new ptsbe_batch);
    bt->plan = pl;
    bt->n_sets = n_sets;
    {
      std::lock_guard<std::mutex> lock(pl->mu);
      bt->ws_tmp_own = pl->take_workspace();
      bt->ws_out_own = pl->take_workspace();
    }
    bt->shots_host.assign(n_sets, shots_per_set);
    bt->total_shots = n_sets * (uint64_t)shots_per_set;
    cudaStream_t st = pl->stream;
    const uint32_t n_out = site_off[pl->g];
    bt->kraus.alloc(std::max<size_t>(16, n_sets * pl->g), st);
    bt->shots.alloc(n_sets * 4, st);
    bt->ids.alloc(n_sets * 4, st);
    DevBuf cdf((size_t)n_out * 8, st), off(((size_t)pl->g + 1) * 4, st);
    CK(cudaMemcpyAsync(cdf.p, site_cdf, (size_t)n_out * 8, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(off.p, site_off, ((size_t)pl->g + 1) * 4, cudaMemcpyHostToDevice, st));
    fill_u32_kernel<<<cdiv(n_sets, 256), 256, 0, st>>>(bt->shots.as<uint32_t>(), (uint32_t)n_sets, shots_per_set);
    iota_kernel<<<cdiv(n_sets, 256), 256, 0, st>>>(bt->ids.as<uint32_t>(), (uint32_t)n_sets, first_id);
    if (pl->g)
      presample_kernel<<<cdiv(n_sets * pl->g, 256), 256, 0, st>>>(
          cdf.as<double>(), off.as<uint32_t>(), pl->g, n_sets, first_id, (uint32_t)seed, (uint32_t)(seed >> 32),
          bt->kraus.as<uint8_t>());
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(st));
    *out = bt.release();
  });
}

int ptsbe_batch_kraus(ptsbe_batch* bt, uint8_t* out_host) {
  return guarded([&] {
    if (!bt || !out_host) throw Failure(PTSBE_EINVAL, "null argument");
    CK(cudaSetDevice(bt->plan->device));
    CK(cudaMemcpyAsync(out_host, bt->kraus.p, bt->n_sets * bt->plan->g, cudaMemcpyDeviceToHost, bt->plan->stream));
    CK(cudaStreamSynchronize(bt->plan->stream));
  });
}

int ptsbe_batch_run(ptsbe_batch* bt, uint64_t seed, uint64_t* n_records, ptsbe_run_stats* stats) {
  return guarded([&] {
    if (!bt) throw Failure(PTSBE_EINVAL, "null batch");
    ptsbe_run_stats local;
    std::lock_guard<std::mutex> lock(bt->plan->mu);
    run_batch(bt, seed, 1, stats ? stats : &local);
    if (n_records) *n_records = bt->merged.n;
  });
}

static void fetch_merged(ptsbe_batch* bt, uint64_t** keys, uint64_t** counts, uint64_t* n) {
  ptsbe_plan* pl = bt->plan;
  const uint64_t nr = bt->merged.n;
  uint64_t* k = (uint64_t*)g_host_pool.get(std::max<uint64_t>(nr, 1) * 8 * pl->words);
  uint64_t* c = (uint64_t*)g_host_pool.get(std::max<uint64_t>(nr, 1) * 8);
  if (!k || !c) throw Failure(PTSBE_ECAPACITY, "host allocation of the histogram failed");
  if (nr) {
    CK(cudaMemcpyAsync(k, bt->merged.keys.p, nr * 8 * pl->words, cudaMemcpyDeviceToHost, pl->stream));
    CK(cudaMemcpyAsync(c, bt->merged.counts.p, nr * 8, cudaMemcpyDeviceToHost, pl->stream));
    CK(cudaStreamSynchronize(pl->stream));
  }
  *keys = k;
  *counts = c;
  *n = nr;
}

// Merged histogram as [n][2] u32 (high half of the key word, count): plans of at most 32 measured qubits and runs of fewer
// than 2^32 shots need 8 bytes per record on the PCIe link instead of 16.
__global__ void pack_records_kernel(const uint64_t* __restrict__ keys, const uint64_t* __restrict__ counts,
                                    uint2* __restrict__ out, uint64_t n) {
  const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i < n) out[i] = make_uint2((uint32_t)(keys[i] >> 32), (uint32_t)counts[i]);  // qubit q at bit 31 - q
}

static void fetch_packed(ptsbe_batch* bt, uint32_t** records, uint64_t* n) {
  ptsbe_plan* pl = bt->plan;
  if (pl->words != 1 || pl->n > 32) throw Failure(PTSBE_EINVAL, "packed records need at most 32 measured qubits");
  if (bt->total_shots >= (1ull << 32)) throw Failure(PTSBE_EINVAL, "packed records need fewer than 2^32 shots per call");
  const uint64_t nr = bt->merged.n;
  uint32_t* r = (uint32_t*)g_host_pool.get(std::max<uint64_t>(nr, 1) * 8);
  if (!r) throw Failure(PTSBE_ECAPACITY, "host allocation of the histogram failed");
  if (nr) {
    WorkspaceScope tmp_scope(&bt->ws_tmp());
    const Workspace::Mark mark = bt->ws_tmp().mark();
    DevBuf packed(nr * 8, pl->stream);
    pack_records_kernel<<<cdiv(nr, 256), 256, 0, pl->stream>>>(bt->merged.keys.as<uint64_t>(), bt->merged.counts.as<uint64_t>(),
                                                               packed.as<uint2>(), nr);
    g_launches++;
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(r, packed.p, nr * 8, cudaMemcpyDeviceToHost, pl->stream));
    CK(cudaStreamSynchronize(pl->stream));
    bt->ws_tmp().rewind(mark);
  }
  *records = r;
  *n = nr;
}

int ptsbe_batch_fetch(ptsbe_batch* bt, uint64_t** keys, uint64_t** counts, uint64_t* n_records) {
  return guarded([&] {
    if (!bt) throw Failure(PTSBE_EINVAL, "null batch");
    std::lock_guard<std::mutex> lock(bt->plan->mu);
    CK(cudaSetDevice(bt->plan->device));
    fetch_merged(bt, keys, counts, n_records);
  });
}

void ptsbe_batch_destroy(ptsbe_batch* bt) {
  if (!bt) return;
  cudaSetDevice(bt->plan->device);
  cudaStreamSynchronize(bt->plan->stream);
  {
    std::lock_guard<std::mutex> lock(bt->plan->mu);
    bt->plan->give_workspace(std::move(bt->ws_tmp_own));
    bt->plan->give_workspace(std::move(bt->ws_out_own));
  }
  delete bt;
}

// Per-error-set records of a run -> host buffers of the C-ABI layout (keys [n][words] u64, counts u64,
// error-set position u32, optional probability tags).  Layout conversion runs on the device and the
// copies land in recycled page-locked buffers, like the merged histogram.
static void fetch_per_set(ptsbe_plan* pl, const RunOutput& out, bool with_probs, uint64_t** keys,
                          uint32_t** rec_eset, uint64_t** counts, double** probs, uint64_t* n_records) {
  cudaStream_t st = pl->stream;
  const uint32_t words = pl->words;
  const uint64_t nr = out.n, cap = std::max<uint64_t>(nr, 1);
  uint64_t* k = (uint64_t*)g_host_pool.get(cap * 8 * words);
  uint64_t* c = (uint64_t*)g_host_pool.get(cap * 8);
  uint32_t* es = (uint32_t*)g_host_pool.get(cap * 4);
  double* pr = probs ? (double*)g_host_pool.get(cap * 8) : nullptr;
  if (!k || !c || !es || (probs && !pr)) throw Failure(PTSBE_ECAPACITY, "host allocation of the records failed");
  if (nr) {
    DevBuf aos(nr * 8 * words, st), c64(nr * 8, st);
    untranspose_keys_kernel<<<cdiv(nr * words, 256), 256, 0, st>>>(out.keys.as<uint64_t>(), aos.as<uint64_t>(), nr, words);
    widen_counts_kernel<<<cdiv(nr, 256), 256, 0, st>>>(out.counts.as<uint32_t>(), c64.as<uint64_t>(), nr);
    g_launches += 2;
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(k, aos.p, nr * 8 * words, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(c, c64.p, nr * 8, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(es, out.eset.p, nr * 4, cudaMemcpyDeviceToHost, st));
    if (pr && with_probs) CK(cudaMemcpyAsync(pr, out.probs.p, nr * 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (pr && !with_probs)
      for (uint64_t i = 0; i < nr; ++i) pr[i] = -1.0;  // no tag in direct mode
  }
  *keys = k; *counts = c; *n_records = nr;
  if (rec_eset) *rec_eset = es; else ptsbe_free(es);
  if (probs) *probs = pr;
}

static int sample_host(ptsbe_plan* pl, const uint8_t* kraus_idx, const uint32_t* shots,
                       const uint32_t* eset_ids, uint64_t n_sets, uint64_t seed, int merged,
                       uint64_t** keys, uint32_t** rec_eset, uint64_t** counts, uint32_t** packed,
                       uint64_t* n_records, ptsbe_run_stats* stats) {
  ptsbe_batch* bt = nullptr;
  ptsbe_run_stats local;
  if (!stats) stats = &local;
  cudaEvent_t e0 = nullptr, e1 = nullptr, e2 = nullptr, e3 = nullptr;
  int rc = guarded([&] {
    if (!pl) throw Failure(PTSBE_EINVAL, "null plan");
    CK(cudaSetDevice(pl->device));
    CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
    CK(cudaEventCreate(&e2)); CK(cudaEventCreate(&e3));
    CK(cudaEventRecord(e0, pl->stream));
  });
  if (rc) return rc;
  rc = ptsbe_batch_upload(pl, kraus_idx, shots, eset_ids, n_sets, &bt);
  if (rc) return rc;
  rc = guarded([&] {
    std::lock_guard<std::mutex> lock(pl->mu);
    CK(cudaEventRecord(e1, pl->stream));
    run_batch(bt, seed, merged, stats);
    CK(cudaEventRecord(e2, pl->stream));
    const uint32_t words = pl->words;
    if (packed) {
      fetch_packed(bt, packed, n_records);
    } else if (merged) {
      fetch_merged(bt, keys, counts, n_records);
      if (rec_eset) *rec_eset = nullptr;
    } else {
      WorkspaceScope tmp_scope(&bt->ws_tmp());
      fetch_per_set(pl, bt->per_set, false, keys, rec_eset, counts, nullptr, n_records);
    }
    CK(cudaEventRecord(e3, pl->stream));
    CK(cudaStreamSynchronize(pl->stream));
    CK(cudaEventElapsedTime(&stats->h2d_ms, e0, e1));
    CK(cudaEventElapsedTime(&stats->d2h_ms, e2, e3));
    stats->h2d_bytes = n_sets * pl->g + n_sets * 4 * (eset_ids ? 2 : 1);
    stats->d2h_bytes = packed ? *n_records * 8ull : *n_records * (8ull * words + (merged ? 8 : 12));
  });
  ptsbe_batch_destroy(bt);
  if (e0) { cudaEventDestroy(e0); cudaEventDestroy(e1); cudaEventDestroy(e2); cudaEventDestroy(e3); }
  return rc;
}

int ptsbe_sample(ptsbe_plan* pl, const uint8_t* kraus_idx, const uint32_t* shots,
                 const uint32_t* eset_ids, uint64_t n_sets, uint64_t seed, int merged,
                 uint64_t** keys, uint32_t** rec_eset, uint64_t** counts, uint64_t* n_records,
                 ptsbe_run_stats* stats) {
  return sample_host(pl, kraus_idx, shots, eset_ids, n_sets, seed, merged, keys, rec_eset, counts, nullptr,
                     n_records, stats);
}

int ptsbe_sample_packed(ptsbe_plan* pl, const uint8_t* kraus_idx, const uint32_t* shots,
                        const uint32_t* eset_ids, uint64_t n_sets, uint64_t seed,
                        uint32_t** records, uint64_t* n_records, ptsbe_run_stats* stats) {
  const int pre = guarded([&] {
    if (!pl || !records || !n_records) throw Failure(PTSBE_EINVAL, "null argument");
    if (pl->words != 1 || pl->n > 32) throw Failure(PTSBE_EINVAL, "packed records need at most 32 measured qubits");
  });
  if (pre) return pre;
  return sample_host(pl, kraus_idx, shots, eset_ids, n_sets, seed, 1, nullptr, nullptr, nullptr, records,
                     n_records, stats);
}

int ptsbe_sample_nonproportional(ptsbe_plan* pl, const uint8_t* kraus_idx, const uint32_t* eset_ids,
                                 uint64_t n_sets, uint64_t seed, uint32_t nonfinal_shots,
                                 uint32_t final_mode, double threshold, uint32_t direct_count,
                                 uint64_t** keys, uint32_t** rec_eset, uint64_t** counts, double** probs,
                                 uint64_t* n_records, ptsbe_run_stats* stats) {
  ptsbe_run_stats local;
  if (!stats) stats = &local;
  return guarded([&] {
    if (!pl || !keys || !rec_eset || !counts || !probs || !n_records) throw Failure(PTSBE_EINVAL, "null argument");
    if (n_sets < 1 || n_sets >= (1ull << 31)) throw Failure(PTSBE_EINVAL, "need 1 .. 2^31 error sets");
    if (nonfinal_shots < 1 || final_mode > 1 || (final_mode == 1 && direct_count < 1))
      throw Failure(PTSBE_EINVAL, "non-proportional sampling needs nonfinal_shots >= 1 and a valid final mode");
    std::lock_guard<std::mutex> lock(pl->mu);
    CK(cudaSetDevice(pl->device));
    cudaStream_t st = pl->stream;
    const uint32_t f = pl->f;
    NonpropParams np{nonfinal_shots, final_mode, direct_count, threshold};
    // slots any stage can need PER ERROR SET: items_j <= nonfinal^(j-1), each with its multiplicity;
    // error sets are processed in chunks whose slot count stays below the chunk bound
    double per_set = 0, items = 1.0;
    for (uint32_t j = 1; j <= f; ++j) {
      const double mult = j < f ? nonfinal_shots : (final_mode == 0 ? std::ldexp(1.0, (int)pl->sizes[f - 1]) : direct_count);
      per_set = std::max(per_set, items * mult);
      items *= nonfinal_shots;
    }
    if (per_set >= 2147483648.0) throw Failure(PTSBE_ECAPACITY, "one error set needs more than 2^31 child slots");
    const double chunk_cap = std::min<double>(2147483647.0, (double)pl->chunk_shots);
    const uint64_t sets_per_chunk = std::max<uint64_t>(1, (uint64_t)(chunk_cap / per_set));
    memset(stats, 0, sizeof *stats);
    stats->first_flagged_id = -1;
    g_launches = 0;
    std::unique_ptr<Workspace> ws_tmp = pl->take_workspace(), ws_out = pl->take_workspace();
    ws_tmp->reset();
    ws_out->reset();
    {
      WorkspaceScope scope(ws_out.get());
      DevBuf kraus(std::max<size_t>(16, n_sets * pl->g), st), ids(n_sets * 4, st), flag(16, st);
      if (pl->g) CK(cudaMemcpyAsync(kraus.p, kraus_idx, n_sets * pl->g, cudaMemcpyHostToDevice, st));
      if (eset_ids) CK(cudaMemcpyAsync(ids.p, eset_ids, n_sets * 4, cudaMemcpyHostToDevice, st));
      else { iota_kernel<<<cdiv(n_sets, 256), 256, 0, st>>>(ids.as<uint32_t>(), (uint32_t)n_sets, 0); g_launches++; }
      CK(cudaMemsetAsync(flag.p, 0xff, 8, st));
      CK(cudaMemsetAsync(flag.as<unsigned char>() + 8, 0, 8, st));
      check_kraus(pl, kraus.as<uint8_t>(), n_sets);
      RunOutput out;
      cudaEvent_t e0, e1;
      CK(cudaEventCreate(&e0));
      CK(cudaEventCreate(&e1));
      CK(cudaEventRecord(e0, st));
      {
        std::vector<RunOutput> outs;
        std::vector<uint64_t> first_set;
        for (uint64_t e = 0; e < n_sets; e += sets_per_chunk) {
          const uint64_t cnt = std::min<uint64_t>(sets_per_chunk, n_sets - e);
          outs.emplace_back();
          first_set.push_back(e);
          WorkspaceScope chunk_scope(ws_tmp.get());
          const Workspace::Mark mark = ws_tmp->mark();
          run_chunk(pl, kraus.as<uint8_t>() + e * pl->g, nullptr, ids.as<uint32_t>() + e, (uint32_t)cnt,
                    (uint64_t)(per_set * (double)cnt), seed, outs.back(), stats, flag.as<unsigned long long>(),
                    flag.as<uint32_t>() + 2, *ws_out, &np);
          ws_tmp->rewind(mark);  // run_chunk returns with the stream drained
        }
        stats->n_chunks = (uint32_t)outs.size();
        if (outs.size() == 1) out = std::move(outs[0]);
        else concat_outputs(outs, first_set, pl->words, out, st);
      }
      CK(cudaEventRecord(e1, st));
      struct { unsigned long long first; uint32_t count; uint32_t pad; } fl;
      CK(cudaMemcpyAsync(&fl, flag.p, 16, cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      CK(cudaEventElapsedTime(&stats->loop_ms, e0, e1));
      cudaEventDestroy(e0);
      cudaEventDestroy(e1);
      stats->flagged_sets = fl.count;
      if (fl.count) {
        stats->first_flag_kind = (uint32_t)(fl.first & 0xff);
        stats->first_flag_stage = (uint32_t)((fl.first >> 8) & 0xff);
        stats->first_flagged_id = (int64_t)(fl.first >> 16);
      }
      {
        WorkspaceScope tmp_scope(ws_tmp.get());
        fetch_per_set(pl, out, final_mode == 0, keys, rec_eset, counts, probs, n_records);
      }
      const uint64_t nr = out.n;
      stats->n_records = nr;
      stats->gpu_launches = g_launches;
    }
    pl->give_workspace(std::move(ws_tmp));
    pl->give_workspace(std::move(ws_out));
  });
}

int ptsbe_project_probe(int device, uint32_t D, uint32_t N, uint64_t n_items, uint32_t n_sets,
                        const uint32_t* eset, const float* v, const float* m, int use_tc, float* out,
                        int reps, float* kernel_ms, float* prep_ms) {
  return guarded([&] {
    if (!eset || !v || !m || !out || !n_items || !n_sets) throw Failure(PTSBE_EINVAL, "null or empty argument");
    if (ptsbe_device_count() <= device) throw Failure(PTSBE_EDEVICE, "no CUDA device: libptsbe_b200 has no CPU fallback");
    CK(cudaSetDevice(device));
    ptsbe_plan pl;
    pl.device = device;
    pl.dtype = PTSBE_C64;
    pl.elem = 8;
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, device));
    pl.sm_count = prop.multiProcessorCount;
    CK(cudaStreamCreateWithFlags(&pl.stream, cudaStreamNonBlocking));
    cudaStream_t st = pl.stream;
    const uint32_t n = (uint32_t)n_items;
    cudaEvent_t e0, e1, e2;
    CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1)); CK(cudaEventCreate(&e2));
    {
      DevBuf es((size_t)n * 4, st), rec((size_t)n_sets * D * N * 8, st), po((size_t)n * N * 4, st);
      CK(cudaMemcpyAsync(es.p, eset, (size_t)n * 4, cudaMemcpyHostToDevice, st));
      CK(cudaMemcpyAsync(rec.p, m, (size_t)n_sets * D * N * 8, cudaMemcpyHostToDevice, st));
      CK(cudaMemsetAsync(po.p, 0xff, (size_t)n * N * 4, st));
      Program pr;
      memset(&pr.d, 0, sizeof pr.d);
      pr.d.proj_d = D;
      pr.d.out_elems = N;
      pr.d.result_ref = 0;
      float pm = 0, km = 0;
      if (use_tc) {
        const TcShape t = tc_shape(D, N);
        if (!t.ok) throw Failure(PTSBE_EINVAL, "tensor-core projection needs N = 32 .. 256 (power of two)");
        DevBuf vr((size_t)n * t.K * 4, st), bh((size_t)n_sets * N * t.K * 4, st), bl((size_t)n_sets * N * t.K * 4, st);
        CK(cudaMemsetAsync(vr.p, 0, (size_t)n * t.K * 4, st));
        CK(cudaMemcpy2DAsync(vr.p, (size_t)t.K * 4, v, (size_t)D * 8, (size_t)D * 8, n, cudaMemcpyHostToDevice, st));
        CK(cudaEventRecord(e0, st));
        launch_tc_prep(&pl, rec.p, D * N, 0, n_sets, D, N, t, bh.as<float>(), bl.as<float>());
        CK(cudaEventRecord(e1, st));
        for (int r = 0; r < std::max(reps, 1); ++r)
          launch_project_tc(&pl, t, vr.p, bh.as<float>(), bl.as<float>(), n_sets, es.as<uint32_t>(), 0, n, N, po.p);
        CK(cudaEventRecord(e2, st));
        CK(cudaStreamSynchronize(st));
        CK(cudaEventElapsedTime(&pm, e0, e1));
        CK(cudaEventElapsedTime(&km, e1, e2));
      } else {
        const uint32_t pitch = vec_pitch(n);
        std::vector<float> vt((size_t)D * pitch * 2, 0.f);
        for (uint32_t i = 0; i < n; ++i)
          for (uint32_t d = 0; d < D; ++d) {
            vt[((size_t)d * pitch + i) * 2] = v[((size_t)i * D + d) * 2];
            vt[((size_t)d * pitch + i) * 2 + 1] = v[((size_t)i * D + d) * 2 + 1];
          }
        DevBuf vd(vt.size() * 4, st);
        CK(cudaMemcpyAsync(vd.p, vt.data(), vt.size() * 4, cudaMemcpyHostToDevice, st));
        CK(cudaEventRecord(e1, st));
        for (int r = 0; r < std::max(reps, 1); ++r)
          launch_project(&pl, pr, vd.p, pitch, rec.p, D * N, es.as<uint32_t>(), 0, n, po.p);
        CK(cudaEventRecord(e2, st));
        CK(cudaStreamSynchronize(st));
        CK(cudaEventElapsedTime(&km, e1, e2));
      }
      CK(cudaMemcpyAsync(out, po.p, (size_t)n * N * 4, cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      if (kernel_ms) *kernel_ms = km / std::max(reps, 1);
      if (prep_ms) *prep_ms = pm;
    }
    cudaEventDestroy(e0); cudaEventDestroy(e1); cudaEventDestroy(e2);
    CK(cudaStreamSynchronize(st));
    cudaStreamDestroy(st);
    pl.stream = nullptr;
  });
}

int ptsbe_batch_histogram_dev(ptsbe_batch* bt, const uint64_t** keys_dev,
                              const uint64_t** counts_dev, uint64_t* n_records) {
  return guarded([&] {
    if (!bt || !keys_dev || !counts_dev || !n_records) throw Failure(PTSBE_EINVAL, "null argument");
    std::lock_guard<std::mutex> lock(bt->plan->mu);
    *keys_dev = bt->merged.keys.as<uint64_t>();
    *counts_dev = bt->merged.counts.as<uint64_t>();
    *n_records = bt->merged.n;
  });
}

int ptsbe_histogram_merge_dev(const uint64_t* keys_dev, const uint64_t* counts_dev, uint64_t n,
                              uint32_t words, int device, uint64_t** out_keys_dev,
                              uint64_t** out_counts_dev, uint64_t* n_out) {
  return guarded([&] {
    if (ptsbe_device_count() <= device)
      throw Failure(PTSBE_EDEVICE, "no CUDA device: libptsbe_b200 has no CPU fallback");
    if (words < 1) throw Failure(PTSBE_EINVAL, "words must be >= 1");
    CK(cudaSetDevice(device));
    g_launches = 0;
    cudaStream_t st;
    CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    {
      const uint64_t m = std::max<uint64_t>(n, 1);
      DevBuf soa;
      const uint64_t* kin = keys_dev;
      if (words > 1 && n) {  // row-major [n][words] -> SoA [words][n]
        soa.alloc(m * 8 * words, st);
        transpose_keys_kernel<<<cdiv(n * words, 256), 256, 0, st>>>(keys_dev, soa.as<uint64_t>(), n, words);
        g_launches++;
        kin = soa.as<uint64_t>();
      }
      Histogram h;
      reduce_by_key(kin, n, words, nullptr, counts_dev, n, 64 * words, h, st);
      CK(cudaStreamSynchronize(st));
      *n_out = h.n;
      // hand the buffers over: detach them from their RAII owners
      *out_keys_dev = h.keys.as<uint64_t>();
      *out_counts_dev = h.counts.as<uint64_t>();
      h.keys.p = nullptr;
      h.counts.p = nullptr;
    }
    cudaStreamSynchronize(st);
    cudaStreamDestroy(st);
  });
}

int ptsbe_measure_fma_peak(int device, double* fp32_tflops, double* fp64_tflops) {
  return guarded([&] {
    if (ptsbe_device_count() <= device)
      throw Failure(PTSBE_EDEVICE, "no CUDA device: libptsbe_b200 has no CPU fallback");
    CK(cudaSetDevice(device));
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, device));
    if (fp32_tflops) *fp32_tflops = fma_peak<float>(prop.multiProcessorCount, 1 << 16);
    if (fp64_tflops) *fp64_tflops = fma_peak<double>(prop.multiProcessorCount, 1 << 12);
  });
}

void ptsbe_free_dev(void* p) {
  if (p) cudaFree(p);
}

int ptsbe_histogram_merge(const uint64_t* keys, const uint64_t* counts, uint64_t n,
                          uint32_t words, uint64_t** out_keys, uint64_t** out_counts,
                          uint64_t* n_out, int device) {
  return guarded([&] {
    if (ptsbe_device_count() <= device)
      throw Failure(PTSBE_EDEVICE, "no CUDA device: libptsbe_b200 has no CPU fallback");
    if (words < 1) throw Failure(PTSBE_EINVAL, "words must be >= 1");
    CK(cudaSetDevice(device));
    g_launches = 0;
    cudaStream_t st;
    CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    {
      // item-major host keys -> SoA device keys
      std::vector<uint64_t> soa(std::max<uint64_t>(n, 1) * words);
      for (uint64_t i = 0; i < n; ++i)
        for (uint32_t w = 0; w < words; ++w) soa[(uint64_t)w * n + i] = keys[i * words + w];
      DevBuf dk(std::max<uint64_t>(n, 1) * 8 * words, st), dc(std::max<uint64_t>(n, 1) * 8, st);
      if (n) {
        CK(cudaMemcpyAsync(dk.p, soa.data(), n * 8 * words, cudaMemcpyHostToDevice, st));
        CK(cudaMemcpyAsync(dc.p, counts, n * 8, cudaMemcpyHostToDevice, st));
      }
      Histogram h;
      reduce_by_key(dk.as<uint64_t>(), n, words, nullptr, dc.as<uint64_t>(), n, 64 * words, h, st);
      uint64_t* k = (uint64_t*)malloc(std::max<uint64_t>(h.n, 1) * 8 * words);
      uint64_t* c = (uint64_t*)malloc(std::max<uint64_t>(h.n, 1) * 8);
      if (h.n) {
        CK(cudaMemcpyAsync(k, h.keys.p, h.n * 8 * words, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(c, h.counts.p, h.n * 8, cudaMemcpyDeviceToHost, st));
      }
      CK(cudaStreamSynchronize(st));
      *out_keys = k; *out_counts = c; *n_out = h.n;
    }
    cudaStreamSynchronize(st);
    cudaStreamDestroy(st);
  });
}

}  // extern "C"
