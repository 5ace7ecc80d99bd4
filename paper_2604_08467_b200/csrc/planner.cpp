// Host-side contraction-path search (north-star subsystem 1): randomized greedy
// descents over the error-free template network, scored with a batch-aware
// cost.  A path is found once per stage and stored; every error set and every
// prefix replays it (engine.py:864-879, planner.py:416-442).
//
// Differences from the reference planner (planner.py:121-251) are deliberate:
//   * native code, so hundreds of descents on 1000-operand networks cost
//     milliseconds instead of minutes;
//   * every operand carries a dependency class (0 = depends on the error set
//     only, k = also on prefix bits measured up to stage k).  A step's cost is
//     flops x (number of distinct instances of its result in the batch), which
//     is what the executor really pays once error-independent subtrees are
//     hoisted and computed once per error set / per earlier-stage prefix;
//   * a soft cap keeps intermediates inside the on-chip arena.
// The flop model itself is the reference's: product of the dims of the union of
// both operands' labels (planner.py:61-103), reported next to the weighted cost.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <queue>
#include <thread>
#include <vector>

#include "../../include/ptsbe_b200.h"

namespace {

struct Rng {  // splitmix64
  uint64_t s;
  explicit Rng(uint64_t seed) : s(seed) {}
  uint64_t next() {
    uint64_t z = (s += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  }
  double uniform() { return ((next() >> 11) + 0.5) * (1.0 / 9007199254740992.0); }
};

// Cost of issuing one step for one work item, in multiply-add equivalents.  Measured on B200
// (cfg5 stage-3/4 per-item programs, CTA per item): time per item ~ 1.1 ns x steps + 0.0015 ns x MACs,
// i.e. a barrier-separated step costs as much as ~700 MACs; lane-per-item programs pay ~30.
// 400 makes the search prefer few-step (cut / projection) forms for the per-item pass.
static double kStepOverheadMacs = 400.0;  // PTSBE_STEP_OVERHEAD overrides (experiments)

struct Cand {
  double key, tie;
  uint32_t x, y, vx, vy;
  bool operator<(const Cand& o) const {  // min-heap through std::priority_queue
    if (key != o.key) return key > o.key;
    return tie > o.tie;
  }
};

struct Problem {
  uint32_t n;
  std::vector<std::vector<int32_t>> labels;  // dense label ids, sorted
  std::vector<double> log2dim;               // per label
  std::vector<uint32_t> cls;
  std::vector<uint8_t> unit;  // 1: rank-1 basis vector (prefix projector): merging it is a gather, not a contraction
  std::vector<double> logw;  // log class weight
  uint32_t n_labels;
  std::vector<double> cap_log2;  // per class
};

struct Descent {
  std::vector<uint32_t> merges;
  double weighted = 0, flops = 0;
};

static Descent descend(const Problem& P, Rng& rng, double temperature, double gamma) {
  const uint32_t n = P.n;
  std::vector<std::vector<int32_t>> lab = P.labels;
  std::vector<uint32_t> cls = P.cls, version(n, 0);
  std::vector<uint8_t> unit = P.unit;
  std::vector<char> alive(n, 1);
  std::vector<double> lsize(n, 0.0);
  std::vector<int32_t> own(2 * (size_t)P.n_labels, -1);
  for (uint32_t t = 0; t < n; ++t)
    for (int32_t l : lab[t]) {
      lsize[t] += P.log2dim[l];
      if (own[2 * l] < 0) own[2 * l] = (int32_t)t; else own[2 * l + 1] = (int32_t)t;
    }
  auto other = [&](int32_t l, uint32_t t) -> int32_t {
    return own[2 * l] == (int32_t)t ? own[2 * l + 1] : own[2 * l];
  };
  std::priority_queue<Cand> heap;
  auto measure = [&](uint32_t x, uint32_t y, double& lunion, double& lshared, double& lout) {
    lshared = 0;
    const auto &a = lab[x], &b = lab[y];
    size_t i = 0, j = 0;
    while (i < a.size() && j < b.size()) {
      if (a[i] < b[j]) ++i;
      else if (a[i] > b[j]) ++j;
      else { lshared += P.log2dim[a[i]]; ++i; ++j; }
    }
    lunion = lsize[x] + lsize[y] - lshared;
    lout = lunion - lshared;
  };
  auto push = [&](uint32_t x, uint32_t y) {
    if (x > y) std::swap(x, y);
    double lu, ls, lo;
    measure(x, y, lu, ls, lo);
    // reference score: flops(step) - prod(shared dims), compared in log space; absorbing a basis
    // vector only selects a slice of the other operand (a view of the other operand: the executor only adds bit * stride to its base)
    const bool slice = unit[x] || unit[y];
    const double score = slice ? 0.05 * std::exp2(lo)
                               : std::max(0.0, std::exp2(std::min(lu, 1000.0)) - std::exp2(ls));
    double key = std::log1p(score) + gamma * P.logw[std::max(cls[x], cls[y])];
    const double cap = P.cap_log2[std::max(cls[x], cls[y])];
    if (lo > cap) key += 50.0 * (lo - cap) + 100.0;
    if (temperature > 0.0) {
      const double u = rng.uniform();
      key += temperature * -std::log(-std::log(u));
    }
    heap.push(Cand{key, rng.uniform(), x, y, version[x], version[y]});
  };
  for (uint32_t t = 0; t < n; ++t)
    for (int32_t l : lab[t]) {
      const int32_t o = other(l, t);
      if (o > (int32_t)t) push(t, (uint32_t)o);
    }
  Descent D;
  D.merges.reserve(2 * (size_t)n);
  uint32_t remaining = n;
  std::vector<int32_t> merged;
  while (remaining > 1) {
    uint32_t x = 0, y = 0;
    bool found = false;
    while (!heap.empty()) {
      const Cand c = heap.top();
      heap.pop();
      if (alive[c.x] && alive[c.y] && version[c.x] == c.vx && version[c.y] == c.vy) {
        x = c.x; y = c.y; found = true;
        break;
      }
    }
    if (!found) {  // disconnected pieces: outer product of the two smallest
      int64_t s1 = -1, s2 = -1;
      for (uint32_t t = 0; t < n; ++t) {
        if (!alive[t]) continue;
        if (s1 < 0 || lsize[t] < lsize[s1]) { s2 = s1; s1 = t; }
        else if (s2 < 0 || lsize[t] < lsize[s2]) s2 = t;
      }
      x = (uint32_t)std::min(s1, s2);
      y = (uint32_t)std::max(s1, s2);
    }
    double lu, ls, lo;
    measure(x, y, lu, ls, lo);
    const uint32_t c = std::max(cls[x], cls[y]);
    const bool is_slice = unit[x] || unit[y];
    const double fl = is_slice ? 0.05 * std::exp2(lo) : std::exp2(std::min(lu, 1000.0));
    D.flops += fl;
    // every interpreted step costs the executor a fixed dispatch (table fetch, sync) on top of
    // its multiply-adds
    D.weighted += (fl + (is_slice ? 0.0 : kStepOverheadMacs)) * std::exp(P.logw[c]);
    merged.clear();
    std::set_symmetric_difference(lab[x].begin(), lab[x].end(), lab[y].begin(), lab[y].end(),
                                  std::back_inserter(merged));
    for (int32_t l : lab[y]) {  // y's labels now live on x; labels shared with x vanish
      if (other(l, y) == (int32_t)x) {
        own[2 * l] = own[2 * l + 1] = -1;
      } else if (own[2 * l] == (int32_t)y) {
        own[2 * l] = (int32_t)x;
      } else {
        own[2 * l + 1] = (int32_t)x;
      }
    }
    lab[x] = merged;
    lab[y].clear();
    lab[y].shrink_to_fit();
    alive[y] = 0;
    cls[x] = c;
    unit[x] = 0;
    lsize[x] = lo;
    version[x]++;
    D.merges.push_back(x);
    D.merges.push_back(y);
    --remaining;
    // re-score the neighbourhood of the merged tensor (each neighbour once)
    std::vector<uint32_t> nb;
    for (int32_t l : lab[x]) {
      const int32_t o = other(l, x);
      if (o >= 0 && o != (int32_t)x && alive[o]) nb.push_back((uint32_t)o);
    }
    std::sort(nb.begin(), nb.end());
    nb.erase(std::unique(nb.begin(), nb.end()), nb.end());
    for (uint32_t z : nb) push(x, z);
  }
  return D;
}

}  // namespace

extern "C" int ptsbe_plan_greedy(uint32_t n_ops, const uint32_t* op_ptr, const int64_t* labels,
                                 const uint32_t* dims, const uint32_t* op_class,
                                 const double* class_weight, const double* class_cap_log2,
                                 const uint8_t* op_unit, uint32_t n_classes, uint32_t hypersamples,
                                 uint64_t seed, double size_cap_log2,
                                 uint32_t* merges_out, double* cost_out, double* flops_out) {
  if (n_ops < 1 || hypersamples < 1 || !op_ptr || !merges_out) return PTSBE_EINVAL;
  if (const char* ov = getenv("PTSBE_STEP_OVERHEAD")) kStepOverheadMacs = atof(ov);
  Problem P;
  P.n = n_ops;
  P.labels.resize(n_ops);
  P.cls.assign(n_ops, 0);
  P.unit.assign(n_ops, 0);
  // densify labels
  std::vector<int64_t> uniq(labels, labels + op_ptr[n_ops]);
  std::sort(uniq.begin(), uniq.end());
  uniq.erase(std::unique(uniq.begin(), uniq.end()), uniq.end());
  P.n_labels = (uint32_t)uniq.size();
  P.log2dim.assign(P.n_labels, 0.0);
  std::vector<uint8_t> uses(P.n_labels, 0);
  for (uint32_t t = 0; t < n_ops; ++t) {
    for (uint32_t k = op_ptr[t]; k < op_ptr[t + 1]; ++k) {
      const int32_t id = (int32_t)(std::lower_bound(uniq.begin(), uniq.end(), labels[k]) - uniq.begin());
      P.labels[t].push_back(id);
      P.log2dim[id] = std::log2((double)dims[k]);
      if (++uses[id] > 2) return PTSBE_ESTRUCT;
    }
    std::sort(P.labels[t].begin(), P.labels[t].end());
    if (op_class) P.cls[t] = op_class[t];
    if (op_unit && op_unit[t] && op_ptr[t + 1] - op_ptr[t] == 1) P.unit[t] = 1;
  }
  uint32_t nc = std::max<uint32_t>(1, n_classes);
  P.logw.assign(nc, 0.0);
  P.cap_log2.assign(nc, size_cap_log2 > 0 ? size_cap_log2 : 1e9);
  for (uint32_t c = 0; c < nc; ++c) {
    if (class_weight) P.logw[c] = std::log(std::max(class_weight[c], 1e-300));
    if (class_cap_log2 && class_cap_log2[c] > 0) P.cap_log2[c] = class_cap_log2[c];
  }
  for (uint32_t t = 0; t < n_ops; ++t)
    if (P.cls[t] >= nc) return PTSBE_EINVAL;
  // The search score is flops x weight^gamma.  gamma = 1 hoists as much as possible out of
  // the per-item classes but lets nearly-free low-class merges run ahead and build blobs the
  // per-item steps then have to chew through; gamma = 0 is the reference's plain greedy, which
  // absorbs the rank-1 prefix projectors first and keeps per-item tensors tiny.  Every descent
  // is judged by the true batch-weighted cost (gamma = 1), so the mix costs nothing.
  // Descents are independent: they run on host threads, descent h always uses the stream
  // seeded by (seed, h), so the result does not depend on the thread count.
  static const double gammas[3] = {1.0, 0.5, 0.0};
  unsigned n_threads = std::max(1u, std::min<unsigned>(std::thread::hardware_concurrency(), 32u));
  if (const char* tv = getenv("PTSBE_PLANNER_THREADS")) n_threads = std::max(1, atoi(tv));
  n_threads = std::min<unsigned>(n_threads, hypersamples);
  std::vector<Descent> bests(n_threads);
  std::vector<uint32_t> best_h(n_threads, UINT32_MAX);
  auto worker = [&](unsigned tix) {
    for (uint32_t h = tix; h < hypersamples; h += n_threads) {
      Rng rng((seed + 0x632BE59BD9B4E019ull * (h + 1)) * 0x9E3779B97F4A7C15ull + 0x1234567ull);
      const double gamma = gammas[h % 3];
      const double temperature = h < 3 ? 0.0 : ((h / 3) % 2 ? 1.0 : 0.5);
      Descent d = descend(P, rng, temperature, gamma);
      if (best_h[tix] == UINT32_MAX || d.weighted < bests[tix].weighted) {
        bests[tix] = std::move(d);
        best_h[tix] = h;
      }
    }
  };
  if (n_threads == 1) {
    worker(0);
  } else {
    std::vector<std::thread> pool;
    for (unsigned t = 0; t < n_threads; ++t) pool.emplace_back(worker, t);
    for (auto& th : pool) th.join();
  }
  Descent best;
  uint32_t bh = UINT32_MAX;
  for (unsigned t = 0; t < n_threads; ++t) {
    if (best_h[t] == UINT32_MAX) continue;
    // ties go to the lowest descent index: same answer for any thread count
    if (bh == UINT32_MAX || bests[t].weighted < best.weighted ||
        (bests[t].weighted == best.weighted && best_h[t] < bh)) {
      best = std::move(bests[t]);
      bh = best_h[t];
    }
  }
  std::copy(best.merges.begin(), best.merges.end(), merges_out);
  if (cost_out) *cost_out = best.weighted;
  if (flops_out) *flops_out = best.flops;
  return PTSBE_OK;
}
