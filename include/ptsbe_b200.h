/*
 * ptsbe_b200.h -- C ABI of libptsbe_b200.so, the B200 (sm_100a) drop-in for the
 * PTSBE proportional hot path of the reference package `ptsbe`.
 *
 * The reference has no FFI seam (pure Python); the entry points below are what
 * a ctypes binding inside the reference would call in place of the Python
 * functions cited next to each of them (paths relative to
 * /root/reference/pkg/src/ptsbe/).  INTEGRATION.md shows that binding.
 *
 * Conventions
 *   - every function returns a ptsbe_status (0 = ok); the message of the last
 *     failure on the calling thread is ptsbe_last_error();
 *   - all pointers are HOST pointers unless the name ends in _dev;
 *   - inputs are caller-owned and only read; variable-length outputs are
 *     allocated by the library and released with ptsbe_free();
 *   - a plan is immutable after creation and may be shared by threads; calls
 *     that run kernels serialise on the plan's own CUDA stream;
 *   - there is no CPU fallback: without a CUDA device every compute entry point
 *     fails with PTSBE_EDEVICE.
 */
#ifndef PTSBE_B200_H
#define PTSBE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  PTSBE_OK = 0,
  PTSBE_EINVAL = 1,      /* ValueError                                    */
  PTSBE_ESTRUCT = 2,     /* errors.py: NetworkStructureError              */
  PTSBE_ERESOURCE = 3,   /* errors.py: ResourceLimitError (ceiling/deadline) */
  PTSBE_ENUMERIC = 4,    /* errors.py: NumericalError (engine.py:447-448) */
  PTSBE_EIMPOSSIBLE = 5, /* errors.py: ImpossiblePrefixError (engine.py:475-476) */
  PTSBE_EDEVICE = 6,     /* CUDA missing / runtime failure                */
  PTSBE_ECAPACITY = 7    /* errors.py: CapacityError                      */
} ptsbe_status;

enum { PTSBE_C64 = 0, PTSBE_C128 = 1 };

/* ---- compiled stage program (produced by paper_2604_08467_b200/compiler.py) ----
 *
 * A program is the stored contraction path of one (stage, pass) with every
 * index map precomputed (replaces tensor.py:219-268 execute_path +
 * tensor.py:190-216 contract_pair + engine.py:361-407 marginal_network).
 *
 * leaves : n_leaves x 4 words  {pool_off, size, sel_kind, sel_arg}
 *          sel_kind 0: constant            data = pool[pool_off .. +size)
 *          sel_kind 1: Kraus variant       data = pool[pool_off + kraus_idx[e][sel_arg]*size ..)
 *                      (UPV merge, engine.py:284-313, done once on the host per variant)
 *          sel_kind 2: prefix bit          data = pool[pool_off + bit(sel_arg)*size ..)
 *                      (basis vectors of engine.py:395-399)
 * steps  : n_steps x 20 words {a_kind, a_ref, b_kind, b_ref, o_kind, o_ref,
 *                              out_n, k_n, lo_n, hi_n, tab_off, conj,
 *                              a_memo, b_memo, a_prod | b_prod << 16, own_memo,
 *                              gemm_off, gemm_m, gemm_n, 0}
 *          gemm_m > 0: the step also carries its separable form at tables[gemm_off]:
 *          aOff[gemm_m] bOff[gemm_n] oA[gemm_m] oB[gemm_n] with
 *          out[oA[a] + oB[b]] = sum_k A[aOff[a] + kA[k]] * B[bOff[b] + kB[k]]
 *          conj bit 0 / 1: operand A / B is read complex-conjugated (its node is the
 *          conjugate twin -- bra copy -- of the node that was actually computed);
 *          bit 2: B is a prefix-bit basis vector e_x contracted over its only label, so the
 *          step is the slice out[c] = A[.. + kA[x]] (no multiply-adds);
 *          bit 3: slice views -- the step's table block ends with [nA, (qubit, stride) x nA,
 *          nB, (qubit, stride) x nB]: operand bases advance by stride when the measured bit
 *          of that qubit is 1 (the operand is a slice of a stored tensor, never materialised)
 *          bit 4: the step always runs (it writes a record or the result);
 *          bit 5 / 6: the offsets of operand A / B do not depend on the output index (loA, hiA all 0);
 *          a_prod / b_prod: index of the step of this program that produces operand A / B
 *          (0xFFFF: a leaf or an earlier pass), a_memo / b_memo / own_memo: offsets of the
 *          operands' and the step's own variant-0 value in the program's memo (memo_elems > 0)
 *          operand kind 0: arena offset (elements), 1: leaf index,
 *                       2 + p: record of pass p of the same stage, a_ref = offset in record
 *          output  kind 0: arena offset, 1: offset in this pass's output record
 * tables : u32 offsets; for a step: loA[lo_n] loB[lo_n] hiA[hi_n] hiB[hi_n] kA[k_n] kB[k_n]
 *          out[c] = sum_k A[loA[c%lo_n]+hiA[c/lo_n]+kA[k]] * B[loB[..]+hiB[..]+kB[k]]
 */
typedef struct {
  uint32_t n_leaves;
  uint32_t n_steps;
  uint32_t n_table_words;
  uint32_t arena_fast_elems;  /* per-item shared-memory arena, in complex elements   */
  uint32_t arena_spill_elems; /* per-item global spill arena (offsets >= arena_fast) */
  uint32_t out_elems;         /* complex elements per output record                  */
  uint32_t threads_per_item;  /* 8, 16, 32 (lanes per item) or a CTA size up to 256          */
  uint32_t level;             /* 1-based item level this pass iterates over          */
  uint32_t result_kind;       /* where the finished record lives: 0 arena, 1 leaf, 2+p record of
                                 pass p, 3 projection form (marginal pass only)               */
  uint32_t result_ref;
  uint32_t proj_d;            /* projection form: the steps leave a vector v[proj_d] in the pass's
                                 output record; the stage result is Re(sum_d v[d] * M[d][c]) with
                                 M[proj_d][out_elems] at offset result_ref of pass 0's record (one
                                 per error set) -- run as a dense product over all work items of
                                 an error set (csrc/project.cuh)                                 */
  uint32_t memo_elems;        /* > 0: class-0 program with a variant-0 memo.  The value of every
                                 step under Kraus index 0 at every site is computed once per plan;
                                 a work item re-executes only the steps that depend on a site with
                                 a non-zero index (the UPV merge of engine.py:284-313 leaves all
                                 other tensors of the template untouched) plus the always-run ones */
  const uint32_t* leaves;
  const uint32_t* steps;
  const uint32_t* tables;
  const uint32_t* memo_ptr;   /* [n_memo_sites + 2] CSR row starts into memo_idx; row s = steps that
                                 depend on gate site s, row n_memo_sites = always-run steps        */
  const uint32_t* memo_idx;   /* [n_memo_idx] step indices                                          */
  uint32_t n_memo_idx;
  uint32_t n_memo_sites;
} ptsbe_program_desc;

typedef struct {
  uint32_t dtype;     /* PTSBE_C64 | PTSBE_C128 */
  uint32_t n_qubits;
  uint32_t n_sites;   /* g: gate sites = columns of kraus_idx */
  uint32_t n_stages;  /* f */
  const uint32_t* stage_sizes; /* b_1..b_f (engine.py:76-142 BatchPlan.sizes) */
  const void* pool;   /* operand values: interleaved re,im of dtype precision */
  uint64_t pool_elems;
  /* stage j (1-based) owns passes 0..j-1; pass p iterates over the unique
   * prefixes entering stage p+1 (p = j-1 is the marginal pass itself) */
  const ptsbe_program_desc* programs; /* stage-major, f*(f+1)/2 entries */
  uint64_t max_intermediate;          /* ceiling, informational (checked at compile time) */
  /* [n_sites] number of operator variants (Kraus indices 0..v-1) of every gate site in this plan's
   * tables, or NULL.  When given, every Kraus-index matrix handed to the plan is checked on the
   * device and an out-of-range index (e.g. error sets encoded against other tables) is refused
   * with PTSBE_EINVAL instead of gathering outside the operand pool. */
  const uint8_t* site_variants;
} ptsbe_plan_desc;

typedef struct ptsbe_plan ptsbe_plan;

/* per-run statistics (mirrors engine.py:155-181 EngineStats + RunResult counters) */
#define PTSBE_MAX_STAGES 64
typedef struct {
  uint64_t stage_events[PTSBE_MAX_STAGES]; /* U_j = unique prefixes contracted in stage j */
  float stage_ms[PTSBE_MAX_STAGES];        /* device time per stage (CUDA events)          */
  uint64_t gpu_launches;                   /* kernels launched by this call               */
  uint64_t total_shots;
  uint64_t n_records;
  float loop_ms;      /* contraction + sampling + local histogram, device timed */
  float h2d_ms;
  float d2h_ms;
  uint64_t h2d_bytes;
  uint64_t d2h_bytes;
  uint32_t n_chunks;
  uint32_t flagged_sets; /* error sets with vanishing mass / negative diagonal */
  int64_t first_flagged_id;
  uint32_t first_flag_kind; /* PTSBE_ENUMERIC or PTSBE_EIMPOSSIBLE */
  uint32_t first_flag_stage;
  /* per-kernel device time inside each stage (CUDA events on the plan's stream) */
  float hoist_ms[PTSBE_MAX_STAGES];   /* exec_kernel, hoist passes 0..j-2          */
  float marg_ms[PTSBE_MAX_STAGES];    /* exec_kernel, marginal pass (per-item steps) */
  float project_ms[PTSBE_MAX_STAGES]; /* project_kernel, dense root step           */
  float sampler_ms[PTSBE_MAX_STAGES]; /* sample_kernel                             */
  float compact_ms[PTSBE_MAX_STAGES]; /* scans + expand + rank (next work list)    */
  float histogram_ms;                 /* final sort + reduce-by-key                */
  uint32_t marg_launches[PTSBE_MAX_STAGES];
  float descent_ms[PTSBE_MAX_STAGES]; /* tree_build_kernel + descent_kernel (per-qubit descent sampler) */
  uint64_t descent_items[PTSBE_MAX_STAGES]; /* work items sampled by descent instead of project + sample */
} ptsbe_run_stats;

const char* ptsbe_last_error(void);
int ptsbe_device_count(void);
const char* ptsbe_version(void);

/* replaces: building + caching the stage networks and paths once per run
 * (engine.py:864-879 warm loop; planner.py:343-442 PathCache) */
int ptsbe_plan_create(const ptsbe_plan_desc* desc, int device, ptsbe_plan** out);
void ptsbe_plan_destroy(ptsbe_plan* plan);

/* Per-stage choice between the two samplers of rng.multinomial's categorical draw
 * (engine.py:519): kinds[j] = 0 flat inverse-CDF sampler over the 2^b population vector,
 * 1 per-qubit descent (few shots per work item), -1 decide per chunk from its work list (default).
 * A fixed choice makes complex64 results independent of how error sets are grouped into calls,
 * chunks and ranks (determinism under sharding, reference tests/test_engine.py:455-463): the host
 * derives it once per plan from a pilot run of the error-free circuit. */
int ptsbe_plan_set_stage_samplers(ptsbe_plan* plan, const int32_t* kinds, uint32_t n_stages);

/* replaces: conditional_marginal / _contract_marginal for a batch of W work
 * items of one stage (engine.py:417-477).
 *   kraus_idx [W][g] variant index per site, prefixes [W][words] packed bits
 *   (qubit q -> word q/64, bit 63-(q%64)), words = ceil(n_qubits/64) (>=1).
 *   out_probs [W][2^b] UNNORMALISED clamped populations, float64;
 *   out_mass[W], out_min[W] = sum and minimum before clamping (guards are the
 *   caller's: engine.py:445-450, 475-476). */
int ptsbe_marginals(ptsbe_plan* plan, uint32_t stage, const uint8_t* kraus_idx,
                    const uint64_t* prefixes, uint64_t n_items, double* out_probs,
                    double* out_mass, double* out_min);

/* replaces: execute_path / contract_pair on one constant network
 * (tensor.py:190-268): runs the single program of a 1-stage plan for one item
 * and returns the complex result (out_elems values of the plan's dtype). */
int ptsbe_execute_raw(ptsbe_plan* plan, void* out_complex);

/* replaces: the multinomial split of one stage (engine.py:519-522) on given
 * float64 marginals, for sampler parity tests.  item w draws mult[w] outcomes
 * from probs[w][0..2^b) with Philox-4x32-10 counters
 * (draw, rank[w], stage, eset_id[w]) and key = seed.  Outputs: child_item[],
 * child_index[], child_count[] in item-major, index-ascending order. */
int ptsbe_sample_stage(uint32_t b, uint32_t stage, uint64_t seed, uint64_t n_items,
                       const double* probs, const uint32_t* mult, const uint32_t* eset_id,
                       const uint32_t* rank, uint32_t** child_item, uint32_t** child_index,
                       uint32_t** child_count, uint64_t* n_children, int device);

/* replaces: the fan-out over error sets + merge_records
 * (engine.py:885-906, sample_proportional engine.py:493-524, merge_records 815-829).
 *   kraus_idx [E][g], shots [E] (>=1), eset_ids [E] global ids used for the RNG
 *   streams (results do not depend on how error sets are split across calls).
 *   merged != 0: one histogram over all error sets, records sorted by key;
 *   merged == 0: per-error-set records, sorted by (position in this call, key),
 *                rec_eset[] filled with the position.
 *   keys [n_records][words]. */
int ptsbe_sample(ptsbe_plan* plan, const uint8_t* kraus_idx, const uint32_t* shots,
                 const uint32_t* eset_ids, uint64_t n_sets, uint64_t seed, int merged,
                 uint64_t** keys, uint32_t** rec_eset, uint64_t** counts,
                 uint64_t* n_records, ptsbe_run_stats* stats);

/* ptsbe_sample(merged != 0) with the histogram returned as records [n_records][2] uint32
 * (key, count), sorted by key: same run, same RNG streams, half the device-to-host bytes.
 * key = the high 32 bits of ptsbe_sample's key word (qubit q at bit 31 - q).
 * For plans that measure at most 32 qubits and calls of fewer than 2^32 shots in total
 * (PTSBE_EINVAL otherwise).  replaces: the same fan-out + merge_records (engine.py:885-906, 815-829)
 * for callers that fill RunResult.records from narrow integers. */
int ptsbe_sample_packed(ptsbe_plan* plan, const uint8_t* kraus_idx, const uint32_t* shots,
                        const uint32_t* eset_ids, uint64_t n_sets, uint64_t seed,
                        uint32_t** records, uint64_t* n_records, ptsbe_run_stats* stats);

/* replaces: sample_nonproportional per error set (engine.py:527-576), the data-harvesting mode.
 *   Every non-final stage branches each prefix into up to `nonfinal_shots` DISTINCT children
 *   (weighted choice without replacement, engine.py:549-556; outcomes below 2^-40 (c128) / 2^-17 (c64)
 *   of the row maximum count as zero probability); the final stage emits, per prefix,
 *   final_mode 0: every outcome whose conditional probability reaches `threshold`, count 1, tagged
 *                 with that probability in probs[] (engine.py:562-568),
 *   final_mode 1: a multinomial split of `direct_count` shots, probs[] = -1 (engine.py:569-574).
 *   Records are per error set, sorted by (position in this call, key): rec_eset[] holds the position.
 *   Uniforms: Philox counters (draw, prefix rank, stage, global error-set id), key = seed. */
int ptsbe_sample_nonproportional(ptsbe_plan* plan, const uint8_t* kraus_idx, const uint32_t* eset_ids,
                                 uint64_t n_sets, uint64_t seed, uint32_t nonfinal_shots,
                                 uint32_t final_mode, double threshold, uint32_t direct_count,
                                 uint64_t** keys, uint32_t** rec_eset, uint64_t** counts, double** probs,
                                 uint64_t* n_records, ptsbe_run_stats* stats);

/* resident variant for device-timed throughput: inputs are uploaded once,
 * every run leaves its histogram on the device and returns only its length. */
typedef struct ptsbe_batch ptsbe_batch;
int ptsbe_batch_upload(ptsbe_plan* plan, const uint8_t* kraus_idx, const uint32_t* shots,
                       const uint32_t* eset_ids, uint64_t n_sets, ptsbe_batch** out);
/* replaces: presample_errors / draw_realization (engine.py:232-281) for a uniform allocation of
 * shots_per_set shots: the Kraus-index matrix of error sets [first_id, first_id + n_sets) is drawn ON THE
 * DEVICE from the per-site outcome distributions and becomes a resident batch (no uint8[E][g] upload).
 *   site_off [g + 1], site_cdf [site_off[g]]: inclusive cumulative outcome probabilities per site
 *   (outcome 0 = no error, same order as the variant tables of the plan).
 *   uniform of (error set id, site): Philox counter (site, id, 'PRES', 0), key = seed. */
int ptsbe_batch_presample(ptsbe_plan* plan, const double* site_cdf, const uint32_t* site_off,
                          uint64_t n_sets, uint32_t first_id, uint32_t shots_per_set, uint64_t seed,
                          ptsbe_batch** out);
/* copy the Kraus-index matrix [n_sets][g] of a resident batch to the host (caller-allocated) */
int ptsbe_batch_kraus(ptsbe_batch* batch, uint8_t* out_host);
int ptsbe_batch_run(ptsbe_batch* batch, uint64_t seed, uint64_t* n_records,
                    ptsbe_run_stats* stats);
/* copy the histogram of the last run to the host (library-allocated) */
int ptsbe_batch_fetch(ptsbe_batch* batch, uint64_t** keys, uint64_t** counts,
                      uint64_t* n_records);
void ptsbe_batch_destroy(ptsbe_batch* batch);

/* replaces: merge_records across ranks after the gather (engine.py:815-829):
 * sums counts of equal keys, output sorted by key. keys [n][words]. */
int ptsbe_histogram_merge(const uint64_t* keys, const uint64_t* counts, uint64_t n,
                          uint32_t words, uint64_t** out_keys, uint64_t** out_counts,
                          uint64_t* n_out, int device);

/* replaces: find_path_greedy (planner.py:121-251), host code.
 *   operands are given as CSR lists of (label, dim); op_class / class_weight
 *   (optional, may be NULL) weight a step by the number of distinct instances
 *   of its result across the batch (error-independent hoisting);
 *   class_cap_log2 (optional) is a soft cap on log2(result entries) per class
 *   (records of hoisted classes may be larger than per-item on-chip buffers),
 *   size_cap_log2 the default for classes without one (0 = none);
 *   op_unit (optional) marks rank-1 basis-vector operands (prefix projectors):
 *   contracting one selects a slice of the other operand and is costed as such.
 *   merges_out [2*(n_ops-1)] stable-id pairs (result keeps the smaller id). */
int ptsbe_plan_greedy(uint32_t n_ops, const uint32_t* op_ptr, const int64_t* labels,
                      const uint32_t* dims, const uint32_t* op_class,
                      const double* class_weight, const double* class_cap_log2,
                      const uint8_t* op_unit, uint32_t n_classes, uint32_t hypersamples,
                      uint64_t seed, double size_cap_log2, uint32_t* merges_out,
                      double* cost_out, double* flops_out);

/* ---- device-pointer variants for the multi-GPU gather (one process per GPU;
 * the caller moves the buffers with NCCL and must synchronise its own stream
 * before handing pointers to the library) ---------------------------------- */

/* histogram of the last ptsbe_batch_run, left in HBM: keys_dev [n][words] u64,
 * counts_dev [n] u64.  Valid until the next run or ptsbe_batch_destroy. */
int ptsbe_batch_histogram_dev(ptsbe_batch* batch, const uint64_t** keys_dev,
                              const uint64_t** counts_dev, uint64_t* n_records);

/* ptsbe_histogram_merge on device buffers (merge_records after the NCCL gather,
 * engine.py:815-829).  Outputs are device buffers released with ptsbe_free_dev. */
int ptsbe_histogram_merge_dev(const uint64_t* keys_dev, const uint64_t* counts_dev, uint64_t n,
                              uint32_t words, int device, uint64_t** out_keys_dev,
                              uint64_t** out_counts_dev, uint64_t* n_out);
void ptsbe_free_dev(void* p_dev);

/* measurement helper for bench.py's roofline denominators: sustained
 * non-tensor FMA throughput of the device (independent FFMA / DFMA chains). */
int ptsbe_measure_fma_peak(int device, double* fp32_tflops, double* fp64_tflops);

void ptsbe_free(void* p);

/* Test / measurement probe of the dense projection step P[i][c] = Re(sum_d v_i[d] M_e(i)[d][c])
 * (the last np.tensordot of execute_path, tensor.py:190-216, engine.py:442-445) on raw complex64
 * arrays: v [n_items][D], m [n_sets][D][N], eset [n_items] sorted error-set rows; out [n_items][N].
 * use_tc = 1: tcgen05 / TMEM / TMA kernel (csrc/project_tc.cuh), 0: FP32 FMA kernel (csrc/project.cuh).
 * kernel_ms: device time of one launch (average of reps), prep_ms: building the B images (tc only). */
int ptsbe_project_probe(int device, uint32_t D, uint32_t N, uint64_t n_items, uint32_t n_sets,
                        const uint32_t* eset, const float* v, const float* m, int use_tc, float* out,
                        int reps, float* kernel_ms, float* prep_ms);

#ifdef __cplusplus
}
#endif
#endif /* PTSBE_B200_H */
