/*
 * mmgpu.h — C ABI of the B200 metric + move-method engine (libmmgpu.so).
 *
 * This is the drop-in boundary for the reference library's hot path
 * (/root/reference/proj/include/modmetrics/{metrics,parallel,suggest}.hpp).
 * Plain C: fixed-width integers, raw pointers and sizes, no C++ or torch
 * types, no exception crosses it. Every entry point returns an mm_status;
 * the status codes map one-to-one onto the exception types the reference
 * throws (see MM_E_RANGE / MM_E_ARG below), and include/modmetrics/gpu.hpp
 * rethrows exactly those types for C++ callers.
 *
 * Each function cites the reference interface it replaces (file:line, paths
 * relative to /root/reference/proj/include/modmetrics/).
 *
 * Threading: one mm_ctx == one CUDA device + one CUDA stream. A context is
 * not thread-safe; distinct contexts — one per GPU, or several on one GPU to
 * pipeline requests — may be driven from distinct host threads or processes
 * (tests/test_gpu_concurrency.py).
 */
#ifndef MMGPU_H
#define MMGPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MMGPU_ABI_VERSION 1

typedef enum mm_status {
    MM_OK = 0,
    MM_E_RANGE = 1,       /* std::out_of_range  (metrics.hpp:97-100, suggest.hpp:89-90, model.hpp:66-67) */
    MM_E_ARG = 2,         /* std::invalid_argument (suggest.hpp:91-96, :313, parallel.hpp:29, generate.hpp:97-100) */
    MM_E_CUDA = 3,        /* CUDA runtime failure (no device, launch error, ...) */
    MM_E_OOM = 4,         /* device allocation failed */
    MM_E_STATE = 5,       /* call order violated (e.g. sweep before upload) */
    MM_E_UNSUPPORTED = 6, /* outside this engine's scope (e.g. Criterion::Similarity) */
    MM_E_CAPACITY = 7,    /* caller buffer too small; *n_out holds the needed count */
    MM_E_PARSE = 8,       /* modmetrics::ParseError      (facts.hpp:22-24), see mmfacts.h */
    MM_E_VALIDATION = 9,  /* modmetrics::ValidationError (facts.hpp:28-37) */
    MM_E_IO = 10,         /* modmetrics::IoError         (facts.hpp:39-41) */
    MM_E_NCCL = 11        /* NCCL missing or failing (multi-GPU groups, mm_group_*) */
} mm_status;

/* Criterion bits: bit (1 << Criterion) with Criterion as in suggest.hpp:17
 * (Similarity = 0, Cohesion = 1, Coupling = 2). */
#define MM_CRIT_SIMILARITY (1u << 0)
#define MM_CRIT_COHESION (1u << 1)
#define MM_CRIT_COUPLING (1u << 2)

/* Combine, suggest.hpp:296 */
#define MM_COMBINE_UNION 0
#define MM_COMBINE_INTERSECTION 1

/*
 * A system snapshot in CSR form: SystemModel + DependencyTable
 * (model.hpp:19-53) with every vector<vector<u32>> flattened to
 * (offsets, values). Host memory; mm_upload copies it.
 *
 * Preconditions are the reference's: the model passes validate()
 * (model.hpp:113-212): ids dense, membership partitions each id space and
 * agrees with the owner tables, every member/dependency list sorted unique,
 * no self-calls. mm_upload range-checks every id on the device and fails
 * with MM_E_ARG instead of faulting; the sorted/unique/partition invariants
 * are the caller's contract exactly as in the reference.
 * Edge counts are limited to < 2^32 per table (u32 offsets).
 * method_owner / attribute_owner may be NULL: the device then derives them
 * from the membership lists (identical under the precondition above) and
 * the upload moves 4·(n_methods + n_attributes) fewer bytes.
 */
typedef struct mm_system {
    uint32_t n_classes;
    uint32_t n_methods;
    uint32_t n_attributes;
    uint32_t reserved;
    const uint32_t* method_owner;     /* [n_methods]      SystemModel::method_owner (model.hpp:35) */
    const uint32_t* attribute_owner;  /* [n_attributes]   SystemModel::attribute_owner (model.hpp:36) */
    const uint32_t* class_method_off; /* [n_classes + 1]  ClassRecord::method_ids, concatenated (model.hpp:23) */
    const uint32_t* class_methods;    /* [n_methods] */
    const uint32_t* class_attr_off;   /* [n_classes + 1]  ClassRecord::attribute_ids, concatenated (model.hpp:22) */
    const uint32_t* class_attrs;      /* [n_attributes] */
    const uint32_t* call_off;         /* [n_methods + 1]  DependencyTable::calls (model.hpp:49) */
    const uint32_t* call_tgt;         /* [call_off[n_methods]] */
    const uint32_t* acc_off;          /* [n_methods + 1]  DependencyTable::accesses (model.hpp:50) */
    const uint32_t* acc_tgt;          /* [acc_off[n_methods]] */
} mm_system;

/* WhatIfMetrics, suggest.hpp:72-85 (same field order and types). */
typedef struct mm_whatif {
    double lcom_origin_before;
    double lcom_origin_after;
    double lcom_dest_before;
    double lcom_dest_after;
    uint32_t cbo_origin_before;
    uint32_t cbo_origin_after;
    uint32_t cbo_dest_before;
    uint32_t cbo_dest_after;
    uint8_t origin_degenerate_after;
    uint8_t dest_degenerate_after;
    uint8_t pad[6];
} mm_whatif; /* 56 bytes */

/* MoveSuggestion, suggest.hpp:124-132: 64-byte record. `criteria` is the
 * sorted-unique criteria vector as a bit set of MM_CRIT_* bits. */
typedef struct mm_suggestion {
    double lcom_origin_before;
    double lcom_origin_after;
    double lcom_dest_before;
    double lcom_dest_after;
    uint32_t method;
    uint32_t origin;
    uint32_t destination;
    uint32_t cbo_origin_before;
    uint32_t cbo_origin_after;
    uint32_t cbo_dest_before;
    uint32_t cbo_dest_after;
    uint8_t criteria;
    uint8_t origin_degenerate_after;
    uint8_t dest_degenerate_after;
    uint8_t pad;
} mm_suggestion; /* 64 bytes */

/* ThresholdOverrides / Thresholds, suggest.hpp:28-41. has_* = optional engaged. */
typedef struct mm_overrides {
    uint8_t has_similarity, has_lcom, has_cbo, pad;
    double similarity;
    double lcom;
    double cbo;
} mm_overrides;

typedef struct mm_thresholds {
    double similarity;
    double lcom;
    double cbo;
    uint8_t explicit_mode;
    uint8_t pad[7];
} mm_thresholds;

/* Parameters of one candidate sweep: suggest_all (suggest.hpp:303) over
 * criteria ⊆ {Cohesion, Coupling}, or a single suggest_by_* when one bit is
 * set. `class_begin/class_end` restrict the sweep to origins in that class
 * range (the multi-GPU shard); [0, n_classes) is the whole system.
 * top_k: 0 or 1 = the reference's best-only mode; k > 1 keeps the k best
 * passing destinations per (criterion, method) (an extension; ordered like
 * all_candidates output). all_candidates = SuggestOptions::all_candidates
 * (suggest.hpp:134-138) and overrides top_k. */
typedef struct mm_sweep_params {
    uint32_t criteria;       /* MM_CRIT_* bits */
    uint32_t combine;        /* MM_COMBINE_* */
    uint32_t all_candidates; /* 0/1 */
    uint32_t top_k;          /* 0/1 = best only */
    double thr_lcom;         /* Thresholds::lcom  (gate: lcom[c] > thr_lcom, suggest.hpp:246) */
    double thr_cbo;          /* Thresholds::cbo   (gate: (double)cbo[c] > thr_cbo, suggest.hpp:273) */
    uint32_t class_begin;
    uint32_t class_end;      /* 0 == n_classes, unless flags has MM_SWEEP_EXACT_RANGE */
    uint32_t threshold_source; /* MM_THR_EXPLICIT: thr_lcom/thr_cbo above;
                                  MM_THR_DEVICE_MEANS: the means computed on the device by the
                                  last mm_compute_metrics (compute_thresholds with no overrides),
                                  read without a host round trip */
    uint32_t flags;          /* MM_SWEEP_* */
} mm_sweep_params;

#define MM_THR_EXPLICIT 0
#define MM_THR_DEVICE_MEANS 1
/* class_end is taken literally (an empty range [b, b) sweeps nothing) */
#define MM_SWEEP_EXACT_RANGE 1u

typedef struct mm_sweep_stats {
    uint64_t candidates;     /* (method, destination) pairs scored, ungated: Σ|used_classes(u)| */
    uint64_t gated_whatifs;  /* what-ifs the reference would evaluate: per criterion, gated classes only */
    uint64_t suggestions;    /* records emitted */
    uint64_t methods;        /* methods swept */
} mm_sweep_stats;

typedef struct mm_kernel_stat {
    char name[32];
    uint64_t launches;
    double total_ms; /* CUDA-event time summed over launches (profiling on) */
} mm_kernel_stat;

typedef struct mm_ctx mm_ctx;

/* ---- context ---------------------------------------------------------- */
mm_status mm_ctx_create(int device, mm_ctx** out);
void mm_ctx_destroy(mm_ctx* ctx);
const char* mm_last_error(const mm_ctx* ctx); /* never NULL */
int mm_abi_version(void);
/* CUDA devices visible to this process (0 when none or no driver). */
int mm_device_count(void);
/* Run all work on this cudaStream_t (e.g. torch's current stream). NULL = the ctx's own stream. */
mm_status mm_ctx_set_stream(mm_ctx* ctx, void* cuda_stream);
mm_status mm_ctx_synchronize(mm_ctx* ctx);
/* The stream the context's work runs on (its own, or the one set above). */
mm_status mm_ctx_stream(mm_ctx* ctx, void** cuda_stream);
/* Per-kernel CUDA-event timing (adds two event records per launch). */
mm_status mm_ctx_set_profiling(mm_ctx* ctx, int on);
mm_status mm_kernel_stats(mm_ctx* ctx, mm_kernel_stat* out, int cap, int* n_out);
mm_status mm_reset_kernel_stats(mm_ctx* ctx);

/* ---- model upload (replaces passing const SystemModel&, const DependencyTable&) ---- */
mm_status mm_upload(mm_ctx* ctx, const mm_system* sys);
/* Bytes of the uploaded CSR (what one H2D of the system costs). */
uint64_t mm_system_bytes(const mm_system* sys);

/* ---- class metric pass ------------------------------------------------ */
/* Device-resident recompute of per-class LCOM (normalized), LCOM-CK, CBO and
 * the class×class use-count table. Replaces full_report's class loop
 * (metrics.hpp:253-261) / parallel_class_metrics (parallel.hpp:149) +
 * parallel_lcom_ck (parallel.hpp:164). No host copy. */
mm_status mm_compute_metrics(mm_ctx* ctx);
/* Copies results (any pointer may be NULL). Runs mm_compute_metrics first if
 * the model changed since the last pass.
 *   lcom    == lcom_normalized per class (metrics.hpp:128)
 *   lcom_ck == lcom_ck per class         (metrics.hpp:159)
 *   cbo     == cbo per class             (metrics.hpp:187) */
mm_status mm_class_metrics(mm_ctx* ctx, double* lcom, uint64_t* lcom_ck, uint32_t* cbo);
/* The same copies, only enqueued: they run on a copy stream behind the work
 * already launched and overlap what is launched next (e.g. mm_sweep). The
 * buffers (pinned, for a truly asynchronous copy) hold the results after
 * mm_ctx_synchronize; the next metric pass waits for the copies. */
mm_status mm_class_metrics_async(mm_ctx* ctx, double* lcom, uint64_t* lcom_ck, uint32_t* cbo);
/* Per-method fan metrics (either pointer may be NULL), MetricsReport::fan_in
 * / fan_out: fan_in[p] = number of call lists containing p (metrics.hpp:79-85,
 * = parallel_fan_metrics' fan_in for a validated model, parallel.hpp:186-206),
 * fan_out[p] = |calls(p)| (metrics.hpp:87-93). */
mm_status mm_fan_metrics(mm_ctx* ctx, uint32_t* fan_in, uint32_t* fan_out);
/* WorkloadEstimate, metrics.hpp:195-233 (same fields and order): the largest
 * call / access set from a device max-reduce, the closed forms of
 * estimate_workload_counts on top. */
typedef struct mm_workload {
    uint64_t m, c, k_m, k_a, n_fan, n_sim, n_lcom, n_cbo, n_total;
} mm_workload;
mm_status mm_estimate_workload(mm_ctx* ctx, mm_workload* out);
/* Single-class accessors with the reference's error behaviour
 * (out_of_range on a bad id, metrics.hpp:97-100). */
mm_status mm_lcom_normalized(mm_ctx* ctx, uint32_t cls, double* out);
mm_status mm_lcom_ck(mm_ctx* ctx, uint32_t cls, uint64_t* out);
mm_status mm_cbo(mm_ctx* ctx, uint32_t cls, uint32_t* out);

/* ---- thresholds (compute_thresholds, suggest.hpp:46-61) --------------- */
/* compute_thresholds(full_report(...), ov): means of the device-resident
 * per-class lcom / cbo (computed on the device by the metric pass) and of the
 * device similarity table's values in table order (built here when absent,
 * like full_report's similarity field), each bit-identical to the reference's
 * sequential double sum; an override replaces its mean and sets
 * explicit_mode. */
mm_status mm_compute_thresholds(mm_ctx* ctx, const mm_overrides* ov, mm_thresholds* out);
/* compute_thresholds(report, ov) (suggest.hpp:46-61) on a caller's report:
 * report.lcom, report.cbo and report.similarity's values (host memory,
 * copied), each mean computed on the device with the reference's sequential
 * left-to-right double-sum semantics, bit-identical; empty -> 0. */
mm_status mm_report_thresholds(mm_ctx* ctx, const double* lcom, uint64_t n_lcom, const uint32_t* cbo, uint64_t n_cbo,
                               const double* similarity, uint64_t n_sim, const mm_overrides* ov, mm_thresholds* out);
/* Mean of caller-supplied doubles with compute_thresholds' sequential
 * left-to-right double-sum semantics (suggest.hpp:48-53), bit-identical,
 * computed on the device (always the parallel exact emulation when its
 * preconditions hold; serial device loop otherwise). *fast_path (may be NULL)
 * reports which ran.
 * Used for caller-built report vectors and to test the threshold kernel. */
mm_status mm_sequential_mean(mm_ctx* ctx, const double* values, uint64_t n, double* out, int* fast_path);

/* ---- similarity table (all_similarities, metrics.hpp:39-77) ----------- */
/* SimilarityEntry, metrics.hpp:31-37 (same field order and types). */
typedef struct mm_similarity {
    uint32_t first;   /* first < second */
    uint32_t second;
    double value;     /* |shared properties| / |union|, the reference's single division */
} mm_similarity;      /* 16 bytes */
/* Every unordered method pair with a nonzero Jaccard similarity of their
 * property sets (calls and accesses, the two id spaces kept apart), ordered
 * by (first, second) — all_similarities / parallel_similarities
 * (parallel.hpp:71-121). Two-call size query: out may be NULL; *n_out gets
 * the count; MM_E_CAPACITY when cap is smaller. Any row length: rows beyond
 * a warp's shared-memory buffer go through global scratch in batches.
 * MM_E_UNSUPPORTED only past 2^32 - 1 pairs in all (u32 row offsets). */
mm_status mm_similarities(mm_ctx* ctx, mm_similarity* out, uint64_t cap, uint64_t* n_out);

/* suggest_by_similarity (suggest.hpp:200-232): pairs of `table` (the
 * caller's report.similarity; NULL = the device table of mm_similarities)
 * with value > thr and methods in different classes make both methods
 * candidates, destinations = the partner's class + the owners of what the
 * method calls; a move passes when both lcoms strictly drop, best by
 * lcom_key (lowest destination on ties) or every passing one
 * (all_candidates). Records carry MM_CRIT_SIMILARITY, ordered by method
 * then destination (the reference's order). Two-call size query. */
mm_status mm_suggest_similarity(mm_ctx* ctx, const mm_similarity* table, uint64_t n_table, double thr,
                                uint32_t all_candidates, mm_suggestion* out, uint64_t cap, uint64_t* n_out);

/* ---- what-if (what_if_move, suggest.hpp:87-122) ----------------------- */
mm_status mm_what_if(mm_ctx* ctx, uint32_t method, uint32_t origin, uint32_t destination,
                     mm_whatif* out);

/* ---- candidate sweep (suggest_by_cohesion/coupling, suggest_all) ------- */
/* Class gates from the caller's MetricsReport (report.lcom / report.cbo,
 * n_classes entries each, host memory, copied): the reference gates on the
 * report it is given (suggest.hpp:246, :273), which need not be this
 * engine's own metrics. Both NULL: gate on the device-computed metrics
 * (the default). */
mm_status mm_set_gates(mm_ctx* ctx, const double* lcom, const uint32_t* cbo);
/* Runs the sweep on the device; the ordered result stays resident.
 * n_out (may be NULL) receives the record count (a D2H of 8 bytes). */
mm_status mm_sweep(mm_ctx* ctx, const mm_sweep_params* p, uint64_t* n_out);
/* One full step — mm_compute_metrics + mm_sweep(p) — replayed from a CUDA
 * graph captured on the first call (re-captured when the parameters, the
 * model, the gates, the stream or profiling change). No host
 * synchronisation. MMGPU_NO_GRAPH=1 runs it eagerly. */
mm_status mm_run(mm_ctx* ctx, const mm_sweep_params* p);
/* With profiling on and a graph replay, accumulates the kernel times of the
 * LAST replay into mm_kernel_stats (synchronises the context's streams). */
mm_status mm_collect_timings(mm_ctx* ctx);
/* Device pointer to the last sweep's records (mm_suggestion[n]), for
 * device-side exchange (NCCL all-gather) without a host round trip. */
mm_status mm_sweep_device_result(mm_ctx* ctx, const void** dev_records, uint64_t* n);
/* Device address of the last sweep's record count (uint64, written by the
 * sweep's kernels on the context's stream): device-side exchanges read it
 * without a host round trip (mm_group_run all-gathers it over NCCL). */
mm_status mm_sweep_device_count(mm_ctx* ctx, const uint64_t** dev_count);
mm_status mm_sweep_stats_get(mm_ctx* ctx, mm_sweep_stats* out);
/* Copies the last sweep's records to host memory; MM_E_CAPACITY (with
 * *n_out = needed) when cap is too small. */
mm_status mm_copy_suggestions(mm_ctx* ctx, mm_suggestion* out, uint64_t cap, uint64_t* n_out);
/* mm_sweep + mm_copy_suggestions: the reference-facing one-call form of
 * suggest_all(model, deps, report, thresholds, criteria, combine, opts). */
mm_status mm_suggest(mm_ctx* ctx, const mm_sweep_params* p, mm_suggestion* out, uint64_t cap,
                     uint64_t* n_out);

/* Page-locked host buffers for the caller's inputs/outputs: copies from/to
 * pinned memory run at full DMA rate (pageable memory is staged by the
 * driver). */
mm_status mm_pinned_alloc(uint64_t bytes, void** out);
void mm_pinned_free(void* p);

/* ---- multi-GPU groups (SURVEY.md §8b mm_comm_init, §8e) ---------------- */
/* One process, n GPUs: the reference's n_workers (parallel.hpp:149, :164,
 * plan_partition :20-41) mapped to GPUs. Each GPU holds the whole system and
 * recomputes the metric pass (replicas); the candidate sweep runs on
 * cost-balanced contiguous class ranges (mm_plan_shards), and the shard
 * lists are exchanged over NCCL with exact counts — an all-gather of the
 * per-GPU record counts, then one broadcast per non-empty shard of exactly
 * its records into every GPU's assembled list — which in rank order is
 * suggest_all's ordered list (suggest.hpp:344-348). NCCL is dlopen'ed
 * (libnccl.so.2); a one-GPU group needs none. devices == NULL: 0..n-1.
 * n == 0 -> MM_E_ARG (plan_partition's zero-worker check, parallel.hpp:29);
 * a bad or repeated device -> MM_E_RANGE; NCCL unusable for n > 1 ->
 * MM_E_NCCL. mm_group_ctx gives each GPU's context (metrics, what-if, ...). */
typedef struct mm_group mm_group;
mm_status mm_group_create(const int* devices, int n, mm_group** out);
void mm_group_destroy(mm_group* g);
const char* mm_group_last_error(const mm_group* g);
int mm_group_size(const mm_group* g);
int mm_group_uses_nccl(const mm_group* g);
mm_ctx* mm_group_ctx(mm_group* g, int i);
/* Upload to every GPU (one host thread each) and plan the shards. */
mm_status mm_group_upload(mm_group* g, const mm_system* sys);
/* Shard i's class range [*class_begin, *class_end). */
mm_status mm_group_shard(const mm_group* g, int i, uint32_t* class_begin, uint32_t* class_end);
/* mm_set_gates on every GPU. */
mm_status mm_group_set_gates(mm_group* g, const double* lcom, const uint32_t* cbo);
/* One step on every GPU — metric pass + the sweep of its shard (mm_run with
 * p's criteria/modes/thresholds; p's class range is replaced by the shard)
 * — then the exact-count exchange. n_out (may be NULL: no host sync)
 * receives the assembled list's length. */
mm_status mm_group_run(mm_group* g, const mm_sweep_params* p, uint64_t* n_out);
mm_status mm_group_synchronize(mm_group* g);
/* Per-shard record counts (n entries, may be NULL) and their total. */
mm_status mm_group_counts(const mm_group* g, uint64_t* counts, uint64_t* total);
/* GPU i's copy of the assembled list (device memory). */
mm_status mm_group_device_result(mm_group* g, int i, const void** dev_records, uint64_t* n);
/* The assembled list to host memory (from GPU 0); MM_E_CAPACITY when small. */
mm_status mm_group_copy_suggestions(mm_group* g, mm_suggestion* out, uint64_t cap, uint64_t* n_out);

/* ---- host-side helpers (no GPU needed) --------------------------------- */
/* Contiguous class ranges balanced by sweep cost (Σ over members of
 * 1 + |calls| + |accesses|), the GPU analogue of plan_partition
 * (parallel.hpp:28-41). bounds has n_shards + 1 entries. n_shards == 0 ->
 * MM_E_ARG like plan_partition's zero-worker check. */
mm_status mm_plan_shards(const mm_system* sys, uint32_t n_shards, uint32_t* bounds);

/* Synthetic systems. mm_gen_config mirrors GeneratorConfig (generate.hpp:39-47);
 * zipf_s > 0 selects the skewed-size variant:
 * class sizes ∝ 1/rank^s, ids shuffled over classes by SplitMix64, deps drawn
 * exactly as generate.hpp:124-161. */
typedef struct mm_gen_config {
    uint64_t seed;
    uint32_t n_classes;
    uint32_t n_methods;
    uint32_t n_attributes;
    uint32_t k_max_calls;
    uint32_t k_max_accesses;
    uint32_t pad;
    double intra_class_bias;
    double zipf_s; /* 0 = reference round-robin generate() */
} mm_gen_config;

typedef struct mm_host_system mm_host_system;
mm_status mm_generate(const mm_gen_config* cfg, mm_host_system** out);
const mm_system* mm_host_system_view(const mm_host_system* h);
void mm_host_system_free(mm_host_system* h);

#ifdef __cplusplus
}
#endif
#endif /* MMGPU_H */
