// mm_api.cu — the C ABI (include/mmgpu.h): context, upload, metric pass,
// thresholds, what-if, sweep. Host orchestration only; all arithmetic on the
// hot path runs in the kernels of k_metrics.cu / k_sweep.cu. There is no CPU
// fallback: without a usable CUDA device every compute entry point fails
// with MM_E_CUDA.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstddef>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <map>
#include <new>
#include <string>
#include <type_traits>
#include <vector>

#include "../../include/mmgpu.h"
#include "mm_device.cuh"
#include "mm_kernels.h"

using namespace mmg;

namespace {

// CTA-path classes count foreign classes in an smem histogram when 4·C fits this
constexpr uint64_t kHistMaxBytes = 64 * 1024;
constexpr int kMaxTiers = 8;  // CTA-path launch groups (shared-memory tier x CTA size)
constexpr uint64_t kBigCtaMembers = 2048;  // classes this large launch 1024-thread CTAs
constexpr int kUploadArrays = 10;
constexpr uint32_t kNoSlot = 0xffffffffu;
constexpr uint64_t kCkMmaMin = 128;      // dense classes this large count LCOM-CK pairs with tcgen05 MMA
constexpr uint64_t kCkMmaMaxMembers = 3328;  // operand rows × 64 B must fit shared memory

struct Ctl {  // small device-resident control block
    uint32_t bad;
    uint32_t n_large;
    uint32_t max_deg;
    uint32_t ucursor;
    uint32_t dense_cursor;
    uint32_t n_big;     // warp-path classes with > 32 U-row keys
    uint32_t tile_counter;
    uint32_t err;
    uint32_t n_emit;
    uint32_t n_wide;    // top-k / all-candidates methods with >= 32 used classes (side table)
    uint32_t n_fallback;  // best-only: methods k_score_fast handed to the per-thread kernel
    uint32_t n_hideg;     // upload plan: methods with more than kRecMaxEnt edges
    unsigned long long stats[4];
    DevThresholds thr;
    DevThresholds thr_aux;  // mm_sequential_mean / the similarity mean (never the metric pass's means)
    uint32_t n_groups;      // upload plan: k_class_group warps
    uint32_t n_solo;        // upload plan: lean classes for k_class_lean
    uint32_t n_nl;          // upload plan: positions of the classes that are not lean
};

struct KStat {
    uint64_t launches = 0;
    double total_ms = 0.0;
};

struct Pending {
    std::string name;
    cudaEvent_t a, b;
};

template <class T>
struct DBuf {  // owning device buffer (freed on release() or destruction)
    T* p = nullptr;
    size_t n = 0;
    DBuf() = default;
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    ~DBuf() { release(); }
    cudaError_t alloc(size_t count) {
        release();
        n = count;
        if (count == 0) return cudaSuccess;
        return cudaMalloc(reinterpret_cast<void**>(&p), count * sizeof(T));
    }
    cudaError_t ensure(size_t count) { return count <= n && p ? cudaSuccess : alloc(count); }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
};

template <class T>
struct HBuf {  // owning pinned host buffer, grown on demand (upload-time staging)
    T* p = nullptr;
    size_t n = 0;
    HBuf() = default;
    HBuf(const HBuf&) = delete;
    HBuf& operator=(const HBuf&) = delete;
    ~HBuf() { release(); }
    cudaError_t ensure(size_t count) {
        if (count <= n && p) return cudaSuccess;
        release();
        n = count ? count : 1;
        return cudaMallocHost(reinterpret_cast<void**>(&p), n * sizeof(T));
    }
    void release() {
        if (p) cudaFreeHost(p);
        p = nullptr;
        n = 0;
    }
};

}  // namespace

struct mm_ctx {
    int device = 0;
    cudaStream_t own = nullptr;
    cudaStream_t stream = nullptr;
    cudaStream_t side = nullptr;       // threshold means run here, overlapping the candidate scoring
    cudaEvent_t ev_metrics = nullptr;  // class tables ready (main -> side)
    // CTA-path tiers run on their own streams, concurrently with the warp path
    cudaStream_t aux[kMaxTiers + 3] = {};  // + the listed warp-path classes, + tensor-core LCOM-CK, + lean classes
    cudaEvent_t ev_fork = nullptr, ev_fork0 = nullptr;
    cudaEvent_t ev_join[kMaxTiers + 3] = {};
    cudaEvent_t ev_up[kUploadArrays] = {};  // per-array copy done (upload validation overlaps the copies)
    cudaStream_t d2h = nullptr;             // mm_class_metrics_async copies
    cudaEvent_t ev_d2h_go = nullptr, ev_d2h_done = nullptr;
    cudaEvent_t ev_thr = nullptr;      // threshold means ready (side -> main)
    std::string err;
    bool profiling = false;
    std::vector<Pending> pending;
    std::map<std::string, KStat> kstats;

    // model
    bool have_model = false;
    bool metrics_valid = false;
    uint32_t C = 0, M = 0, A = 0;
    uint64_t Ec = 0, Ea = 0;
    std::vector<uint32_t> h_cls_moff;
    // upload-time pinned staging: the CTA-path list and foreign counts (D2H),
    // the host-built plan tables (H2D, asynchronous: the next upload syncs
    // the stream before reusing it)
    HBuf<uint32_t> hs_list, hs_fr;
    HBuf<unsigned char> hs_up;
    DBuf<uint32_t> method_owner, attribute_owner, cls_moff, cls_methods, cls_aoff, cls_attrs, call_off, call_tgt,
        acc_off, acc_tgt;
    // plan
    uint32_t n_large = 0, max_deg = 0;
    uint32_t n_maybe_ovf = 0;  // upper bound of record-overflow methods (upload plan)
    struct LargeGroup {
        uint32_t first, count, smem;
        int key;           // 2 * shared-memory tier + (1024-thread CTAs)
        uint32_t threads;
        uint32_t item_first, n_items, split_first, n_split;  // split LCOM-CK work of this group
        uint32_t giant_first, n_giant_items;                  // k_giant_p1 work of this group
    };
    std::vector<LargeGroup> large_groups;  // CTA-path launches, grouped by shared-memory need
    DBuf<uint32_t> dense;                  // exact U-row bitmaps of dense classes
    uint32_t dense_cap = 0;
    uint64_t hist_max_bytes = kHistMaxBytes;  // env MMGPU_HIST_MAX_BYTES (tuning / tests)
    uint64_t giant_min = kGiantMembers;       // env MMGPU_GIANT_MIN (tuning / tests)
    uint64_t ck_mma_min = kCkMmaMin;          // env MMGPU_CK_MMA_MIN: tensor-core LCOM-CK from this many members
    DBuf<uint32_t> mma_list;                  // classes whose LCOM-CK runs on the tensor cores
    uint32_t n_mma = 0, mma_smem = 0;
    DBuf<uint2> ck_items;                  // (large index, first member) chunks of split LCOM-CK classes
    DBuf<uint32_t> split_list;             // the split classes
    uint32_t n_ck_items = 0, n_split = 0;
    DBuf<uint2> giant_items;           // k_giant_p1 CTAs
    DBuf<uint32_t> gcnt;               // giants' foreign-class histograms (C words each)
    DBuf<unsigned long long> gH;       // giants' H
    uint32_t n_giant = 0;
    uint64_t grows_words = 0;              // global attribute-bitmap scratch in use
    DBuf<uint4> cplan;         // per class (first member position, M, A, kind)
    DBuf<uint4> cedge;         // per class: its call and access edge ranges in the class-order rows
    DBuf<uint8_t> pc_mem, pa_mem;  // per class-order edge: member index inside its class (255: beyond)
    bool lean_fused = true;    // env MMGPU_LEAN=0: lean classes through k_method + k_class_small (A/B)
    uint32_t n_lean = 0;       // classes k_class_lean handles (0 when lean_fused is off)
    DBuf<uint32_t> nl_pos;     // class-order positions of the other classes (k_method's list when mixed)
    uint32_t n_nl = 0;
    bool group_on = true;        // env MMGPU_GROUP=0: every lean class on k_class_lean (warp per class)
    DBuf<uint2> groups;          // k_class_group: (first class, classes)
    DBuf<uint32_t> solo;         // lean classes outside the groups (member degree > 8)
    uint32_t n_groups = 0, n_solo = 0;
    bool score_fast = true;      // env MMGPU_SCORE_FAST=0: best-only scoring on the general per-thread kernel
    int prio_lo = 0, prio_hi = 0;  // stream priority range of the device
    DBuf<uint32_t> big_list;   // kKindWarpBig classes
    uint32_t n_big = 0;
    DBuf<uint32_t> large_list, foreign, cmaxdeg;
    DBuf<LargePlan> plans;
    DBuf<uint32_t> gkeys;
    DBuf<uint32_t> grows;
    // derived
    DBuf<uint32_t> cbo, ux, un;
    DBuf<MethRec> recs;
    DBuf<uint64_t> own_mask;
    DBuf<uint2> attr_info;
    DBuf<uint32_t> fan;  // mm_fan_metrics: fan_in[m] then fan_out[m]
    // similarity table: inverted indices, per-row counts / offsets, the pairs
    DBuf<uint32_t> sim_u32;               // uc_off | uc | ua_off | ua | cursors | totals | row_cnt | row_off | wide
    DBuf<unsigned long long> sim_ctl;     // [0] Σ pairs, [1] (n_wide, err, grand)
    DBuf<mm_similarity> sim_out;
    DBuf<mm_similarity> sim_caller;       // a caller's table (mm_suggest_similarity)
    DBuf<uint32_t> simc_u32;              // partner counts / offsets / cursors / classes, record counts / offsets
    DBuf<mm_suggestion> simc_out;
    uint64_t sim_n = 0;
    bool sim_valid = false;
    DBuf<uint32_t> pos_owner;
    DBuf<uint32_t> pc_off, pc_tgt, pa_off, pa_tgt, pos_scan;  // dependency rows in class order (+ scan scratch)
    DBuf<uint4> res;
    DBuf<uint4> emit_list;  // compact emitter records (k_offsets -> k_write)
    DBuf<uint4> wide_cnt;  // top-k / all-candidates: pass counts of methods with >= 32 used classes
    DBuf<uint32_t> fallback;  // best-only: record-overflow positions (k_score_fast -> k_score_thread)
    bool thr_side = true;     // env MMGPU_THR_SIDE=0: threshold means on the main stream, ahead of the sweep
    DBuf<double> gate_lcom;
    DBuf<uint32_t> gate_cbo;
    bool gates_set = false;
    DBuf<ClassRec> rec;
    DBuf<double> lcom;
    DBuf<uint64_t> ck;
    // control / sweep
    DBuf<Ctl> ctl;
    DBuf<unsigned long long> tile_state;
    DBuf<mm_suggestion> out;
    DBuf<mm_whatif> whatif;
    DBuf<char> thr_scratch;
    bool sweep_valid = false;
    // CUDA graph of one full step (mm_run)
    bool capturing = false;
    bool graph_disabled = false;
    cudaGraphExec_t graph_exec = nullptr;
    std::vector<uint8_t> graph_key;
    std::vector<Pending> graph_events;  // event pairs recorded by graph nodes (profiling)
    uint64_t layout_gen = 0;            // bumped whenever a device buffer the graph uses moves

    DevModel dev() const {
        DevModel s;
        s.C = C; s.M = M; s.A = A;
        s.method_owner = method_owner.p; s.attribute_owner = attribute_owner.p;
        s.cls_moff = cls_moff.p; s.cls_methods = cls_methods.p;
        s.cls_aoff = cls_aoff.p; s.cls_attrs = cls_attrs.p;
        s.call_off = call_off.p; s.call_tgt = call_tgt.p;
        s.acc_off = acc_off.p; s.acc_tgt = acc_tgt.p;
        s.attr_info = attr_info.p;
        s.pc_off = pc_off.p; s.pc_tgt = pc_tgt.p;
        s.pa_off = pa_off.p; s.pa_tgt = pa_tgt.p;
        return s;
    }
};

namespace {

mm_status fail(mm_ctx* ctx, mm_status st, const std::string& msg) {
    if (ctx) ctx->err = msg;
    return st;
}

mm_status cuda_fail(mm_ctx* ctx, cudaError_t e, const char* where) {
    return fail(ctx, e == cudaErrorMemoryAllocation ? MM_E_OOM : MM_E_CUDA,
                std::string(where) + ": " + cudaGetErrorString(e));
}

#define MM_CUDA(ctx, call)                                   \
    do {                                                     \
        cudaError_t e_ = (call);                             \
        if (e_ != cudaSuccess) return cuda_fail(ctx, e_, #call); \
    } while (0)

template <class F>
mm_status run_on(mm_ctx* ctx, cudaStream_t st, const char* name, F&& launch) {
    Pending pe;
    // during graph capture the timing events must become external event-record
    // nodes, readable after each replay
    const unsigned rec_flags = ctx->capturing ? cudaEventRecordExternal : cudaEventRecordDefault;
    if (ctx->profiling) {
        cudaEventCreate(&pe.a);
        cudaEventCreate(&pe.b);
        cudaEventRecordWithFlags(pe.a, st, rec_flags);
    }
    mm_status inner = MM_OK;
    if constexpr (std::is_same_v<decltype(launch()), mm_status>) inner = launch();
    else launch();
    const cudaError_t e = cudaGetLastError();
    if (ctx->profiling) {
        cudaEventRecordWithFlags(pe.b, st, rec_flags);
        pe.name = name;
        (ctx->capturing ? ctx->graph_events : ctx->pending).push_back(pe);
    }
    if (inner != MM_OK) return inner;
    if (e != cudaSuccess) return cuda_fail(ctx, e, name);
    return MM_OK;
}

template <class F>
mm_status run(mm_ctx* ctx, const char* name, F&& launch) {
    return run_on(ctx, ctx->stream, name, launch);
}

// main stream waits for the side stream's threshold means
mm_status join_thresholds(mm_ctx* ctx) {
    const cudaError_t e = cudaStreamWaitEvent(ctx->stream, ctx->ev_thr, 0);
    if (e != cudaSuccess) return fail(ctx, MM_E_CUDA, std::string("join_thresholds: ") + cudaGetErrorString(e));
    return MM_OK;
}

void resolve_pending(mm_ctx* ctx) {
    for (Pending& p : ctx->pending) {
        cudaEventSynchronize(p.b);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, p.a, p.b);
        KStat& k = ctx->kstats[p.name];
        ++k.launches;
        k.total_ms += ms;
        cudaEventDestroy(p.a);
        cudaEventDestroy(p.b);
    }
    ctx->pending.clear();
}

void free_model(mm_ctx* c) {
    for (DBuf<uint32_t>* b : {&c->method_owner, &c->attribute_owner, &c->cls_moff, &c->cls_methods, &c->cls_aoff,
                              &c->cls_attrs, &c->call_off, &c->call_tgt, &c->acc_off, &c->acc_tgt,
                              &c->large_list, &c->foreign, &c->cmaxdeg, &c->grows, &c->cbo, &c->ux,
                              &c->un, &c->nl_pos})
        b->release();
    c->cedge.release();
    c->groups.release();
    c->solo.release();
    c->pc_mem.release();
    c->pa_mem.release();
    c->recs.release();
    c->own_mask.release();
    c->attr_info.release();
    c->giant_items.release();
    c->mma_list.release();
    c->gcnt.release();
    c->gH.release();
    c->fan.release();
    c->sim_u32.release();
    c->sim_ctl.release();
    c->sim_out.release();
    c->sim_caller.release();
    c->simc_u32.release();
    c->simc_out.release();
    c->pos_owner.release();
    for (DBuf<uint32_t>* b : {&c->pc_off, &c->pc_tgt, &c->pa_off, &c->pa_tgt, &c->pos_scan}) b->release();
    c->cplan.release();
    c->big_list.release();
    c->plans.release();
    c->gkeys.release();
    c->dense.release();
    c->ck_items.release();
    c->split_list.release();
    c->rec.release();
    c->lcom.release();
    c->ck.release();
    c->have_model = c->metrics_valid = c->sweep_valid = false;
}

mm_status set_device(mm_ctx* ctx) {
    MM_CUDA(ctx, cudaSetDevice(ctx->device));
    return MM_OK;
}

template <class T>
mm_status upload_array(mm_ctx* ctx, DBuf<T>& d, const T* h, size_t n, const char* what) {
    if (n && !h) return fail(ctx, MM_E_ARG, std::string("mm_upload: NULL ") + what);
    MM_CUDA(ctx, d.ensure(n ? n : 1));
    if (n) MM_CUDA(ctx, cudaMemcpyAsync(d.p, h, n * sizeof(T), cudaMemcpyHostToDevice, ctx->stream));
    return MM_OK;
}

uint32_t next_pow2(uint32_t v) {
    uint32_t n = 1;
    while (n < v) n <<= 1;
    return n;
}

mm_status ensure_metrics(mm_ctx* ctx) {
    if (!ctx->have_model) return fail(ctx, MM_E_STATE, "no model uploaded");
    if (mm_status st = set_device(ctx)) return st;
    if (!ctx->metrics_valid) return mm_compute_metrics(ctx);
    return MM_OK;
}

}  // namespace

extern "C" {

int mm_abi_version(void) { return MMGPU_ABI_VERSION; }

int mm_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
    return n;
}

const char* mm_last_error(const mm_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

mm_status mm_ctx_create(int device, mm_ctx** out) {
    if (!out) return MM_E_ARG;
    *out = nullptr;
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) return MM_E_CUDA;
    if (device < 0 || device >= n) return MM_E_RANGE;
    mm_ctx* ctx = new (std::nothrow) mm_ctx();
    if (!ctx) return MM_E_OOM;
    ctx->device = device;
    if (cudaSetDevice(device) != cudaSuccess ||
        cudaStreamCreateWithFlags(&ctx->own, cudaStreamNonBlocking) != cudaSuccess ||
        // the side stream (threshold means beside the scoring kernel) at the
        // highest priority: its cluster launch must not wait for the scoring
        // kernel's blocks to drain
        cudaDeviceGetStreamPriorityRange(&ctx->prio_lo, &ctx->prio_hi) != cudaSuccess ||
        cudaStreamCreateWithPriority(&ctx->side, cudaStreamNonBlocking, ctx->prio_hi) != cudaSuccess ||
        cudaEventCreateWithFlags(&ctx->ev_metrics, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&ctx->ev_thr, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventRecord(ctx->ev_thr, ctx->side) != cudaSuccess ||
        cudaEventCreateWithFlags(&ctx->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&ctx->ev_fork0, cudaEventDisableTiming) != cudaSuccess ||
        ctx->ctl.alloc(1) != cudaSuccess || ctx->whatif.alloc(1) != cudaSuccess) {
        mm_ctx_destroy(ctx);
        return MM_E_CUDA;
    }
    for (int k = 0; k <= kMaxTiers + 2; ++k)
        if (cudaStreamCreateWithFlags(&ctx->aux[k], cudaStreamNonBlocking) != cudaSuccess ||
            cudaEventCreateWithFlags(&ctx->ev_join[k], cudaEventDisableTiming) != cudaSuccess) {
            mm_ctx_destroy(ctx);
            return MM_E_CUDA;
        }
    for (int k = 0; k < kUploadArrays; ++k)
        if (cudaEventCreateWithFlags(&ctx->ev_up[k], cudaEventDisableTiming) != cudaSuccess) {
            mm_ctx_destroy(ctx);
            return MM_E_CUDA;
        }
    if (cudaStreamCreateWithFlags(&ctx->d2h, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&ctx->ev_d2h_go, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&ctx->ev_d2h_done, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventRecord(ctx->ev_d2h_done, ctx->d2h) != cudaSuccess) {
        mm_ctx_destroy(ctx);
        return MM_E_CUDA;
    }
    ctx->stream = ctx->own;
    if (const char* v = std::getenv("MMGPU_HIST_MAX_BYTES")) ctx->hist_max_bytes = std::strtoull(v, nullptr, 10);
    if (const char* v = std::getenv("MMGPU_GIANT_MIN")) ctx->giant_min = std::strtoull(v, nullptr, 10);
    if (const char* v = std::getenv("MMGPU_CK_MMA_MIN")) ctx->ck_mma_min = std::strtoull(v, nullptr, 10);
    if (const char* v = std::getenv("MMGPU_THR_SIDE")) ctx->thr_side = v[0] != '0';
    if (const char* v = std::getenv("MMGPU_LEAN")) ctx->lean_fused = v[0] != '0';
    if (const char* v = std::getenv("MMGPU_SCORE_FAST")) ctx->score_fast = v[0] != '0';
    if (const char* v = std::getenv("MMGPU_GROUP")) ctx->group_on = v[0] != '0';
    *out = ctx;
    return MM_OK;
}

void mm_ctx_destroy(mm_ctx* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    cudaStreamSynchronize(ctx->side);
    if (ctx->d2h) cudaStreamSynchronize(ctx->d2h);
    resolve_pending(ctx);
    if (ctx->graph_exec) cudaGraphExecDestroy(ctx->graph_exec);
    for (Pending& p : ctx->graph_events) {
        cudaEventDestroy(p.a);
        cudaEventDestroy(p.b);
    }
    free_model(ctx);
    ctx->ctl.release();
    ctx->whatif.release();
    ctx->thr_scratch.release();
    ctx->tile_state.release();
    ctx->out.release();
    ctx->res.release();
    ctx->emit_list.release();
    ctx->wide_cnt.release();
    ctx->fallback.release();
    ctx->gate_lcom.release();
    ctx->gate_cbo.release();
    if (ctx->own) cudaStreamDestroy(ctx->own);
    if (ctx->side) cudaStreamDestroy(ctx->side);
    if (ctx->ev_metrics) cudaEventDestroy(ctx->ev_metrics);
    if (ctx->ev_thr) cudaEventDestroy(ctx->ev_thr);
    if (ctx->ev_fork) cudaEventDestroy(ctx->ev_fork);
    if (ctx->ev_fork0) cudaEventDestroy(ctx->ev_fork0);
    for (int k = 0; k <= kMaxTiers + 2; ++k) {
        if (ctx->aux[k]) cudaStreamDestroy(ctx->aux[k]);
        if (ctx->ev_join[k]) cudaEventDestroy(ctx->ev_join[k]);
    }
    for (int k = 0; k < kUploadArrays; ++k)
        if (ctx->ev_up[k]) cudaEventDestroy(ctx->ev_up[k]);
    if (ctx->d2h) cudaStreamDestroy(ctx->d2h);
    if (ctx->ev_d2h_go) cudaEventDestroy(ctx->ev_d2h_go);
    if (ctx->ev_d2h_done) cudaEventDestroy(ctx->ev_d2h_done);
    delete ctx;
}

mm_status mm_ctx_set_stream(mm_ctx* ctx, void* s) {
    if (!ctx) return MM_E_ARG;
    ctx->stream = s ? static_cast<cudaStream_t>(s) : ctx->own;
    return MM_OK;
}

mm_status mm_ctx_synchronize(mm_ctx* ctx) {
    if (!ctx) return MM_E_ARG;
    MM_CUDA(ctx, cudaStreamSynchronize(ctx->d2h));
    MM_CUDA(ctx, cudaStreamSynchronize(ctx->side));
    MM_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    return MM_OK;
}

mm_status mm_ctx_stream(mm_ctx* ctx, void** s) {
    if (!ctx || !s) return MM_E_ARG;
    *s = ctx->stream;
    return MM_OK;
}

mm_status mm_ctx_set_profiling(mm_ctx* ctx, int on) {
    if (!ctx) return MM_E_ARG;
    ctx->profiling = on != 0;
    return MM_OK;
}

mm_status mm_kernel_stats(mm_ctx* ctx, mm_kernel_stat* out, int cap, int* n_out) {
    if (!ctx || !n_out) return MM_E_ARG;
    resolve_pending(ctx);
    int i = 0;
    for (const auto& kv : ctx->kstats) {
        if (out && i < cap) {
            std::memset(&out[i], 0, sizeof out[i]);
            std::strncpy(out[i].name, kv.first.c_str(), sizeof(out[i].name) - 1);
            out[i].launches = kv.second.launches;
            out[i].total_ms = kv.second.total_ms;
        }
        ++i;
    }
    *n_out = i;
    return (out && cap < i) ? MM_E_CAPACITY : MM_OK;
}

mm_status mm_reset_kernel_stats(mm_ctx* ctx) {
    if (!ctx) return MM_E_ARG;
    resolve_pending(ctx);
    ctx->kstats.clear();
    return MM_OK;
}

uint64_t mm_system_bytes(const mm_system* s) {
    if (!s) return 0;
    const uint64_t Ec = s->call_off ? s->call_off[s->n_methods] : 0;
    const uint64_t Ea = s->acc_off ? s->acc_off[s->n_methods] : 0;
    return 4ull * ((s->method_owner ? 2ull : 1ull) * s->n_methods + (s->attribute_owner ? 2ull : 1ull) * s->n_attributes +
                   2ull * (s->n_classes + 1) + 2ull * (s->n_methods + 1) + Ec + Ea);
}

// MMGPU_UPLOAD_TRACE=1: per-phase times of mm_upload on stderr (events on the
// main stream + host clock); a diagnostic, off by default
struct UploadTrace {
    bool on = false;
    cudaStream_t st = nullptr;
    std::vector<cudaEvent_t> ev;
    std::vector<const char*> name;
    std::vector<std::pair<const char*, double>> host;
    std::chrono::steady_clock::time_point h0;
    void init(cudaStream_t s) {
        static const bool env = std::getenv("MMGPU_UPLOAD_TRACE") != nullptr;
        on = env;
        st = s;
        if (on) h0 = std::chrono::steady_clock::now();
    }
    void mark(const char* n) {
        if (!on) return;
        cudaEvent_t e;
        cudaEventCreate(&e);
        cudaEventRecord(e, st);
        ev.push_back(e);
        name.push_back(n);
    }
    void hmark(const char* n) {
        if (on) host.push_back({n, std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - h0).count()});
    }
    ~UploadTrace() {
        if (!on) return;
        cudaStreamSynchronize(st);
        std::fprintf(stderr, "[mm_upload trace] device (us since %s):", ev.empty() ? "-" : name[0]);
        for (size_t i = 1; i < ev.size(); ++i) {
            float ms = 0;
            cudaEventElapsedTime(&ms, ev[0], ev[i]);
            std::fprintf(stderr, " %s=%.1f", name[i], ms * 1e3);
        }
        std::fprintf(stderr, " | host (us since entry):");
        for (auto& h : host) std::fprintf(stderr, " %s=%.1f", h.first, h.second);
        std::fprintf(stderr, "\n");
        for (auto e : ev) cudaEventDestroy(e);
    }
};

mm_status mm_upload(mm_ctx* ctx, const mm_system* s) {
    if (!ctx || !s) return MM_E_ARG;
    if (mm_status st = set_device(ctx)) return st;
    UploadTrace tr;
    tr.init(ctx->stream);
    MM_CUDA(ctx, cudaStreamSynchronize(ctx->side));
    MM_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    // device buffers are reused across uploads (grown on demand, never shrunk)
    ctx->have_model = ctx->metrics_valid = ctx->sweep_valid = false;
    ctx->sim_valid = false;
    ctx->gates_set = false;
    ++ctx->layout_gen;
    if (!s->call_off || !s->acc_off || !s->class_method_off || !s->class_attr_off)
        return fail(ctx, MM_E_ARG, "mm_upload: NULL offsets");
    const uint32_t C = s->n_classes, M = s->n_methods, A = s->n_attributes;
    const uint64_t Ec = s->call_off[M], Ea = s->acc_off[M];
    ctx->C = C; ctx->M = M; ctx->A = A; ctx->Ec = Ec; ctx->Ea = Ea;
    ctx->h_cls_moff.assign(s->class_method_off, s->class_method_off + C + 1);

    // H2D copies on the main stream; each array's range validation runs on an
    // aux stream as soon as its copy lands, overlapping the next copies.
    // Offsets are checked against the host totals, ids against their id space.
    Ctl* ctl = ctx->ctl.p;
    uint32_t* bad = &ctl->bad;
    MM_CUDA(ctx, cudaMemsetAsync(ctl, 0, sizeof(Ctl), ctx->stream));
    tr.hmark("synced");
    tr.mark("start");
    cudaStream_t vs = ctx->aux[0];
    int n_up = 0;
    auto up = [&](DBuf<uint32_t>& d, const uint32_t* h, size_t n, const char* what, auto&& validate) -> mm_status {
        if (mm_status st = upload_array(ctx, d, h, n, what)) return st;
        MM_CUDA(ctx, cudaEventRecord(ctx->ev_up[n_up], ctx->stream));
        MM_CUDA(ctx, cudaStreamWaitEvent(vs, ctx->ev_up[n_up], 0));
        ++n_up;
        validate(d.p);
        MM_CUDA(ctx, cudaGetLastError());
        return MM_OK;
    };
    auto ids = [&](size_t n, uint32_t bound) { return [=](const uint32_t* p) { launch_validate_ids(p, n, bound, bad, vs); }; };
    auto offs = [&](size_t n1, uint32_t total) {
        return [=](const uint32_t* p) { launch_validate_offsets(p, n1, total, bad, vs); };
    };
    const bool derive_mo = !s->method_owner, derive_ao = !s->attribute_owner;
    // every buffer first: the expansion below captures pointers while later
    // arrays are still being copied
    MM_CUDA(ctx, ctx->method_owner.ensure(M ? M : 1));
    MM_CUDA(ctx, ctx->attribute_owner.ensure(A ? A : 1));
    MM_CUDA(ctx, ctx->call_off.ensure(M + 1ull));
    MM_CUDA(ctx, ctx->call_tgt.ensure(Ec ? Ec : 1));
    MM_CUDA(ctx, ctx->acc_off.ensure(M + 1ull));
    MM_CUDA(ctx, ctx->acc_tgt.ensure(Ea ? Ea : 1));
    MM_CUDA(ctx, ctx->pos_owner.ensure(M ? M : 1));
    MM_CUDA(ctx, ctx->attr_info.ensure(A ? A : 1));
    // expansion of the membership lists, on the validation stream as soon as
    // the lists (and any owner tables) are in, under the remaining copies: the
    // class-order owner table, the attribute (owner, rank) table and — when
    // the caller left them out — the owner tables (the validate()
    // precondition makes them equal; unowned ids stay kNone and fail the
    // range check)
    auto expand = [&]() -> mm_status {
        return run_on(ctx, vs, "expand", [&] {
            launch_expand(ctx->dev(), derive_mo ? ctx->method_owner.p : nullptr,
                          derive_ao ? ctx->attribute_owner.p : nullptr, ctx->pos_owner.p, ctx->attr_info.p, vs);
            if (derive_mo) launch_validate_ids(ctx->method_owner.p, M, C, bad, vs);
            if (derive_ao) launch_validate_ids(ctx->attribute_owner.p, A, C, bad, vs);
        });
    };
    mm_status st = MM_OK;
    if ((st = up(ctx->cls_moff, s->class_method_off, C + 1ull, "class_method_off", offs(C + 1ull, M))) ||
        (st = up(ctx->cls_methods, s->class_methods, M, "class_methods", ids(M, M))) ||
        (st = up(ctx->cls_aoff, s->class_attr_off, C + 1ull, "class_attr_off", offs(C + 1ull, A))) ||
        (st = up(ctx->cls_attrs, s->class_attrs, A, "class_attrs", ids(A, A))) ||
        (!derive_mo && (st = up(ctx->method_owner, s->method_owner, M, "method_owner", ids(M, C)))) ||
        (!derive_ao && (st = up(ctx->attribute_owner, s->attribute_owner, A, "attribute_owner", ids(A, C)))) ||
        (st = expand()) ||
        (st = up(ctx->call_off, s->call_off, M + 1ull, "call_off", offs(M + 1ull, (uint32_t)Ec))) ||
        (st = up(ctx->call_tgt, s->call_tgt, Ec, "call_tgt", ids(Ec, M))) ||
        (st = up(ctx->acc_off, s->acc_off, M + 1ull, "acc_off", offs(M + 1ull, (uint32_t)Ea))) ||
        (st = up(ctx->acc_tgt, s->acc_tgt, Ea, "acc_tgt", ids(Ea, A))))
        return st;
    tr.mark("copies");
    tr.hmark("copies_issued");
    MM_CUDA(ctx, cudaEventRecord(ctx->ev_join[0], vs));
    MM_CUDA(ctx, cudaStreamWaitEvent(ctx->stream, ctx->ev_join[0], 0));
    tr.mark("validated");
    // the dependency rows in class order (the method pass streams them)
    MM_CUDA(ctx, ctx->pc_off.ensure(M + 1ull));
    MM_CUDA(ctx, ctx->pa_off.ensure(M + 1ull));
    MM_CUDA(ctx, ctx->pc_tgt.ensure(Ec ? Ec : 1));
    MM_CUDA(ctx, ctx->pa_tgt.ensure(Ea ? Ea : 1));
    MM_CUDA(ctx, ctx->pos_scan.ensure(2ull * ((M + 255ull) / 256) + 2));  // per-tile degree sums (pc, pa)
    MM_CUDA(ctx, ctx->pc_mem.ensure(Ec ? Ec : 1));
    MM_CUDA(ctx, ctx->pa_mem.ensure(Ea ? Ea : 1));
    MM_CUDA(ctx, ctx->foreign.ensure(C ? C : 1));
    MM_CUDA(ctx, ctx->cmaxdeg.ensure(C ? C : 1));
    st = run(ctx, "upload_rows", [&] {
        launch_pos_rows(ctx->dev(), ctx->pos_owner.p, ctx->pc_off.p, ctx->pc_tgt.p, ctx->pa_off.p, ctx->pa_tgt.p,
                        ctx->pc_mem.p, ctx->pa_mem.p, ctx->pos_scan.p, ctx->foreign.p, ctx->cmaxdeg.p, &ctl->n_hideg, ctx->stream);
    });
    if (st) return st;
    tr.mark("pos_rows");

    // class plan (bounds-checked, so it is safe on a model validation rejects):
    // warp path vs CTA path, scratch for the CTA path. One sync for both.
    MM_CUDA(ctx, ctx->cplan.ensure(C ? C : 1));
    MM_CUDA(ctx, ctx->cedge.ensure(C ? C : 1));
    MM_CUDA(ctx, ctx->big_list.ensure(C ? C : 1));
    MM_CUDA(ctx, ctx->large_list.ensure(C ? C : 1));
    const DevModel dm = ctx->dev();
    st = run(ctx, "plan", [&] {
        launch_plan_classes(dm, ctx->cplan.p, ctx->cedge.p, ctx->large_list.p, &ctl->n_large, ctx->big_list.p,
                            &ctl->n_big, &ctl->max_deg, ctx->foreign.p, ctx->cmaxdeg.p, ctx->stream);
    });
    if (st) return st;
    const bool grouping = ctx->lean_fused && ctx->group_on;
    if (ctx->lean_fused) {  // k_method's position list (classes that are not lean)
        MM_CUDA(ctx, ctx->nl_pos.ensure(M ? M : 1));
        st = run(ctx, "plan_nl", [&] {
            launch_nl_positions(ctx->pos_owner.p, ctx->cplan.p, M, ctx->nl_pos.p, &ctl->n_nl, ctx->stream);
        });
        if (st) return st;
    }
    if (grouping) {
        MM_CUDA(ctx, ctx->groups.ensure(C ? C : 1));
        MM_CUDA(ctx, ctx->solo.ensure(C ? C : 1));
        st = run(ctx, "plan_groups", [&] {
            launch_plan_groups(ctx->cplan.p, ctx->foreign.p, ctx->cmaxdeg.p, C, ctx->groups.p, &ctl->n_groups,
                               ctx->solo.p, &ctl->n_solo, ctx->stream);
        });
        if (st) return st;
    }
    tr.mark("plans");
    Ctl h{};
    MM_CUDA(ctx, cudaMemcpyAsync(&h, ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, ctx->stream));
    MM_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    tr.hmark("ctl_synced");
    if (h.bad) return fail(ctx, MM_E_ARG, (h.bad & 2u) ? "mm_upload: malformed offsets" : "mm_upload: id out of range");
    ctx->n_large = h.n_large;
    ctx->n_big = h.n_big;
    ctx->max_deg = h.max_deg;
    ctx->n_groups = grouping ? h.n_groups : 0;
    ctx->n_solo = grouping ? h.n_solo : 0;
    // lean classes take the fused method + class kernel; k_method then runs
    // only over the other classes' positions (a list, when there are both)
    ctx->n_lean = ctx->lean_fused ? C - h.n_large - h.n_big : 0;
    ctx->n_nl = ctx->lean_fused ? h.n_nl : 0;
    // methods k_score_fast may hand to the per-thread kernel: more edges
    // than a record's entries, or (class ids ≥ 2^24) any
    ctx->n_maybe_ovf = C >= (1u << 24) ? M : h.n_hideg;
    if (ctx->n_large) {
        MM_CUDA(ctx, ctx->hs_list.ensure(ctx->n_large));
        MM_CUDA(ctx, ctx->hs_fr.ensure(C));
        MM_CUDA(ctx, cudaMemcpyAsync(ctx->hs_list.p, ctx->large_list.p, 4ull * ctx->n_large, cudaMemcpyDeviceToHost,
                                     ctx->stream));
        MM_CUDA(ctx, cudaMemcpyAsync(ctx->hs_fr.p, ctx->foreign.p, 4ull * C, cudaMemcpyDeviceToHost, ctx->stream));
        MM_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
        tr.hmark("lists_d2h");
        // the list in class order (the device appends it in atomic order): a
        // pass over a class bitmap, O(C), instead of a comparison sort
        std::vector<uint32_t> list(ctx->n_large);
        {
            std::vector<uint8_t> mark(C, 0);
            for (uint32_t i = 0; i < ctx->n_large; ++i)
                if (ctx->hs_list.p[i] < C) mark[ctx->hs_list.p[i]] = 1;
            uint32_t k = 0;
            for (uint32_t c = 0; c < C && k < ctx->n_large; ++c)
                if (mark[c]) list[k++] = c;
            if (k != ctx->n_large) return fail(ctx, MM_E_ARG, "mm_upload: malformed class plan");
        }
        const uint32_t* fr = ctx->hs_fr.p;
        int dev_smem = 0;
        cudaDeviceGetAttribute(&dev_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, ctx->device);
        const uint64_t budget = dev_smem > 8192 ? (uint64_t)dev_smem - 8192 : 40 * 1024;
        std::vector<LargePlan> plans(ctx->n_large);
        std::vector<uint64_t> need(ctx->n_large);
        uint64_t n_dense = 0;
        for (uint32_t i = 0; i < ctx->n_large; ++i) {
            const uint32_t c = list[i];
            const uint64_t Mc = s->class_method_off[c + 1] - s->class_method_off[c];
            const uint64_t Ac = s->class_attr_off[c + 1] - s->class_attr_off[c];
            LargePlan& pl = plans[i];
            std::memset(&pl, 0, sizeof pl);
            pl.keys_cap = next_pow2(std::max<uint32_t>(fr[c], 1));
            n_dense += fr[c] > kDenseRowMin;
            // shared memory, in order of benefit: the class histogram or the keys
            // (sorted in place), then the LCOM-CK structure
            uint64_t used = 0;
            const uint64_t kbytes = (4ull * pl.keys_cap + 15) & ~15ull;
            const uint64_t hbytes = (4ull * C + 15) & ~15ull;
            if (hbytes <= ctx->hist_max_bytes && C <= 16ull * pl.keys_cap) {
                // few classes, many keys: an smem histogram over all C replaces sorting
                pl.hist = 1;
                pl.keys_cap = 0;
                used += hbytes;
            } else if (kbytes <= budget) {
                pl.keys_in_smem = 1;
                used += kbytes;
            }
            const uint64_t WA = (Ac + 63) / 64;
            const uint64_t mbytes = 8 * Mc * WA;
            pl.pre_slot = kNoSlot;
            if (WA <= 4 && used + mbytes <= budget) {
                pl.ck_masks = 1;
                used += mbytes;
                // A ≤ 64: the method pass's masks are complete, B·Bᵀ on the tensor cores
                pl.ck_mma = WA == 1 && Mc >= ctx->ck_mma_min && Mc <= kCkMmaMaxMembers;
            }
            else if (pl.hist && Mc >= ctx->giant_min) {
                // giant: phase 1 over many CTAs (k_giant_p1) into a global histogram;
                // its attribute bitmaps live in global scratch (split LCOM-CK)
                pl.pre_slot = 0;
            } else {
                const uint64_t rbytes = 4 * Ac * ((Mc + 31) / 32);
                if (used + rbytes <= budget) { pl.rows_in_smem = 1; used += rbytes; }
            }
            need[i] = used;
        }
        // launch groups by shared-memory tier and CTA size, so small CTAs are not
        // held to one per SM by a giant and giants get 1024 threads
        static const uint64_t tiers[] = {16 * 1024, 48 * 1024, 100 * 1024, ~0ull};
        std::vector<int> gkey(ctx->n_large);
        for (uint32_t i = 0; i < ctx->n_large; ++i) {
            const uint32_t c = list[i];
            const uint64_t Mc = s->class_method_off[c + 1] - s->class_method_off[c];
            int tier = 0;
            while (need[i] > tiers[tier]) ++tier;
            gkey[i] = 2 * tier + ((tier >= 3 || Mc >= kBigCtaMembers) ? 1 : 0);
        }
        // stable counting sort by group key (class order within a group)
        std::vector<uint32_t> order(ctx->n_large);
        {
            uint32_t start[2 * 4 + 1] = {};
            for (uint32_t i = 0; i < ctx->n_large; ++i) ++start[gkey[i] + 1];
            for (int g = 0; g < 2 * 4; ++g) start[g + 1] += start[g];
            for (uint32_t i = 0; i < ctx->n_large; ++i) order[start[gkey[i]]++] = i;
        }
        std::vector<uint32_t> list2(ctx->n_large);
        std::vector<LargePlan> plans2(ctx->n_large);
        uint64_t koff = 0, roff = 0;
        ctx->large_groups.clear();
        for (uint32_t j = 0; j < ctx->n_large; ++j) {
            const uint32_t i = order[j];
            list2[j] = list[i];
            plans2[j] = plans[i];
            LargePlan& pl = plans2[j];
            if (!pl.keys_in_smem) { pl.keys_off = koff; koff += pl.keys_cap; }
            const uint32_t c = list[i];
            const uint64_t Mc = s->class_method_off[c + 1] - s->class_method_off[c];
            const uint64_t Ac = s->class_attr_off[c + 1] - s->class_attr_off[c];
            if (!pl.ck_masks && !pl.rows_in_smem) { pl.rows_off = roff; roff += Ac * ((Mc + 31) / 32); }
            const uint32_t smem = (uint32_t)std::max<uint64_t>(16, (need[i] + 15) & ~15ull);
            if (ctx->large_groups.empty() || ctx->large_groups.back().key != gkey[i])
                ctx->large_groups.push_back({j, 0, smem, gkey[i], (gkey[i] & 1) ? 1024u : 256u, 0, 0, 0, 0, 0, 0});
            auto& g = ctx->large_groups.back();
            ++g.count;
            g.smem = std::max(g.smem, smem);
        }
        // classes whose attribute bitmaps live in global scratch: LCOM-CK split over kCkChunk-member chunks
        std::vector<uint2> items;
        std::vector<uint32_t> split;
        std::vector<uint2> gitems;  // giants: (index into the large list, first member) per k_giant_p1 CTA
        uint32_t n_giant = 0;
        for (auto& g : ctx->large_groups) {  // per group: its split classes' work follows it on its stream
            g.item_first = (uint32_t)items.size();
            g.split_first = (uint32_t)split.size();
            g.giant_first = (uint32_t)gitems.size();
            for (uint32_t j = g.first; j < g.first + g.count; ++j) {
                LargePlan& pl = plans2[j];
                if (pl.pre_slot == kNoSlot) continue;
                pl.pre_slot = n_giant++;
                const uint32_t c = list2[j];
                const uint32_t Mc = s->class_method_off[c + 1] - s->class_method_off[c];
                for (uint32_t b = 0; b < Mc; b += kGiantChunk) gitems.push_back(make_uint2(j, b));
            }
            g.n_giant_items = (uint32_t)gitems.size() - g.giant_first;
            for (uint32_t j = g.first; j < g.first + g.count; ++j) {
                const LargePlan& pl = plans2[j];
                if (pl.ck_masks || pl.rows_in_smem) continue;
                const uint32_t c = list2[j];
                const uint32_t Mc = s->class_method_off[c + 1] - s->class_method_off[c];
                split.push_back(c);
                for (uint32_t b = 0; b < Mc; b += kCkChunk) items.push_back(make_uint2(j, b));
            }
            g.n_items = (uint32_t)items.size() - g.item_first;
            g.n_split = (uint32_t)split.size() - g.split_first;
        }
        ctx->n_ck_items = (uint32_t)items.size();
        ctx->n_split = (uint32_t)split.size();
        ctx->n_giant = n_giant;
        MM_CUDA(ctx, ctx->giant_items.ensure(gitems.size() ? gitems.size() : 1));
        MM_CUDA(ctx, ctx->gcnt.ensure(n_giant ? (size_t)n_giant * C : 1));
        MM_CUDA(ctx, ctx->gH.ensure(n_giant ? n_giant : 1));
        tr.hmark("host_plan");
        // every host-built table travels in one pinned staging block, asynchronously
        struct Part { void* dst; const void* src; size_t bytes; };
        std::vector<Part> parts;
        auto stage = [&](void* dst, const void* src, size_t bytes) { if (bytes) parts.push_back({dst, src, bytes}); };
        stage(ctx->giant_items.p, gitems.data(), sizeof(uint2) * gitems.size());
        MM_CUDA(ctx, ctx->ck_items.ensure(items.size() ? items.size() : 1));
        MM_CUDA(ctx, ctx->split_list.ensure(split.size() ? split.size() : 1));
        stage(ctx->ck_items.p, items.data(), sizeof(uint2) * items.size());
        stage(ctx->split_list.p, split.data(), 4 * split.size());
        stage(ctx->large_list.p, list2.data(), 4ull * ctx->n_large);
        std::vector<uint32_t> mma;
        uint32_t mma_max = 0;
        for (uint32_t j = 0; j < ctx->n_large; ++j)
            if (plans2[j].ck_mma) {
                mma.push_back(list2[j]);
                mma_max = std::max<uint32_t>(mma_max, s->class_method_off[list2[j] + 1] - s->class_method_off[list2[j]]);
            }
        ctx->n_mma = (uint32_t)mma.size();
        MM_CUDA(ctx, ctx->mma_list.ensure(mma.size() ? mma.size() : 1));
        if (!mma.empty()) {
            stage(ctx->mma_list.p, mma.data(), 4 * mma.size());
            ctx->mma_smem = ck_mma_smem_bytes(mma_max);
            MM_CUDA(ctx, set_ck_mma_smem(ctx->mma_smem));
        }
        MM_CUDA(ctx, ctx->plans.ensure(ctx->n_large));
        stage(ctx->plans.p, plans2.data(), sizeof(LargePlan) * ctx->n_large);
        size_t total = 0;
        for (const Part& q : parts) total += (q.bytes + 15) & ~size_t(15);
        MM_CUDA(ctx, ctx->hs_up.ensure(total));
        size_t at = 0;
        for (const Part& q : parts) {
            std::memcpy(ctx->hs_up.p + at, q.src, q.bytes);
            MM_CUDA(ctx, cudaMemcpyAsync(q.dst, ctx->hs_up.p + at, q.bytes, cudaMemcpyHostToDevice, ctx->stream));
            at += (q.bytes + 15) & ~size_t(15);
        }
        tr.hmark("plans_h2d");
        MM_CUDA(ctx, ctx->gkeys.ensure(koff ? koff : 1));
        MM_CUDA(ctx, ctx->grows.ensure(roff ? roff : 1));
        ctx->grows_words = roff;
        uint32_t max_smem = 0;
        for (const auto& g : ctx->large_groups) max_smem = std::max(max_smem, g.smem);
        MM_CUDA(ctx, set_class_large_smem(max_smem));
        // exact bitmaps for dense U rows: ≤ one per CTA-path class with > kDenseRowMin
        // foreign keys, capped at 256 MB (classes past the cap keep Bloom + scan)
        const uint64_t words = 2ull * ((C + 31) / 32) * n_dense;  // membership + singletons
        ctx->dense_cap = (uint32_t)std::min<uint64_t>(words, 64ull << 20);
        MM_CUDA(ctx, ctx->dense.ensure(ctx->dense_cap ? ctx->dense_cap : 1));
    } else {
        ctx->large_groups.clear();
        ctx->dense_cap = 0;
        ctx->n_ck_items = ctx->n_split = 0;
        ctx->n_giant = 0;
        ctx->n_mma = 0;
        ctx->grows_words = 0;
    }
    // derived tables
    // M 32-byte records, then their M 32-bit headers (rec_hdrs)
    MM_CUDA(ctx, ctx->recs.ensure(M ? M + (M + 7) / 8 : 1));
    MM_CUDA(ctx, ctx->own_mask.ensure(M ? M : 1));
    MM_CUDA(ctx, ctx->rec.ensure(C ? C : 1));
    MM_CUDA(ctx, ctx->lcom.ensure(C ? C : 1));
    MM_CUDA(ctx, ctx->ck.ensure(C ? C : 1));
    MM_CUDA(ctx, ctx->cbo.ensure(C ? C : 1));
    MM_CUDA(ctx, ctx->thr_scratch.ensure(thresholds_scratch_bytes(C)));
    // U rows: kSmallRowCap slots per member for the warp-path classes (static
    // placement), then the CTA-path classes (bounded by their foreign edges)
    if ((uint64_t)kSmallRowCap * M + Ec + Ea + 1 >= (1ull << 32))
        return fail(ctx, MM_E_RANGE, "mm_upload: system too large for 32-bit U-row offsets");
    MM_CUDA(ctx, ctx->ux.ensure((size_t)kSmallRowCap * M + Ec + Ea + 1));
    MM_CUDA(ctx, ctx->un.ensure((size_t)kSmallRowCap * M + Ec + Ea + 1));
    tr.hmark("done");
    tr.mark("end");
    ctx->have_model = true;
    ctx->metrics_valid = false;
    ctx->sweep_valid = false;
    return MM_OK;
}

mm_status mm_compute_metrics(mm_ctx* ctx) {
    if (!ctx) return MM_E_ARG;
    if (!ctx->have_model) return fail(ctx, MM_E_STATE, "mm_compute_metrics: no model uploaded");
    if (mm_status st = set_device(ctx)) return st;
    Ctl* ctl = ctx->ctl.p;
    MM_CUDA(ctx, cudaStreamWaitEvent(ctx->stream, ctx->ev_d2h_done, 0));  // async copies of the last results
    MM_CUDA(ctx, cudaMemsetAsync(&ctl->ucursor, 0, 2 * sizeof(uint32_t), ctx->stream));  // ucursor, dense_cursor
    const DevModel dm = ctx->dev();
    // lean classes: one fused kernel (no k_method records needed), on its own
    // stream when other classes need the method pass, else on the main stream
    const bool lean = ctx->n_lean > 0, others = ctx->n_lean < ctx->C;
    cudaStream_t ls = others ? ctx->aux[kMaxTiers + 2] : ctx->stream;
    mm_status st = MM_OK;
    if (lean) {
        if (others) {
            MM_CUDA(ctx, cudaEventRecord(ctx->ev_fork0, ctx->stream));
            MM_CUDA(ctx, cudaStreamWaitEvent(ls, ctx->ev_fork0, 0));
        }
        const bool grouped = ctx->lean_fused && ctx->group_on;
        if (grouped) {
            st = run_on(ctx, ls, "class_group", [&] {
                launch_class_group(dm, ctx->cplan.p, ctx->groups.p, ctx->n_groups, ctx->pos_owner.p, ctx->recs.p,
                                   ctx->rec.p, ctx->lcom.p, ctx->ck.p, ctx->cbo.p, ctx->ux.p, ctx->un.p, ls);
            });
            if (st) return st;
        }
        if (!grouped || ctx->n_solo) {
            st = run_on(ctx, ls, "class_lean", [&] {
                launch_class_lean(dm, ctx->cplan.p, ctx->cedge.p, ctx->pc_mem.p, ctx->pa_mem.p, ctx->recs.p,
                                  ctx->rec.p, ctx->lcom.p, ctx->ck.p, ctx->cbo.p, ctx->ux.p, ctx->un.p,
                                  grouped ? ctx->solo.p : nullptr, ctx->n_solo, ls);
            });
            if (st) return st;
        }
        if (others) MM_CUDA(ctx, cudaEventRecord(ctx->ev_join[kMaxTiers + 2], ls));
    }
    if (others) {
        st = run(ctx, "method", [&] {
            launch_method(dm, ctx->recs.p, ctx->own_mask.p, ctx->pos_owner.p, ctx->max_deg,
                          lean ? ctx->nl_pos.p : nullptr, ctx->n_nl, ctx->stream);
        });
        if (st) return st;
    }
    // class pass: the CTA-path tiers fork onto their own streams (longest
    // tier first) and overlap each other and the warp path on the main stream
    st = run(ctx, "class_pass", [&] {
        if (ctx->grows_words) MM_CUDA(ctx, cudaMemsetAsync(ctx->grows.p, 0, 4ull * ctx->grows_words, ctx->stream));
        if (ctx->n_giant) {
            MM_CUDA(ctx, cudaMemsetAsync(ctx->gcnt.p, 0, 4ull * ctx->n_giant * ctx->C, ctx->stream));
            MM_CUDA(ctx, cudaMemsetAsync(ctx->gH.p, 0, 8ull * ctx->n_giant, ctx->stream));
        }
        const size_t ng = ctx->large_groups.size();
        if (ng) MM_CUDA(ctx, cudaEventRecord(ctx->ev_fork, ctx->stream));
        for (size_t k = 0; k < ng; ++k) {
            const auto& g = ctx->large_groups[ng - 1 - k];
            cudaStream_t as = ctx->aux[k];
            MM_CUDA(ctx, cudaStreamWaitEvent(as, ctx->ev_fork, 0));
            if (g.n_giant_items)
                if (mm_status e = run_on(ctx, as, "giant_p1", [&] {
                        launch_giant_p1(dm, ctx->large_list.p, ctx->plans.p, ctx->giant_items.p + g.giant_first,
                                        g.n_giant_items, ctx->recs.p, ctx->gcnt.p, ctx->gH.p, ctx->grows.p, as);
                    }))
                    return e;
            if (mm_status e = run_on(ctx, as, "class_large", [&] {
                    launch_class_large(dm, g.count, ctx->large_list.p + g.first, ctx->plans.p + g.first, g.smem,
                                       ctx->recs.p, ctx->own_mask.p, ctx->rec.p, ctx->lcom.p, ctx->ck.p, ctx->cbo.p,
                                       ctx->ux.p, ctx->un.p, &ctl->ucursor, ctx->gkeys.p, ctx->grows.p,
                                       ctx->dense_cap ? ctx->dense.p : nullptr, ctx->dense_cap, &ctl->dense_cursor,
                                       ctx->gcnt.p, ctx->gH.p, g.threads, as);
                }))
                return e;
            if (g.n_items)
                if (mm_status e = run_on(ctx, as, "ck_rows", [&] {
                        launch_ck_rows(dm, ctx->large_list.p, ctx->plans.p, ctx->ck_items.p + g.item_first,
                                       g.n_items, ctx->grows.p, ctx->split_list.p + g.split_first, g.n_split,
                                       ctx->ck.p, as);
                    }))
                    return e;
            MM_CUDA(ctx, cudaEventRecord(ctx->ev_join[k], as));
        }
        // warp-path classes with > 32 U-row keys: their own stream too
        cudaStream_t bs = ctx->aux[kMaxTiers];
        if ((ctx->n_big || ctx->n_mma) && !ng) MM_CUDA(ctx, cudaEventRecord(ctx->ev_fork, ctx->stream));
        if (ctx->n_big) MM_CUDA(ctx, cudaStreamWaitEvent(bs, ctx->ev_fork, 0));
        // tensor-core LCOM-CK of the dense classes: needs only the method pass
        cudaStream_t ms = ctx->aux[kMaxTiers + 1];
        if (ctx->n_mma) {
            MM_CUDA(ctx, cudaStreamWaitEvent(ms, ctx->ev_fork, 0));
            if (mm_status e = run_on(ctx, ms, "ck_mma", [&] {
                    launch_ck_mma(dm, ctx->mma_list.p, ctx->n_mma, ctx->mma_smem, ctx->own_mask.p, ctx->ck.p, ms);
                }))
                return e;
            MM_CUDA(ctx, cudaEventRecord(ctx->ev_join[kMaxTiers + 1], ms));
        }
        if (mm_status e = run(ctx, "class_small", [&] {
                launch_class_small(dm, ctx->cplan.p, ctx->big_list.p, ctx->n_big, ctx->recs.p, ctx->own_mask.p,
                                   ctx->rec.p, ctx->lcom.p, ctx->ck.p, ctx->cbo.p, ctx->ux.p, ctx->un.p, !lean,
                                   ctx->stream, bs);
            }))
            return e;
        if (ctx->n_big) {
            MM_CUDA(ctx, cudaEventRecord(ctx->ev_join[kMaxTiers], bs));
            MM_CUDA(ctx, cudaStreamWaitEvent(ctx->stream, ctx->ev_join[kMaxTiers], 0));
        }
        if (ctx->n_mma) MM_CUDA(ctx, cudaStreamWaitEvent(ctx->stream, ctx->ev_join[kMaxTiers + 1], 0));
        for (size_t k = 0; k < ng; ++k) MM_CUDA(ctx, cudaStreamWaitEvent(ctx->stream, ctx->ev_join[k], 0));
        if (lean && others) MM_CUDA(ctx, cudaStreamWaitEvent(ctx->stream, ctx->ev_join[kMaxTiers + 2], 0));
        return MM_OK;
    });
    if (st) return st;
    // threshold means: on the main stream, ahead of the sweep (the cluster
    // kernel takes 8 SMs for a few µs; launched beside the scoring kernel it
    // could not be placed until whole SMs drained). MMGPU_THR_SIDE=1: on the
    // side stream, overlapping the scoring (only the emission pass waits).
    cudaStream_t ts = ctx->thr_side ? ctx->side : ctx->stream;
    if (ctx->thr_side) {
        MM_CUDA(ctx, cudaEventRecord(ctx->ev_metrics, ctx->stream));
        MM_CUDA(ctx, cudaStreamWaitEvent(ctx->side, ctx->ev_metrics, 0));
    }
    cudaError_t te = cudaSuccess;
    st = run_on(ctx, ts, "thresholds", [&] {
        te = launch_thresholds(ctx->lcom.p, ctx->cbo.p, ctx->C, &ctl->thr, ctx->thr_scratch.p, ctx->thr_scratch.n, ts);
    });
    if (st) return st;
    if (te != cudaSuccess) return cuda_fail(ctx, te, "thresholds");
    MM_CUDA(ctx, cudaEventRecord(ctx->ev_thr, ts));
    ctx->metrics_valid = true;
    ctx->sweep_valid = false;
    return MM_OK;
}


mm_status mm_class_metrics(mm_ctx* ctx, double* lcom, uint64_t* lcom_ck, uint32_t* cbo) {
    if (!ctx) return MM_E_ARG;
    if (mm_status st = ensure_metrics(ctx)) return st;
    const size_t C = ctx->C;
    if (C && lcom) MM_CUDA(ctx, cudaMemcpyAsync(lcom, ctx->lcom.p, 8 * C, cudaMemcpyDeviceToHost, ctx->stream));
    if (C && lcom_ck) MM_CUDA(ctx, cudaMemcpyAsync(lcom_ck, ctx->ck.p, 8 * C, cudaMemcpyDeviceToHost, ctx->stream));
    if (C && cbo) MM_CUDA(ctx, cudaMemcpyAsync(cbo, ctx->cbo.p, 4 * C, cudaMemcpyDeviceToHost, ctx->stream));
    MM_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    return MM_OK;
}

mm_status mm_fan_metrics(mm_ctx* ctx, uint32_t* fan_in, uint32_t* fan_out) {
    if (!ctx) return MM_E_ARG;
    if (!ctx->have_model) return fail(ctx, MM_E_STATE, "mm_fan_metrics: no model uploaded");
    if (mm_status st = set_device(ctx)) return st;
    const size_t M = ctx->M;
    if (!M) return MM_OK;
    MM_CUDA(ctx, ctx->fan.ensure(2 * M));
    mm_status st = run(ctx, "fan", [&] {
        launch_fan(ctx->dev(), fan_in ? ctx->fan.p : nullptr, fan_out ? ctx->fan.p + M : nullptr, nullptr,
                   ctx->stream);
    });
    if (st) return st;
    if (fan_in) MM_CUDA(ctx, cudaMemcpyAsync(fan_in, ctx->fan.p, 4 * M, cudaMemcpyDeviceToHost, ctx->stream));
    if (fan_out) MM_CUDA(ctx, cudaMemcpyAsync(fan_out, ctx->fan.p + M, 4 * M, cudaMemcpyDeviceToHost, ctx->stream));
    MM_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    return MM_OK;
}

static mm_status compute_similarities(mm_ctx* ctx) {
    const uint64_t M = ctx->M, A = ctx->A, Ec = ctx->Ec, Ea = ctx->Ea;
    const uint64_t mx = std::max(M, A) + 1;
    const uint64_t nb = (mx + 1023) / 1024 + 1;
    // layout of the u32 scratch
    const uint64_t o_ucoff = 0, o_uc = o_ucoff + M + 1, o_uaoff = o_uc + (Ec ? Ec : 1), o_ua = o_uaoff + A + 1,
                   o_cur = o_ua + (Ea ? Ea : 1), o_tot = o_cur + mx, o_cnt = o_tot + nb, o_off = o_cnt + M + 1,
                   o_wide = o_off + M + 1, o_huge = o_wide + M + 1, o_end = o_huge + M + 1;
    MM_CUDA(ctx, ctx->sim_u32.ensure(o_end));
    MM_CUDA(ctx, ctx->sim_ctl.ensure(4 + M + 1));  // control words, then the huge rows' candidate counts
    uint32_t* u = ctx->sim_u32.p;
    unsigned long long* ctl = ctx->sim_ctl.p;
    uint32_t* small = reinterpret_cast<uint32_t*>(ctl + 1);  // n_wide, err, grand, n_huge
    unsigned long long* huge_tot = ctl + 4;
    MM_CUDA(ctx, cudaMemsetAsync(ctl, 0, 4 * sizeof(unsigned long long), ctx->stream));
    const DevModel dm = ctx->dev();
    mm_status st = run(ctx, "similarity", [&] {
        launch_similarity_index(dm, Ec, Ea, u + o_ucoff, u + o_uc, u + o_uaoff, u + o_ua, u + o_cur, u + o_tot,
                                small + 2, ctx->stream);
        launch_similarity_rows(dm, 0, u + o_ucoff, u + o_uc, u + o_uaoff, u + o_ua, u + o_cnt, nullptr, nullptr,
                               u + o_wide, small, small + 1, ctl, u + o_huge, huge_tot, small + 3, ctx->stream);
    });
    if (st) return st;
    unsigned long long h[3] = {0, 0, 0};
    MM_CUDA(ctx, cudaMemcpyAsync(h, ctl, sizeof h, cudaMemcpyDeviceToHost, ctx->stream));
    MM_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    // rows beyond the warp buffers: in batches through global scratch (any length)
    const uint32_t n_huge = static_cast<uint32_t>(h[2] >> 32);
    std::vector<uint32_t> hrows(n_huge);
    std::vector<unsigned long long> htot(n_huge);
    struct Batch { uint32_t first, count; uint64_t items; };
    std::vector<Batch> batches;
    DBuf<uint32_t> hseg, hkeys, hsorted;
    DBuf<char> htemp;
    if (n_huge) {
        MM_CUDA(ctx, cudaMemcpy(hrows.data(), u + o_huge, 4ull * n_huge, cudaMemcpyDeviceToHost));
        MM_CUDA(ctx, cudaMemcpy(htot.data(), huge_tot, 8ull * n_huge, cudaMemcpyDeviceToHost));
        const uint64_t kBatchItems = 64ull << 20;  // 256 MB of keys per batch (a longer row gets its own)
        uint64_t max_items = 0;
        for (uint32_t k = 0; k < n_huge;) {
            Batch b{k, 0, 0};
            while (k < n_huge && (b.count == 0 || b.items + htot[k] <= kBatchItems)) b.items += htot[k++], ++b.count;
            if (b.items >= (1ull << 31)) return fail(ctx, MM_E_UNSUPPORTED, "mm_similarities: one method's candidate "
                                                                             "list exceeds 2^31 entries");
            max_items = std::max(max_items, b.items);
            batches.push_back(b);
        }
        MM_CUDA(ctx, hseg.alloc(n_huge + batches.size()));
        MM_CUDA(ctx, hkeys.alloc(max_items ? max_items : 1));
        MM_CUDA(ctx, hsorted.alloc(max_items ? max_items : 1));
        MM_CUDA(ctx, htemp.alloc(std::max<size_t>(1, similarity_huge_temp_bytes((uint32_t)max_items, n_huge))));
        std::vector<uint32_t> seg;
        seg.reserve(n_huge + batches.size());
        for (const Batch& b : batches) {
            uint64_t acc = 0;
            for (uint32_t k = b.first; k < b.first + b.count; ++k) {
                seg.push_back((uint32_t)acc);
                acc += htot[k];
            }
            seg.push_back((uint32_t)acc);
        }
        MM_CUDA(ctx, cudaMemcpyAsync(hseg.p, seg.data(), 4 * seg.size(), cudaMemcpyHostToDevice, ctx->stream));
    }
    auto huge_pass = [&](int pass) -> mm_status {
        uint32_t seg_at = 0;
        for (const Batch& b : batches) {
            cudaError_t e = cudaSuccess;
            mm_status s2 = run(ctx, "similarity", [&] {
                e = launch_similarity_huge(dm, pass, u + o_ucoff, u + o_uc, u + o_uaoff, u + o_ua, u + o_huge + b.first,
                                           b.count, hseg.p + seg_at, (uint32_t)b.items, hkeys.p, hsorted.p, htemp.p,
                                           htemp.n, u + o_cnt, u + o_off, ctx->sim_out.p, ctl, ctx->stream);
            });
            if (s2) return s2;
            if (e != cudaSuccess) return cuda_fail(ctx, e, "similarity (huge rows)");
            seg_at += b.count + 1;
        }
        return MM_OK;
    };
    if (n_huge) {
        if (mm_status s2 = huge_pass(0)) return s2;
        MM_CUDA(ctx, cudaMemcpyAsync(h, ctl, sizeof(unsigned long long), cudaMemcpyDeviceToHost, ctx->stream));
        MM_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    }
    if (h[0] >= (1ull << 32)) return fail(ctx, MM_E_UNSUPPORTED, "mm_similarities: more than 2^32 - 1 pairs");
    ctx->sim_n = h[0];
    MM_CUDA(ctx, ctx->sim_out.ensure(ctx->sim_n ? ctx->sim_n : 1));
    st = run(ctx, "similarity", [&] {
        launch_scan(u + o_cnt, u + o_off, static_cast<uint32_t>(M), u + o_tot, small + 2, ctx->stream);
        launch_similarity_rows(dm, 1, u + o_ucoff, u + o_uc, u + o_uaoff, u + o_ua, u + o_cnt, u + o_off,
                               ctx->sim_out.p, u + o_wide, small, small + 1, ctl, u + o_huge, huge_tot, small + 3,
                               ctx->stream);
    });
    if (st) return st;
    if (n_huge)
        if (mm_status s2 = huge_pass(1)) return s2;
    MM_CUDA(ctx, cudaStreamSynchronize(ctx->stream));  // the batch scratch is freed on return
    ctx->sim_valid = true;
    return MM_OK;
}

mm_status mm_similarities(mm_ctx* ctx, mm_similarity* out, uint64_t cap, uint64_t* n_out) {
    if (!ctx || !n_out) return MM_E_ARG;
    if (!ctx->have_model) return fail(ctx, MM_E_STATE, "mm_similarities: no model uploaded");
    if (mm_status st = set_device(ctx)) return st;
    if (!ctx->sim_valid)
        if (mm_status st = compute_similarities(ctx)) return st;
    *n_out = ctx->sim_n;
    if (!out) return MM_OK;
    if (cap < ctx->sim_n) return fail(ctx, MM_E_CAPACITY, "mm_similarities: buffer too small");
    if (ctx->sim_n)
        MM_CUDA(ctx, cudaMemcpyAsync(out, ctx->sim_out.p, sizeof(mm_similarity) * ctx->sim_n, cudaMemcpyDeviceToHost,
                                     ctx->stream));
    MM_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    return MM_OK;
}

mm_status mm_suggest_similarity(mm_ctx* ctx, const mm_similarity* table, uint64_t n_table, double thr,
                                uint32_t all_candidates, mm_suggestion* out, uint64_t cap, uint64_t* n_out) {
    if (!ctx || !n_out || (n_table && !table)) return MM_E_ARG;
    if (mm_status st = ensure_metrics(ctx)) return st;
    const uint64_t M = ctx->M;
    // the pairs: the caller's report.similarity, else the device table
    const mm_similarity* tab = nullptr;
    uint64_t ntab = 0;
    if (table) {
        MM_CUDA(ctx, ctx->sim_caller.ensure(n_table ? n_table : 1));
        if (n_table)
            MM_CUDA(ctx, cudaMemcpyAsync(ctx->sim_caller.p, table, sizeof(mm_similarity) * n_table,
                                         cudaMemcpyHostToDevice, ctx->stream));
        tab = ctx->sim_caller.p;
        ntab = n_table;
    } else {
        if (!ctx->sim_valid)
            if (mm_status st = compute_similarities(ctx)) return st;
        tab = ctx->sim_out.p;
        ntab = ctx->sim_n;
    }
    for (uint64_t k = 0; table && k < n_table; ++k)
        if (table[k].first >= M || table[k].second >= M)
            return fail(ctx, MM_E_RANGE, "mm_suggest_similarity: unknown method id in the table");
    const uint64_t nb = (M + 1 + 1023) / 1024 + 1;
    const uint64_t o_cnt = 0, o_off = M + 1, o_cur = 2 * (M + 1), o_rc = 3 * (M + 1), o_ro = 4 * (M + 1),
                   o_tot = 5 * (M + 1), o_grand = o_tot + nb, o_part = o_grand + 1, o_end = o_part + 2 * ntab + 1;
    MM_CUDA(ctx, ctx->simc_u32.ensure(o_end));
    uint32_t* u = ctx->simc_u32.p;
    SweepArgs a{};
    a.s = ctx->dev();
    a.rec = ctx->rec.p;
    a.recs = ctx->recs.p;
    a.pos_owner = ctx->pos_owner.p;
    a.ux = ctx->ux.p;
    a.un = ctx->un.p;
    a.dense = ctx->dense.p;
    a.pos_begin = 0;
    a.pos_end = M;
    a.maxdeg_fast = ctx->max_deg <= 8 ? 8u : 16u;
    mm_status st = run(ctx, "sim_criterion", [&] {
        launch_sim_partners(tab, ntab, thr, ctx->method_owner.p, static_cast<uint32_t>(M), u + o_cnt, u + o_off,
                            u + o_cur, u + o_part, u + o_tot, u + o_grand, ctx->stream);
        cudaMemsetAsync(u + o_rc, 0, 4ull * (M + 1), ctx->stream);
        launch_sim_emit(a, 0, u + o_off, u + o_part, u + o_rc, nullptr, all_candidates, ctx->stream);
        launch_scan(u + o_rc, u + o_ro, static_cast<uint32_t>(M + 1), u + o_tot, u + o_grand, ctx->stream);
    });
    if (st) return st;
    uint32_t n = 0;
    MM_CUDA(ctx, cudaMemcpyAsync(&n, u + o_ro + M, 4, cudaMemcpyDeviceToHost, ctx->stream));
    MM_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    *n_out = n;
    if (!out) return n ? fail(ctx, MM_E_CAPACITY, "output buffer too small") : MM_OK;
    if (cap < n) return fail(ctx, MM_E_CAPACITY, "output buffer too small");
    if (!n) return MM_OK;
    MM_CUDA(ctx, ctx->simc_out.ensure(n));
    a.out = ctx->simc_out.p;
    st = run(ctx, "sim_criterion", [&] {
        launch_sim_emit(a, 1, u + o_off, u + o_part, u + o_rc, u + o_ro, all_candidates, ctx->stream);
    });
    if (st) return st;
    MM_CUDA(ctx, cudaMemcpyAsync(out, ctx->simc_out.p, sizeof(mm_suggestion) * n, cudaMemcpyDeviceToHost,
                                 ctx->stream));
    MM_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    return MM_OK;
}

mm_status mm_estimate_workload(mm_ctx* ctx, mm_workload* out) {
    if (!ctx || !out) return MM_E_ARG;
    if (!ctx->have_model) return fail(ctx, MM_E_STATE, "mm_estimate_workload: no model uploaded");
    if (mm_status st = set_device(ctx)) return st;
    MM_CUDA(ctx, ctx->fan.ensure(2 * (size_t)ctx->M + 2));
    uint32_t* kmax = ctx->fan.p + 2 * (size_t)ctx->M;
    mm_status st = run(ctx, "fan", [&] { launch_fan(ctx->dev(), nullptr, nullptr, kmax, ctx->stream); });
    if (st) return st;
    uint32_t k[2] = {0, 0};
    MM_CUDA(ctx, cudaMemcpyAsync(k, kmax, sizeof k, cudaMemcpyDeviceToHost, ctx->stream));
    MM_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    // estimate_workload_counts, metrics.hpp:211-226 (closed forms, exact in 64 bits)
    const uint64_t m = ctx->M, c = ctx->C;
    out->m = m;
    out->c = c;
    out->k_m = k[0];
    out->k_a = k[1];
    out->n_fan = 2 * m;
    out->n_sim = m == 0 ? 0 : m * (m - 1) / 2;
    out->n_lcom = c * (m + 1);
    out->n_cbo = c * (m + 1);
    out->n_total = out->n_fan + out->n_sim + out->n_lcom + out->n_cbo;
    return MM_OK;
}

mm_status mm_class_metrics_async(mm_ctx* ctx, double* lcom, uint64_t* lcom_ck, uint32_t* cbo) {
    if (!ctx) return MM_E_ARG;
    if (mm_status st = ensure_metrics(ctx)) return st;
    const size_t C = ctx->C;
    MM_CUDA(ctx, cudaEventRecord(ctx->ev_d2h_go, ctx->stream));
    MM_CUDA(ctx, cudaStreamWaitEvent(ctx->d2h, ctx->ev_d2h_go, 0));
    if (C && lcom) MM_CUDA(ctx, cudaMemcpyAsync(lcom, ctx->lcom.p, 8 * C, cudaMemcpyDeviceToHost, ctx->d2h));
    if (C && lcom_ck) MM_CUDA(ctx, cudaMemcpyAsync(lcom_ck, ctx->ck.p, 8 * C, cudaMemcpyDeviceToHost, ctx->d2h));
    if (C && cbo) MM_CUDA(ctx, cudaMemcpyAsync(cbo, ctx->cbo.p, 4 * C, cudaMemcpyDeviceToHost, ctx->d2h));
    MM_CUDA(ctx, cudaEventRecord(ctx->ev_d2h_done, ctx->d2h));
    return MM_OK;
}

static mm_status single(mm_ctx* ctx, uint32_t cls, void* dst, const void* src, size_t sz) {
    if (!ctx || !dst) return MM_E_ARG;
    if (mm_status st = ensure_metrics(ctx)) return st;
    if (cls >= ctx->C) return fail(ctx, MM_E_RANGE, "unknown class id " + std::to_string(cls));  // metrics.hpp:97-100
    MM_CUDA(ctx, cudaMemcpyAsync(dst, static_cast<const char*>(src) + sz * cls, sz, cudaMemcpyDeviceToHost,
                                 ctx->stream));
    MM_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    return MM_OK;
}

mm_status mm_lcom_normalized(mm_ctx* ctx, uint32_t cls, double* out) {
    return single(ctx, cls, out, ctx ? ctx->lcom.p : nullptr, 8);
}
mm_status mm_lcom_ck(mm_ctx* ctx, uint32_t cls, uint64_t* out) {
    return single(ctx, cls, out, ctx ? ctx->ck.p : nullptr, 8);
}
mm_status mm_cbo(mm_ctx* ctx, uint32_t cls, uint32_t* out) {
    return single(ctx, cls, out, ctx ? ctx->cbo.p : nullptr, 4);
}

// mean of n doubles on the device with compute_thresholds' sequential-sum
// semantics (the threshold kernel), into ctl->thr_aux; `values` is device memory
static mm_status device_mean(mm_ctx* ctx, const double* values, uint64_t n, double* mean, int* fast) {
    if (n >= 0xffffffffull) return fail(ctx, MM_E_RANGE, "mean: n too large");
    DevThresholds* dt = &ctx->ctl.p->thr_aux;
    DBuf<char> scratch;
    MM_CUDA(ctx, scratch.alloc(thresholds_scratch_bytes((uint32_t)n)));
    cudaError_t te = cudaSuccess;
    mm_status st = run(ctx, "thresholds", [&] {
        te = launch_thresholds(values, nullptr, (uint32_t)n, dt, scratch.p, scratch.n, ctx->stream, false);
    });
    if (st) return st;
    if (te != cudaSuccess) return cuda_fail(ctx, te, "thresholds");
    DevThresholds h{};
    MM_CUDA(ctx, cudaMemcpyAsync(&h, dt, sizeof h, cudaMemcpyDeviceToHost, ctx->stream));
    MM_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    *mean = h.lcom;
    if (fast) *fast = (int)h.fast_path_ok;
    return MM_OK;
}

mm_status mm_compute_thresholds(mm_ctx* ctx, const mm_overrides* ov, mm_thresholds* out) {
    if (!ctx || !out) return MM_E_ARG;
    if (mm_status st = ensure_metrics(ctx)) return st;
    if (mm_status st = join_thresholds(ctx)) return st;
    DevThresholds t{};
    MM_CUDA(ctx, cudaMemcpyAsync(&t, &ctx->ctl.p->thr, sizeof t, cudaMemcpyDeviceToHost, ctx->stream));
    MM_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    // similarity: the mean of full_report's similarity table (suggest.hpp:55-56),
    // the device table (built here when absent), in table order
    double sim_mean = 0.0;
    if (!(ov && ov->has_similarity)) {
        if (!ctx->sim_valid)
            if (mm_status st = compute_similarities(ctx)) return st;
        if (ctx->sim_n) {
            DBuf<double> vals;
            MM_CUDA(ctx, vals.alloc(ctx->sim_n));
            MM_CUDA(ctx, cudaMemcpy2DAsync(vals.p, sizeof(double), &ctx->sim_out.p->value, sizeof(mm_similarity),
                                           sizeof(double), ctx->sim_n, cudaMemcpyDeviceToDevice, ctx->stream));
            if (mm_status st = device_mean(ctx, vals.p, ctx->sim_n, &sim_mean, nullptr)) return st;
        }
    }
    std::memset(out, 0, sizeof *out);
    out->similarity = (ov && ov->has_similarity) ? ov->similarity : sim_mean;
    out->lcom = (ov && ov->has_lcom) ? ov->lcom : t.lcom;
    out->cbo = (ov && ov->has_cbo) ? ov->cbo : t.cbo;
    out->explicit_mode = (uint8_t)(ov && (ov->has_similarity || ov->has_lcom || ov->has_cbo));
    return MM_OK;
}

mm_status mm_report_thresholds(mm_ctx* ctx, const double* lcom, uint64_t n_lcom, const uint32_t* cbo, uint64_t n_cbo,
                               const double* similarity, uint64_t n_sim, const mm_overrides* ov, mm_thresholds* out) {
    if (!ctx || !out || (n_lcom && !lcom) || (n_cbo && !cbo) || (n_sim && !similarity)) return MM_E_ARG;
    if (n_lcom >= 0xffffffffull || n_cbo >= 0xffffffffull || n_sim >= 0xffffffffull)
        return fail(ctx, MM_E_RANGE, "compute_thresholds: too many values");
    if (mm_status st = set_device(ctx)) return st;
    const bool need_l = !(ov && ov->has_lcom), need_c = !(ov && ov->has_cbo), need_s = !(ov && ov->has_similarity);
    double ml = 0.0, mc = 0.0, ms = 0.0;
    DevThresholds* dt = &ctx->ctl.p->thr_aux;
    auto means = [&](const double* l, const uint32_t* c, uint64_t n, double* out_l, double* out_c) -> mm_status {
        if (!n) return MM_OK;
        DBuf<double> dl;
        DBuf<uint32_t> dc;
        MM_CUDA(ctx, dl.alloc(n));
        if (l) MM_CUDA(ctx, cudaMemcpyAsync(dl.p, l, 8 * n, cudaMemcpyHostToDevice, ctx->stream));
        else MM_CUDA(ctx, cudaMemsetAsync(dl.p, 0, 8 * n, ctx->stream));
        if (c) {
            MM_CUDA(ctx, dc.alloc(n));
            MM_CUDA(ctx, cudaMemcpyAsync(dc.p, c, 4 * n, cudaMemcpyHostToDevice, ctx->stream));
        }
        DBuf<char> scratch;
        MM_CUDA(ctx, scratch.alloc(thresholds_scratch_bytes((uint32_t)n)));
        cudaError_t te = cudaSuccess;
        mm_status st = run(ctx, "thresholds", [&] {
            te = launch_thresholds(dl.p, dc.p, (uint32_t)n, dt, scratch.p, scratch.n, ctx->stream, true);
        });
        if (st) return st;
        if (te != cudaSuccess) return cuda_fail(ctx, te, "thresholds");
        DevThresholds h{};
        MM_CUDA(ctx, cudaMemcpyAsync(&h, dt, sizeof h, cudaMemcpyDeviceToHost, ctx->stream));
        MM_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
        if (out_l) *out_l = h.lcom;
        if (out_c) *out_c = h.cbo;
        return MM_OK;
    };
    if (need_l && need_c && n_lcom == n_cbo) {
        if (mm_status st = means(lcom, cbo, n_lcom, &ml, &mc)) return st;
    } else {
        if (need_l)
            if (mm_status st = means(lcom, nullptr, n_lcom, &ml, nullptr)) return st;
        if (need_c)
            if (mm_status st = means(nullptr, cbo, n_cbo, nullptr, &mc)) return st;
    }
    if (need_s && n_sim) {
        DBuf<double> d;
        MM_CUDA(ctx, d.alloc(n_sim));
        MM_CUDA(ctx, cudaMemcpyAsync(d.p, similarity, 8 * n_sim, cudaMemcpyHostToDevice, ctx->stream));
        if (mm_status st = device_mean(ctx, d.p, n_sim, &ms, nullptr)) return st;
    }
    std::memset(out, 0, sizeof *out);
    out->similarity = need_s ? ms : ov->similarity;
    out->lcom = need_l ? ml : ov->lcom;
    out->cbo = need_c ? mc : ov->cbo;
    out->explicit_mode = (uint8_t)(ov && (ov->has_similarity || ov->has_lcom || ov->has_cbo));
    return MM_OK;
}

mm_status mm_what_if(mm_ctx* ctx, uint32_t method, uint32_t origin, uint32_t destination, mm_whatif* out) {
    if (!ctx || !out) return MM_E_ARG;
    if (!ctx->have_model) return fail(ctx, MM_E_STATE, "mm_what_if: no model uploaded");
    // error order of what_if_move, suggest.hpp:89-96
    if (origin >= ctx->C || destination >= ctx->C) return fail(ctx, MM_E_RANGE, "what_if_move: unknown class id");
    if (origin == destination) return fail(ctx, MM_E_ARG, "what_if_move: origin and destination coincide");
    const std::string not_member = "what_if_move: method " + std::to_string(method) +
                                   " is not a member of class " + std::to_string(origin);
    if (method >= ctx->M) return fail(ctx, MM_E_ARG, not_member);
    if (mm_status st = ensure_metrics(ctx)) return st;
    const DevModel dm = ctx->dev();
    mm_status st = run(ctx, "what_if", [&] {
        launch_what_if(dm, ctx->rec.p, ctx->ux.p, ctx->un.p, ctx->dense.p, method, origin, destination,
                       ctx->whatif.p, ctx->stream);
    });
    if (st) return st;
    MM_CUDA(ctx, cudaMemcpyAsync(out, ctx->whatif.p, sizeof *out, cudaMemcpyDeviceToHost, ctx->stream));
    MM_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    if (out->pad[0]) {  // the kernel found method_owner[method] != origin (suggest.hpp:93-96)
        std::memset(out, 0, sizeof *out);
        return fail(ctx, MM_E_ARG, not_member);
    }
    return MM_OK;
}

mm_status mm_set_gates(mm_ctx* ctx, const double* lcom, const uint32_t* cbo) {
    if (!ctx) return MM_E_ARG;
    if (!lcom && !cbo) {
        ctx->gates_set = false;
        ++ctx->layout_gen;
        return MM_OK;
    }
    if (!lcom || !cbo) return fail(ctx, MM_E_ARG, "mm_set_gates: give both vectors or neither");
    if (!ctx->have_model) return fail(ctx, MM_E_STATE, "mm_set_gates: no model uploaded");
    if (mm_status st = set_device(ctx)) return st;
    const size_t C = ctx->C;
    MM_CUDA(ctx, ctx->gate_lcom.ensure(C ? C : 1));
    MM_CUDA(ctx, ctx->gate_cbo.ensure(C ? C : 1));
    if (C) {
        MM_CUDA(ctx, cudaMemcpyAsync(ctx->gate_lcom.p, lcom, 8 * C, cudaMemcpyHostToDevice, ctx->stream));
        MM_CUDA(ctx, cudaMemcpyAsync(ctx->gate_cbo.p, cbo, 4 * C, cudaMemcpyHostToDevice, ctx->stream));
        MM_CUDA(ctx, cudaStreamSynchronize(ctx->stream));  // caller buffers may be pageable/temporary
    }
    ctx->gates_set = true;
    ++ctx->layout_gen;
    return MM_OK;
}

mm_status mm_sweep(mm_ctx* ctx, const mm_sweep_params* p, uint64_t* n_out) {
    if (!ctx || !p) return MM_E_ARG;
    const uint32_t sel = p->criteria & (MM_CRIT_SIMILARITY | MM_CRIT_COHESION | MM_CRIT_COUPLING);
    if (sel == 0) return fail(ctx, MM_E_ARG, "suggest_all: no criteria selected");  // suggest.hpp:313
    if (sel & MM_CRIT_SIMILARITY)
        return fail(ctx, MM_E_UNSUPPORTED, "Criterion::Similarity is outside this engine (needs the O(m^2) table)");
    if (p->combine > MM_COMBINE_INTERSECTION) return fail(ctx, MM_E_ARG, "mm_sweep: bad combine");
    if (!p->all_candidates && p->top_k > 8) return fail(ctx, MM_E_UNSUPPORTED, "mm_sweep: top_k > 8");
    if (mm_status st = ensure_metrics(ctx)) return st;
    const uint32_t cb = p->class_begin,
                   ce = (p->class_end || (p->flags & MM_SWEEP_EXACT_RANGE)) ? p->class_end : ctx->C;
    if (cb > ce || ce > ctx->C) return fail(ctx, MM_E_RANGE, "mm_sweep: class range outside the model");
    const uint32_t pb = ctx->h_cls_moff[cb], pe = ctx->h_cls_moff[ce];
    const uint64_t npos = pe - pb;
    const uint32_t mode = p->all_candidates ? 2u : (p->top_k > 1 ? 1u : 0u);
    const uint64_t per = mode == 0 ? 2ull : (mode == 1 ? 2ull * p->top_k : ~0ull);
    const uint64_t Etot = ctx->Ec + ctx->Ea;
    const uint64_t cap = std::max<uint64_t>(1, mode == 2 ? Etot : std::min(per * npos, Etot));
    const void* before[4] = {ctx->out.p, ctx->tile_state.p, ctx->res.p, ctx->emit_list.p};
    MM_CUDA(ctx, ctx->out.ensure(cap));
    const uint32_t n_tiles = (uint32_t)((npos + kSweepTile - 1) / kSweepTile);
    const uint32_t n_off = offsets_tiles(npos);
    const uint32_t n_state = n_off;
    MM_CUDA(ctx, ctx->tile_state.ensure(n_state ? n_state : 1));
    MM_CUDA(ctx, ctx->res.ensure(npos ? npos : 1));
    MM_CUDA(ctx, ctx->emit_list.ensure(npos ? npos : 1));
    const void* wide_before = ctx->wide_cnt.p;
    if (mode != 0) MM_CUDA(ctx, ctx->wide_cnt.ensure(npos ? npos : 1));
    if (wide_before != ctx->wide_cnt.p) ++ctx->layout_gen;
    const uint64_t n_fb = std::min<uint64_t>(npos, ctx->n_maybe_ovf);
    const void* fb_before = ctx->fallback.p;
    MM_CUDA(ctx, ctx->fallback.ensure(n_fb ? n_fb : 1));
    if (fb_before != ctx->fallback.p) ++ctx->layout_gen;
    const uint32_t fallback_tiles = (uint32_t)((n_fb + kSweepTile - 1) / kSweepTile);
    if (before[0] != ctx->out.p || before[1] != ctx->tile_state.p || before[2] != ctx->res.p ||
        before[3] != ctx->emit_list.p)
        ++ctx->layout_gen;
    Ctl* ctl = ctx->ctl.p;
    if (n_state) MM_CUDA(ctx, cudaMemsetAsync(ctx->tile_state.p, 0, 8ull * n_state, ctx->stream));
    // tile_counter, err, n_emit, n_wide, n_fallback, n_hideg (rezeroed: unused here), stats
    MM_CUDA(ctx, cudaMemsetAsync(&ctl->tile_counter, 0, offsetof(Ctl, thr) - offsetof(Ctl, tile_counter),
                                 ctx->stream));
    SweepArgs a{};
    a.s = ctx->dev();
    a.rec = ctx->rec.p;
    a.recs = ctx->recs.p;
    a.pos_owner = ctx->pos_owner.p;
    a.lcom = ctx->gates_set ? ctx->gate_lcom.p : ctx->lcom.p;
    a.cbo = ctx->gates_set ? ctx->gate_cbo.p : ctx->cbo.p;
    a.res = ctx->res.p - pb;  // indexed by absolute position
    a.emitters = ctx->emit_list.p;
    a.n_emit = &ctl->n_emit;
    a.ux = ctx->ux.p;
    a.un = ctx->un.p;
    a.dense = ctx->dense.p;
    a.dthr = &ctl->thr;
    a.thr_lcom = p->thr_lcom;
    a.thr_cbo = p->thr_cbo;
    a.thr_device = p->threshold_source == MM_THR_DEVICE_MEANS ? 1u : 0u;
    a.crit = sel;
    a.combine = p->combine;
    a.mode = mode;
    a.topk = mode == 1 ? p->top_k : 1u;
    a.pos_begin = pb;
    a.pos_end = pe;
    a.maxdeg_fast = ctx->max_deg <= 8 ? 8u : 16u;  // higher degrees take the streaming path
    a.out = ctx->out.p;
    a.tile_state = ctx->tile_state.p;
    a.tile_counter = &ctl->tile_counter;
    a.stats = ctl->stats;
    a.err = &ctl->err;
    a.wide_cnt = ctx->wide_cnt.p;
    a.n_wide = &ctl->n_wide;
    a.dlcom = ctx->lcom.p;
    a.fallback = ctx->fallback.p;
    a.n_fallback = &ctl->n_fallback;
    mm_status st = MM_OK;
    if (mode == 0 && ctx->score_fast && (uint64_t)ctx->n_maybe_ovf * 8 <= npos) {
        // (when many records may overflow — dense shapes — the general kernel
        // in one pass beats the fast pass plus its fallback list)
        st = run(ctx, "score", [&] { launch_score_fast(a, n_tiles, fallback_tiles, ctx->stream); });
        if (st) return st;
    } else {
        st = run(ctx, "score", [&] { launch_score(a, n_tiles, ctx->stream); });
        if (st) return st;
    }
    if (a.thr_device)
        if (mm_status s2 = join_thresholds(ctx)) return s2;
    st = run(ctx, "offsets", [&] { launch_offsets(a, n_off, ctx->stream); });
    if (st) return st;
    st = run(ctx, "write", [&] { launch_write(a, n_tiles, true, ctx->stream); });
    if (st) return st;
    ctx->sweep_valid = true;
    if (n_out) {
        mm_sweep_stats ss;
        if (mm_status s2 = mm_sweep_stats_get(ctx, &ss)) return s2;
        *n_out = ss.suggestions;
    }
    return MM_OK;
}

static void drop_graph(mm_ctx* ctx) {
    if (ctx->graph_exec) cudaGraphExecDestroy(ctx->graph_exec);
    ctx->graph_exec = nullptr;
    for (Pending& p : ctx->graph_events) {
        cudaEventDestroy(p.a);
        cudaEventDestroy(p.b);
    }
    ctx->graph_events.clear();
    ctx->graph_key.clear();
}

mm_status mm_run(mm_ctx* ctx, const mm_sweep_params* p) {
    if (!ctx || !p) return MM_E_ARG;
    if (!ctx->have_model) return fail(ctx, MM_E_STATE, "mm_run: no model uploaded");
    if (mm_status st = set_device(ctx)) return st;
    static const bool env_off = [] {
        const char* e = getenv("MMGPU_NO_GRAPH");
        return e && e[0] == '1';
    }();
    std::vector<uint8_t> key(sizeof *p + 3 * sizeof(uint64_t));
    std::memcpy(key.data(), p, sizeof *p);
    const uint64_t extra[3] = {ctx->layout_gen, (uint64_t)ctx->profiling, (uint64_t)(uintptr_t)ctx->stream};
    std::memcpy(key.data() + sizeof *p, extra, sizeof extra);
    if (!env_off && !ctx->graph_disabled && ctx->graph_exec && key == ctx->graph_key) {
        MM_CUDA(ctx, cudaGraphLaunch(ctx->graph_exec, ctx->stream));
        ctx->metrics_valid = ctx->sweep_valid = true;
        return MM_OK;
    }
    // eager step (this call's result), which also sizes every buffer the
    // graph will use: allocations cannot be captured
    if (mm_status st = mm_compute_metrics(ctx)) return st;
    if (mm_status st = mm_sweep(ctx, p, nullptr)) return st;
    if (env_off || ctx->graph_disabled) return MM_OK;
    key.resize(sizeof *p);
    key.insert(key.end(), reinterpret_cast<const uint8_t*>(&ctx->layout_gen),
               reinterpret_cast<const uint8_t*>(&ctx->layout_gen) + sizeof(uint64_t));
    const uint64_t more[2] = {(uint64_t)ctx->profiling, (uint64_t)(uintptr_t)ctx->stream};
    key.insert(key.end(), reinterpret_cast<const uint8_t*>(more), reinterpret_cast<const uint8_t*>(more) + sizeof more);
    MM_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    resolve_pending(ctx);
    drop_graph(ctx);
    // capture the same step
    if (cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
        ctx->graph_disabled = true;
        cudaGetLastError();
        return MM_OK;
    }
    ctx->capturing = true;
    const mm_status s1 = mm_compute_metrics(ctx);
    const mm_status s2 = s1 ? s1 : mm_sweep(ctx, p, nullptr);
    ctx->capturing = false;
    cudaGraph_t g = nullptr;
    const cudaError_t e = cudaStreamEndCapture(ctx->stream, &g);
    if (s2 || e != cudaSuccess || !g || cudaGraphInstantiate(&ctx->graph_exec, g, cudaGraphInstantiateFlagUseNodePriority) != cudaSuccess) {
        ctx->graph_disabled = true;  // keep running eagerly (the result above stands)
        ctx->graph_exec = nullptr;
        cudaGetLastError();
    } else {
        ctx->graph_key = key;
    }
    if (g) cudaGraphDestroy(g);
    ctx->metrics_valid = ctx->sweep_valid = true;
    return MM_OK;
}

mm_status mm_collect_timings(mm_ctx* ctx) {
    if (!ctx) return MM_E_ARG;
    MM_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    MM_CUDA(ctx, cudaStreamSynchronize(ctx->side));
    for (Pending& p : ctx->graph_events) {  // the last replay's kernel times
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, p.a, p.b) == cudaSuccess) {
            KStat& k = ctx->kstats[p.name];
            ++k.launches;
            k.total_ms += ms;
        }
    }
    cudaGetLastError();
    return MM_OK;
}

mm_status mm_sweep_stats_get(mm_ctx* ctx, mm_sweep_stats* out) {
    if (!ctx || !out) return MM_E_ARG;
    if (!ctx->sweep_valid) return fail(ctx, MM_E_STATE, "no sweep has run");
    Ctl h{};
    MM_CUDA(ctx, cudaMemcpyAsync(&h, ctx->ctl.p, sizeof h, cudaMemcpyDeviceToHost, ctx->stream));
    MM_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    out->candidates = h.stats[0];
    out->gated_whatifs = h.stats[1];
    out->suggestions = h.stats[2];
    out->methods = h.stats[3];
    return MM_OK;
}

mm_status mm_sweep_device_result(mm_ctx* ctx, const void** dev_records, uint64_t* n) {
    if (!ctx || !dev_records) return MM_E_ARG;
    if (!ctx->sweep_valid) return fail(ctx, MM_E_STATE, "no sweep has run");
    *dev_records = ctx->out.p;
    if (n) {
        mm_sweep_stats ss;
        if (mm_status st = mm_sweep_stats_get(ctx, &ss)) return st;
        *n = ss.suggestions;
    }
    return MM_OK;
}

mm_status mm_sweep_device_count(mm_ctx* ctx, const uint64_t** dev_count) {
    if (!ctx || !dev_count) return MM_E_ARG;
    if (!ctx->sweep_valid) return fail(ctx, MM_E_STATE, "no sweep has run");
    *dev_count = reinterpret_cast<const uint64_t*>(&ctx->ctl.p->stats[2]);
    return MM_OK;
}

mm_status mm_copy_suggestions(mm_ctx* ctx, mm_suggestion* out, uint64_t cap, uint64_t* n_out) {
    if (!ctx || !n_out) return MM_E_ARG;
    if (!out || !cap) {  // size query
        mm_sweep_stats ss;
        if (mm_status st = mm_sweep_stats_get(ctx, &ss)) return st;
        *n_out = ss.suggestions;
        return (!out && !ss.suggestions) || !ss.suggestions ? MM_OK
                                                            : fail(ctx, MM_E_CAPACITY, "output buffer too small");
    }
    if (!ctx->sweep_valid) return fail(ctx, MM_E_STATE, "no sweep has run");
    // one round trip: the count and up to `cap` records travel together (a
    // caller that sized `cap` from the previous sweep of the same system
    // gets exactly its records); a larger count reports MM_E_CAPACITY
    Ctl h{};
    const uint64_t k = std::min<uint64_t>(cap, ctx->out.n);
    MM_CUDA(ctx, cudaMemcpyAsync(&h, ctx->ctl.p, sizeof h, cudaMemcpyDeviceToHost, ctx->stream));
    if (k) MM_CUDA(ctx, cudaMemcpyAsync(out, ctx->out.p, sizeof(mm_suggestion) * k, cudaMemcpyDeviceToHost,
                                        ctx->stream));
    MM_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    *n_out = h.stats[2];
    if (h.stats[2] > cap) return fail(ctx, MM_E_CAPACITY, "output buffer too small");
    return MM_OK;
}

mm_status mm_sequential_mean(mm_ctx* ctx, const double* values, uint64_t n, double* out, int* fast_path) {
    if (!ctx || !out || (n && !values)) return MM_E_ARG;
    if (n >= 0xffffffffull) return fail(ctx, MM_E_RANGE, "mm_sequential_mean: n too large");
    if (mm_status st = set_device(ctx)) return st;
    DBuf<double> d;
    MM_CUDA(ctx, d.alloc(n ? n : 1));
    if (n) MM_CUDA(ctx, cudaMemcpyAsync(d.p, values, 8 * n, cudaMemcpyHostToDevice, ctx->stream));
    return device_mean(ctx, d.p, n, out, fast_path);
}

mm_status mm_pinned_alloc(uint64_t bytes, void** out) {
    if (!out) return MM_E_ARG;
    *out = nullptr;
    if (!bytes) return MM_OK;
    const cudaError_t e = cudaMallocHost(out, bytes);
    if (e == cudaErrorMemoryAllocation) return MM_E_OOM;
    return e == cudaSuccess ? MM_OK : MM_E_CUDA;
}

void mm_pinned_free(void* p) {
    if (p) cudaFreeHost(p);
}

mm_status mm_suggest(mm_ctx* ctx, const mm_sweep_params* p, mm_suggestion* out, uint64_t cap, uint64_t* n_out) {
    if (mm_status st = mm_sweep(ctx, p, nullptr)) return st;
    return mm_copy_suggestions(ctx, out, cap, n_out);
}

}  // extern "C"
