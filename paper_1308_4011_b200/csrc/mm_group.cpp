// mm_group.cpp — one host process driving several GPUs (include/mmgpu.h,
// mm_group_*): SURVEY.md §8b's mm_comm_init and §8e's partitioning.
//
// The reference parallelises over n_workers std::threads (parallel.hpp:109-135,
// plan_partition :20-41); here n_workers maps to GPUs. Each GPU holds a full
// copy of the system and recomputes the metric pass (replicas: the class
// tables every shard's scoring reads are a few MB); the
// candidate sweep is split into contiguous class ranges balanced by cost
// (mm_plan_shards). Ranks own ascending class ranges and each shard's list is
// already in (origin, method, destination) order, so the rank-order
// concatenation is suggest_all's list (suggest.hpp:344-348). The exchange
// moves exact counts over NCCL (one communicator clique from
// ncclCommInitAll, driven from this thread with ncclGroupStart/End):
//   1. ncclAllGather of each GPU's device-resident record count (8 bytes),
//   2. one ncclBroadcast per non-empty shard of exactly its 64-byte records,
//      into that shard's slice of every GPU's assembled list.
// NCCL is loaded with dlopen when a group is created, so libmmgpu.so itself
// has no link-time NCCL dependency (and coexists with the NCCL that torch
// loads); a group of one GPU works without it.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include "../../include/mmgpu.h"

namespace {

struct Nccl {
    void* h = nullptr;
    ncclResult_t (*comm_init_all)(ncclComm_t*, int, const int*) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*group_start)() = nullptr;
    ncclResult_t (*group_end)() = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;

    bool load(std::string& err) {
        // an NCCL already in the process (e.g. the one torch loaded) first: a
        // second libnccl.so.2 of another version would shadow it by soname
        h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h)
            if (const char* p = std::getenv("MMGPU_NCCL_LIB")) h = dlopen(p, RTLD_NOW | RTLD_LOCAL);
        for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
            if (h) break;
            h = dlopen(name, RTLD_NOW | RTLD_LOCAL);
        }
        if (!h) {
            err = "NCCL not found (dlopen libnccl.so.2 failed)";
            return false;
        }
        bool ok = true;
        auto sym = [&](auto& fn, const char* n) {
            fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, n));
            ok = ok && fn;
        };
        sym(comm_init_all, "ncclCommInitAll");
        sym(comm_destroy, "ncclCommDestroy");
        sym(all_gather, "ncclAllGather");
        sym(broadcast, "ncclBroadcast");
        sym(group_start, "ncclGroupStart");
        sym(group_end, "ncclGroupEnd");
        sym(error_string, "ncclGetErrorString");
        if (!ok) err = "NCCL library lacks a required symbol";
        return ok;
    }
};

}  // namespace

struct mm_group {
    int n = 0;
    std::vector<int> dev;
    std::vector<mm_ctx*> ctx;
    Nccl nccl;
    bool use_nccl = false;
    std::vector<ncclComm_t> comm;
    std::vector<uint32_t> bounds;        // shard i sweeps classes [bounds[i], bounds[i+1])
    std::vector<uint64_t*> d_counts;     // per GPU: n gathered record counts
    std::vector<mm_suggestion*> d_list;  // per GPU: the assembled list
    std::vector<uint64_t> cap;           // records each d_list holds
    std::vector<uint64_t> counts, offs;  // last exchange, per shard
    uint64_t total = 0;
    bool have_model = false, have_list = false;
    std::string err;
};

namespace {

mm_status gfail(mm_group* g, mm_status st, const std::string& msg) {
    if (g) g->err = msg;
    return st;
}

mm_status gcuda(mm_group* g, cudaError_t e, const char* where) {
    return gfail(g, e == cudaErrorMemoryAllocation ? MM_E_OOM : MM_E_CUDA, std::string(where) + ": " +
                                                                              cudaGetErrorString(e));
}

mm_status gnccl(mm_group* g, ncclResult_t r, const char* where) {
    return gfail(g, MM_E_NCCL, std::string(where) + ": " + (g->nccl.error_string ? g->nccl.error_string(r) : "?"));
}

// f(i) on one host thread per GPU; the first failing status (lowest GPU) wins
template <class F>
mm_status per_gpu(mm_group* g, F&& f) {
    std::vector<mm_status> st(g->n, MM_OK);
    std::vector<std::string> msg(g->n);
    auto body = [&](int i) {
        try {
            if (cudaSetDevice(g->dev[i]) != cudaSuccess) {
                st[i] = MM_E_CUDA;
                msg[i] = "cudaSetDevice failed";
                return;
            }
            st[i] = f(i);
            if (st[i] != MM_OK) msg[i] = mm_last_error(g->ctx[i]);
        } catch (const std::bad_alloc&) {
            st[i] = MM_E_OOM;
            msg[i] = "host allocation failed";
        } catch (const std::exception& e) {
            st[i] = MM_E_STATE;
            msg[i] = e.what();
        }
    };
    if (g->n == 1) {
        body(0);
    } else {
        std::vector<std::thread> th;
        th.reserve(g->n);
        for (int i = 0; i < g->n; ++i) th.emplace_back(body, i);
        for (std::thread& t : th) t.join();
    }
    for (int i = 0; i < g->n; ++i)
        if (st[i] != MM_OK) return gfail(g, st[i], "gpu " + std::to_string(g->dev[i]) + ": " + msg[i]);
    return MM_OK;
}

}  // namespace

extern "C" {

mm_status mm_group_create(const int* devices, int n, mm_group** out) {
    if (!out) return MM_E_ARG;
    *out = nullptr;
    if (n <= 0) return MM_E_ARG;  // plan_partition: zero workers (parallel.hpp:29)
    int n_dev = 0;
    if (cudaGetDeviceCount(&n_dev) != cudaSuccess || n_dev == 0) return MM_E_CUDA;
    mm_group* g = new (std::nothrow) mm_group();
    if (!g) return MM_E_OOM;
    g->n = n;
    for (int i = 0; i < n; ++i) {
        const int d = devices ? devices[i] : i;
        if (d < 0 || d >= n_dev || std::count(g->dev.begin(), g->dev.end(), d)) {
            delete g;
            return MM_E_RANGE;
        }
        g->dev.push_back(d);
    }
    g->ctx.assign(n, nullptr);
    for (int i = 0; i < n; ++i)
        if (mm_status st = mm_ctx_create(g->dev[i], &g->ctx[i])) {
            mm_group_destroy(g);
            return st;
        }
    // NCCL for the exchange (a one-GPU group needs none; MMGPU_GROUP_NCCL=0 opts out there)
    const char* env = std::getenv("MMGPU_GROUP_NCCL");
    const bool want = n > 1 || !(env && env[0] == '0');
    if (want) {
        std::string e;
        if (g->nccl.load(e)) {
            g->comm.assign(n, nullptr);
            const ncclResult_t r = g->nccl.comm_init_all(g->comm.data(), n, g->dev.data());
            if (r != ncclSuccess) {
                g->comm.clear();
                if (n > 1) {
                    mm_group_destroy(g);
                    return MM_E_NCCL;
                }
            } else {
                g->use_nccl = true;
            }
        } else if (n > 1) {
            mm_group_destroy(g);
            return MM_E_NCCL;
        }
    }
    g->d_counts.assign(n, nullptr);
    g->d_list.assign(n, nullptr);
    g->cap.assign(n, 0);
    for (int i = 0; i < n; ++i) {
        if (cudaSetDevice(g->dev[i]) != cudaSuccess ||
            cudaMalloc(reinterpret_cast<void**>(&g->d_counts[i]), sizeof(uint64_t) * n) != cudaSuccess) {
            mm_group_destroy(g);
            return MM_E_CUDA;
        }
    }
    *out = g;
    return MM_OK;
}

void mm_group_destroy(mm_group* g) {
    if (!g) return;
    for (size_t i = 0; i < g->comm.size(); ++i)
        if (g->comm[i]) g->nccl.comm_destroy(g->comm[i]);
    for (int i = 0; i < g->n; ++i) {
        if (i < (int)g->dev.size()) cudaSetDevice(g->dev[i]);
        if (i < (int)g->d_counts.size() && g->d_counts[i]) cudaFree(g->d_counts[i]);
        if (i < (int)g->d_list.size() && g->d_list[i]) cudaFree(g->d_list[i]);
        if (i < (int)g->ctx.size() && g->ctx[i]) mm_ctx_destroy(g->ctx[i]);
    }
    // the NCCL library stays loaded (other groups, or torch, may use it)
    delete g;
}

const char* mm_group_last_error(const mm_group* g) { return g ? g->err.c_str() : "null group"; }

int mm_group_size(const mm_group* g) { return g ? g->n : 0; }

mm_ctx* mm_group_ctx(mm_group* g, int i) { return (g && i >= 0 && i < g->n) ? g->ctx[i] : nullptr; }

int mm_group_uses_nccl(const mm_group* g) { return g && g->use_nccl ? 1 : 0; }

mm_status mm_group_upload(mm_group* g, const mm_system* sys) {
    if (!g || !sys) return MM_E_ARG;
    g->have_model = g->have_list = false;
    g->bounds.assign(g->n + 1, 0);
    if (mm_status st = mm_plan_shards(sys, static_cast<uint32_t>(g->n), g->bounds.data()))
        return gfail(g, st, "mm_plan_shards failed");
    if (mm_status st = per_gpu(g, [&](int i) { return mm_upload(g->ctx[i], sys); })) return st;
    g->have_model = true;
    return MM_OK;
}

mm_status mm_group_shard(const mm_group* g, int i, uint32_t* class_begin, uint32_t* class_end) {
    if (!g || i < 0 || i >= g->n || !class_begin || !class_end) return MM_E_ARG;
    if (!g->have_model) return MM_E_STATE;
    *class_begin = g->bounds[i];
    *class_end = g->bounds[i + 1];
    return MM_OK;
}

mm_status mm_group_set_gates(mm_group* g, const double* lcom, const uint32_t* cbo) {
    if (!g) return MM_E_ARG;
    return per_gpu(g, [&](int i) { return mm_set_gates(g->ctx[i], lcom, cbo); });
}

mm_status mm_group_run(mm_group* g, const mm_sweep_params* p, uint64_t* n_out) {
    if (!g || !p) return MM_E_ARG;
    if (!g->have_model) return gfail(g, MM_E_STATE, "mm_group_run: no model uploaded");
    g->have_list = false;
    // 1. every GPU: metric pass + the sweep of its shard (one graph replay each)
    std::vector<cudaStream_t> stream(g->n);
    std::vector<const void*> recs(g->n);
    std::vector<const uint64_t*> dcount(g->n);
    if (mm_status st = per_gpu(g, [&](int i) {
            mm_sweep_params q = *p;
            q.class_begin = g->bounds[i];
            q.class_end = g->bounds[i + 1];
            q.flags |= MM_SWEEP_EXACT_RANGE;  // an empty shard sweeps nothing (still runs the metric pass)
            void* s = nullptr;
            if (mm_status e = mm_ctx_stream(g->ctx[i], &s)) return e;
            stream[i] = static_cast<cudaStream_t>(s);
            if (mm_status e = mm_run(g->ctx[i], &q)) return e;
            if (mm_status e = mm_sweep_device_count(g->ctx[i], &dcount[i])) return e;
            return mm_sweep_device_result(g->ctx[i], &recs[i], nullptr);
        }))
        return st;
    // 2. all-gather the exact counts
    g->counts.assign(g->n, 0);
    if (g->use_nccl) {
        ncclResult_t r = g->nccl.group_start();
        for (int i = 0; i < g->n && r == ncclSuccess; ++i)
            r = g->nccl.all_gather(dcount[i], g->d_counts[i], 1, ncclUint64, g->comm[i], stream[i]);
        const ncclResult_t r2 = g->nccl.group_end();
        if (r != ncclSuccess) return gnccl(g, r, "ncclAllGather (counts)");
        if (r2 != ncclSuccess) return gnccl(g, r2, "ncclGroupEnd (counts)");
        if (cudaSetDevice(g->dev[0]) != cudaSuccess) return gfail(g, MM_E_CUDA, "cudaSetDevice");
        cudaError_t e = cudaMemcpyAsync(g->counts.data(), g->d_counts[0], sizeof(uint64_t) * g->n,
                                        cudaMemcpyDeviceToHost, stream[0]);
        if (e == cudaSuccess) e = cudaStreamSynchronize(stream[0]);
        if (e != cudaSuccess) return gcuda(g, e, "counts D2H");
    } else {  // one GPU, no NCCL: the count is local
        if (cudaSetDevice(g->dev[0]) != cudaSuccess) return gfail(g, MM_E_CUDA, "cudaSetDevice");
        cudaError_t e = cudaMemcpyAsync(g->counts.data(), dcount[0], sizeof(uint64_t), cudaMemcpyDeviceToHost,
                                        stream[0]);
        if (e == cudaSuccess) e = cudaStreamSynchronize(stream[0]);
        if (e != cudaSuccess) return gcuda(g, e, "count D2H");
    }
    g->offs.assign(g->n, 0);
    uint64_t acc = 0;
    for (int i = 0; i < g->n; ++i) {
        g->offs[i] = acc;
        acc += g->counts[i];
    }
    g->total = acc;
    // 3. exactly the records, each shard's into its slice of every GPU's list
    for (int i = 0; i < g->n; ++i) {
        if (g->cap[i] >= std::max<uint64_t>(acc, 1)) continue;
        if (cudaSetDevice(g->dev[i]) != cudaSuccess) return gfail(g, MM_E_CUDA, "cudaSetDevice");
        if (cudaStreamSynchronize(stream[i]) != cudaSuccess) return gfail(g, MM_E_CUDA, "stream sync");
        if (g->d_list[i]) cudaFree(g->d_list[i]);
        g->d_list[i] = nullptr;
        g->cap[i] = 0;
        const uint64_t want = std::max<uint64_t>(acc + acc / 8, 1);
        if (cudaError_t e = cudaMalloc(reinterpret_cast<void**>(&g->d_list[i]), sizeof(mm_suggestion) * want))
            return gcuda(g, e, "group list");
        g->cap[i] = want;
    }
    if (g->use_nccl) {
        ncclResult_t r = g->nccl.group_start();
        for (int s = 0; s < g->n && r == ncclSuccess; ++s) {
            if (!g->counts[s]) continue;
            for (int i = 0; i < g->n && r == ncclSuccess; ++i)
                r = g->nccl.broadcast(i == s ? recs[s] : g->d_list[i] + g->offs[s], g->d_list[i] + g->offs[s],
                                      sizeof(mm_suggestion) * g->counts[s], ncclUint8, s, g->comm[i], stream[i]);
        }
        const ncclResult_t r2 = g->nccl.group_end();
        if (r != ncclSuccess) return gnccl(g, r, "ncclBroadcast (records)");
        if (r2 != ncclSuccess) return gnccl(g, r2, "ncclGroupEnd (records)");
    } else if (g->counts[0]) {
        if (cudaError_t e = cudaMemcpyAsync(g->d_list[0], recs[0], sizeof(mm_suggestion) * g->counts[0],
                                            cudaMemcpyDeviceToDevice, stream[0]))
            return gcuda(g, e, "list copy");
    }
    g->have_list = true;
    if (n_out) {
        *n_out = acc;
        for (int i = 0; i < g->n; ++i) {
            cudaSetDevice(g->dev[i]);
            if (cudaError_t e = cudaStreamSynchronize(stream[i])) return gcuda(g, e, "group sync");
        }
    }
    return MM_OK;
}

mm_status mm_group_synchronize(mm_group* g) {
    if (!g) return MM_E_ARG;
    return per_gpu(g, [&](int i) { return mm_ctx_synchronize(g->ctx[i]); });
}

mm_status mm_group_counts(const mm_group* g, uint64_t* counts, uint64_t* total) {
    if (!g) return MM_E_ARG;
    if (!g->have_list) return MM_E_STATE;
    if (counts) std::copy(g->counts.begin(), g->counts.end(), counts);
    if (total) *total = g->total;
    return MM_OK;
}

mm_status mm_group_device_result(mm_group* g, int i, const void** dev_records, uint64_t* n) {
    if (!g || !dev_records || i < 0 || i >= g->n) return MM_E_ARG;
    if (!g->have_list) return gfail(g, MM_E_STATE, "no group sweep has run");
    *dev_records = g->d_list[i];
    if (n) *n = g->total;
    return MM_OK;
}

mm_status mm_group_copy_suggestions(mm_group* g, mm_suggestion* out, uint64_t cap, uint64_t* n_out) {
    if (!g || !n_out) return MM_E_ARG;
    if (!g->have_list) return gfail(g, MM_E_STATE, "no group sweep has run");
    *n_out = g->total;
    if (!out || cap < g->total) return g->total ? gfail(g, MM_E_CAPACITY, "output buffer too small") : MM_OK;
    if (!g->total) return MM_OK;
    if (cudaSetDevice(g->dev[0]) != cudaSuccess) return gfail(g, MM_E_CUDA, "cudaSetDevice");
    void* s = nullptr;
    mm_ctx_stream(g->ctx[0], &s);
    cudaError_t e = cudaMemcpyAsync(out, g->d_list[0], sizeof(mm_suggestion) * g->total, cudaMemcpyDeviceToHost,
                                    static_cast<cudaStream_t>(s));
    if (e == cudaSuccess) e = cudaStreamSynchronize(static_cast<cudaStream_t>(s));
    if (e != cudaSuccess) return gcuda(g, e, "list D2H");
    return MM_OK;
}

}  // extern "C"
