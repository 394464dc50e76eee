// Host-side shard planning for the multi-GPU candidate sweep.
//
// The reference partitions work into balanced contiguous index ranges by
// COUNT (plan_partition, /root/reference/proj/include/modmetrics/parallel.hpp:28-41),
// which leaves one worker with the giant class under skew.
// Shards here are contiguous CLASS ranges too — so concatenating per-rank
// outputs in rank order preserves the (origin, method, destination) order of
// suggest_all (suggest.hpp:344-348) — but balanced by sweep cost:
// cost(c) = Σ_{p ∈ c} (1 + |calls(p)| + |accesses(p)|).

#include <cstdint>
#include <vector>

#include "../../include/mmgpu.h"

extern "C" mm_status mm_plan_shards(const mm_system* sys, uint32_t n_shards, uint32_t* bounds) {
    if (!sys || !bounds || n_shards == 0) return MM_E_ARG;  // parallel.hpp:29
    const uint32_t C = sys->n_classes;
    std::vector<uint64_t> prefix(C + 1, 0);
    for (uint32_t c = 0; c < C; ++c) {
        uint64_t cost = 0;
        for (uint32_t i = sys->class_method_off[c]; i < sys->class_method_off[c + 1]; ++i) {
            const uint32_t p = sys->class_methods[i];
            cost += 1 + (sys->call_off[p + 1] - sys->call_off[p]) + (sys->acc_off[p + 1] - sys->acc_off[p]);
        }
        prefix[c + 1] = prefix[c] + cost;
    }
    const uint64_t total = prefix[C];
    bounds[0] = 0;
    uint32_t c = 0;
    for (uint32_t k = 1; k < n_shards; ++k) {
        // first class boundary whose prefix cost reaches k/n of the total
        const unsigned __int128 target = (unsigned __int128)total * k;
        while (c < C && (unsigned __int128)prefix[c] * n_shards < target) ++c;
        bounds[k] = c;
    }
    bounds[n_shards] = C;
    return MM_OK;
}
