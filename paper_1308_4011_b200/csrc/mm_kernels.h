// mm_kernels.h — host-visible launchers of the CUDA kernels (libmmgpu internals).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "mm_device.cuh"

namespace mmg {

// Per large class (CTA path) scratch placement, planned on the host at upload.
constexpr uint32_t kCkChunk = 16;  // members per k_ck_rows CTA (2 per warp: latency-bound chains)
constexpr uint32_t kGiantMembers = 512;  // histogram classes this large: phase 1 over many CTAs
constexpr uint32_t kGiantChunk = 256;     // members (= threads) per k_giant_p1 CTA

struct LargePlan {
    uint64_t keys_off;     // u32 element offset into the global key scratch
    uint64_t rows_off;     // u32 element offset into the global row scratch
    uint32_t keys_cap;     // power of two ≥ foreign edge count (≥ foreign keys)
    uint8_t keys_in_smem;
    uint8_t rows_in_smem;
    uint8_t ck_masks;      // 1: per-member own-attribute masks (A ≤ 256) in smem; 0: attribute bitmaps
    uint8_t hist;          // 1: foreign classes counted in an smem histogram over all C (no keys)
    uint32_t pre_slot;     // giants: slot of the global histogram / H that k_giant_p1 fills; else kNone
    uint32_t ck_mma;       // 1: LCOM-CK by k_ck_mma on the tensor cores (this kernel skips phase 4)
};

struct SweepArgs {
    DevModel s;
    const ClassRec* rec;
    const MethRec* recs;  // per-method records in class order (method pass)
    const uint32_t* pos_owner;  // owning class per class-order position
    const double* lcom;         // per-class lcom (gates)
    const uint32_t* cbo;        // per-class cbo (gates)
    uint4* res;                 // per-position pass-1 result
    uint4* emitters;            // pass 2: (position, gated selection x, y, first record) per emitting method
    uint32_t* n_emit;           // their count
    const uint32_t* ux;
    const uint32_t* un;
    const uint32_t* dense;      // exact U-row bitmaps of dense classes (ClassRec::dense)
    const DevThresholds* dthr;  // used when thr_device != 0
    double thr_lcom, thr_cbo;
    uint32_t thr_device;
    uint32_t crit;       // MM_CRIT_COHESION | MM_CRIT_COUPLING subset
    uint32_t combine;    // MM_COMBINE_*
    uint32_t mode;       // 0 best-only, 1 top-k, 2 all candidates
    uint32_t topk;       // mode 1: 2..8
    uint32_t pos_begin, pos_end;  // class-ordered method positions
    uint32_t maxdeg_fast;         // methods with degree ≤ this take the register path
    mm_suggestion* out;
    unsigned long long* tile_state;
    uint32_t* tile_counter;
    unsigned long long* stats;  // [candidates, gated, suggestions, methods]
    uint32_t* err;              // reserved error bits
    uint4* wide_cnt;            // top-k / all modes: counts of methods with ≥ 32 used classes
    uint32_t* n_wide;           // their number
    const double* dlcom;        // the metric pass's lcom per class (lcom_normalized; not the gates)
    uint32_t* fallback;         // best-only: positions k_score_fast handed to the per-thread kernel
    uint32_t* n_fallback;
};

void launch_validate_ids(const uint32_t* v, uint64_t n, uint32_t bound, uint32_t* bad, cudaStream_t st);
void launch_expand(const DevModel& s, uint32_t* mo_out, uint32_t* ao_out, uint32_t* pos_owner, uint2* info,
                   cudaStream_t st);
void launch_fan(const DevModel& s, uint32_t* fan_in, uint32_t* fan_out, uint32_t* kmax, cudaStream_t st);
void launch_validate_offsets(const uint32_t* off, uint64_t n1, uint32_t total, uint32_t* bad, cudaStream_t st);
void launch_plan_classes(const DevModel& s, uint4* cplan, uint4* cedge, uint32_t* large_list,
                         uint32_t* n_large, uint32_t* big_list, uint32_t* n_big, uint32_t* max_deg,
                         const uint32_t* foreign, const uint32_t* cmaxdeg, cudaStream_t st);
// upload: the dependency rows in class order (DevModel::pc_* / pa_*), and the
// class plan's per-class foreign-edge counts / largest degree / n_hideg
void launch_pos_rows(const DevModel& s, const uint32_t* pos_owner, uint32_t* pc_off, uint32_t* pc_tgt,
                     uint32_t* pa_off, uint32_t* pa_tgt, uint8_t* pc_mem, uint8_t* pa_mem, uint32_t* totals,
                     uint32_t* foreign, uint32_t* cmaxdeg, uint32_t* n_hideg, cudaStream_t st);  // totals: 2 per 256-position tile
void launch_class_lean(const DevModel& s, const uint4* cplan, const uint4* cedge, const uint8_t* pc_mem,
                       const uint8_t* pa_mem, MethRec* recs, ClassRec* rec, double* lcom,
                       uint64_t* ck, uint32_t* cbo, uint32_t* ux, uint32_t* un, const uint32_t* list,
                       uint32_t n_list, cudaStream_t st);
void launch_class_group(const DevModel& s, const uint4* cplan, const uint2* groups, uint32_t n_groups,
                        const uint32_t* pos_owner, MethRec* recs, ClassRec* rec, double* lcom, uint64_t* ck,
                        uint32_t* cbo, uint32_t* ux, uint32_t* un, cudaStream_t st);
void launch_nl_positions(const uint32_t* pos_owner, const uint4* cplan, uint32_t M, uint32_t* out, uint32_t* n,
                         cudaStream_t st);
void launch_plan_groups(const uint4* cplan, const uint32_t* foreign, const uint32_t* cmaxdeg, uint32_t C,
                        uint2* groups, uint32_t* n_groups, uint32_t* solo, uint32_t* n_solo, cudaStream_t st);
void launch_method(const DevModel& s, MethRec* recs, uint64_t* own_mask, const uint32_t* pos_owner,
                   uint32_t max_deg, const uint32_t* plist, uint32_t n_pos, cudaStream_t st);
void launch_class_small(const DevModel& s, const uint4* cplan, const uint32_t* big_list, uint32_t n_big,
                        MethRec* recs, const uint64_t* own_mask, ClassRec* rec, double* lcom, uint64_t* ck,
                        uint32_t* cbo, uint32_t* ux, uint32_t* un, bool lean, cudaStream_t st,
                        cudaStream_t st_big);
void launch_class_large(const DevModel& s, uint32_t n_large, const uint32_t* large_list, const LargePlan* plan,
                        uint32_t smem_bytes, MethRec* recs, const uint64_t* own_mask, ClassRec* rec, double* lcom,
                        uint64_t* ck, uint32_t* cbo, uint32_t* ux, uint32_t* un, uint32_t* ucursor,
                        uint32_t* gkeys, uint32_t* grows, uint32_t* dense, uint32_t dense_cap,
                        uint32_t* dense_cursor, const uint32_t* gcnt, const unsigned long long* gH,
                        uint32_t threads, cudaStream_t st);
void launch_giant_p1(const DevModel& s, const uint32_t* large_list, const LargePlan* plan, const uint2* items,
                     uint32_t n_items, const MethRec* recs, uint32_t* gcnt, unsigned long long* gH, uint32_t* grows,
                     cudaStream_t st);
// LCOM-CK of listed dense classes (A ≤ 64) on the tensor cores (k_ck_mma.cu)
uint32_t ck_mma_smem_bytes(uint32_t max_members);
cudaError_t set_ck_mma_smem(uint32_t bytes);
void launch_ck_mma(const DevModel& s, const uint32_t* list, uint32_t n, uint32_t smem_bytes,
                   const uint64_t* own_mask, uint64_t* ck, cudaStream_t st);
// similarity table (k_similarity.cu)
cudaError_t launch_similarity_index(const DevModel& s, uint64_t Ec, uint64_t Ea, uint32_t* uc_off, uint32_t* uc,
                                    uint32_t* ua_off, uint32_t* ua, uint32_t* cur, uint32_t* totals,
                                    uint32_t* grand, cudaStream_t st);
cudaError_t launch_similarity_rows(const DevModel& s, int pass, const uint32_t* uc_off, const uint32_t* uc,
                                   const uint32_t* ua_off, const uint32_t* ua, uint32_t* row_cnt,
                                   const uint32_t* row_off, mm_similarity* out, uint32_t* wide_list, uint32_t* n_wide,
                                   uint32_t* err, unsigned long long* total, uint32_t* huge_list,
                                   unsigned long long* huge_tot, uint32_t* n_huge, cudaStream_t st);
// rows beyond the warp buffers: batches of (rows, segment offsets, items) through global scratch
size_t similarity_huge_temp_bytes(uint32_t max_items, uint32_t max_rows);
cudaError_t launch_similarity_huge(const DevModel& s, int pass, const uint32_t* uc_off, const uint32_t* uc,
                                   const uint32_t* ua_off, const uint32_t* ua, const uint32_t* rows, uint32_t n_rows,
                                   const uint32_t* seg, uint32_t n_items, uint32_t* keys, uint32_t* sorted,
                                   void* temp, size_t temp_bytes, uint32_t* row_cnt, const uint32_t* row_off,
                                   mm_similarity* out, unsigned long long* total, cudaStream_t st);
cudaError_t launch_scan(const uint32_t* in, uint32_t* out, uint32_t n, uint32_t* totals, uint32_t* grand,
                        cudaStream_t st);
// similarity criterion (k_sweep.cu)
void launch_sim_partners(const mm_similarity* tab, uint64_t n, double thr, const uint32_t* owner, uint32_t M,
                         uint32_t* cnt, uint32_t* off, uint32_t* cur, uint32_t* part, uint32_t* totals, uint32_t* grand,
                         cudaStream_t st);
void launch_sim_emit(const SweepArgs& a, int pass, const uint32_t* part_off, const uint32_t* part, uint32_t* rec_cnt,
                     const uint32_t* rec_off, uint32_t all_candidates, cudaStream_t st);
cudaError_t set_class_large_smem(uint32_t bytes);
void launch_ck_rows(const DevModel& s, const uint32_t* large_list, const LargePlan* plan, const uint2* items,
                    uint32_t n_items, const uint32_t* grows, const uint32_t* split_list, uint32_t n_split,
                    uint64_t* ck, cudaStream_t st);
// means with sequential-sum semantics; cbo may be NULL (treated as zeros)
size_t thresholds_scratch_bytes(uint32_t n);
// allow_serial: small n may take the one-warp serial kernel (faster there)
cudaError_t launch_thresholds(const double* lcom, const uint32_t* cbo, uint32_t n, DevThresholds* out,
                              void* scratch, size_t scratch_bytes, cudaStream_t st, bool allow_serial = true);
void launch_score(const SweepArgs& a, uint32_t n_tiles, cudaStream_t st);
uint32_t offsets_tiles(uint64_t npos);
void launch_score_fast(const SweepArgs& a, uint32_t n_tiles, uint32_t fallback_tiles, cudaStream_t st);
void launch_offsets(const SweepArgs& a, uint32_t n_tiles, cudaStream_t st);
void launch_write(const SweepArgs& a, uint32_t n_tiles, bool fast_list, cudaStream_t st);
constexpr uint32_t kSweepTile = 256;
void launch_what_if(const DevModel& s, const ClassRec* rec, const uint32_t* ux, const uint32_t* un,
                    const uint32_t* dense, uint32_t u, uint32_t o, uint32_t d, mm_whatif* out, cudaStream_t st);

}  // namespace mmg
