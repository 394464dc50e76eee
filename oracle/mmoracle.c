/*
 * mmoracle.c — literal CPU restatement of the reference hot path.
 * TEST INFRASTRUCTURE ONLY (see mmoracle.h). Paths below are relative to
 * /root/reference/proj/include/modmetrics/.
 */
#include "mmoracle.h"

#include <stdlib.h>
#include <string.h>

/* |a ∩ b| of two sorted unique lists by linear merge — detail::intersection_count, metrics.hpp:15-25 */
static uint64_t isect_count(const uint32_t* a, size_t na, const uint32_t* b, size_t nb) {
    uint64_t n = 0;
    size_t i = 0, j = 0;
    while (i < na && j < nb) {
        if (a[i] < b[j]) ++i;
        else if (b[j] < a[i]) ++j;
        else { ++n; ++i; ++j; }
    }
    return n;
}

static const uint32_t* acc_row(const mm_system* s, uint32_t p, size_t* n) {
    *n = s->acc_off[p + 1] - s->acc_off[p];
    return s->acc_tgt + s->acc_off[p];
}
static const uint32_t* call_row(const mm_system* s, uint32_t p, size_t* n) {
    *n = s->call_off[p + 1] - s->call_off[p];
    return s->call_tgt + s->call_off[p];
}
static const uint32_t* attrs_of(const mm_system* s, uint32_t c, size_t* n) {
    *n = s->class_attr_off[c + 1] - s->class_attr_off[c];
    return s->class_attrs + s->class_attr_off[c];
}
static const uint32_t* members_of(const mm_system* s, uint32_t c, size_t* n) {
    *n = s->class_method_off[c + 1] - s->class_method_off[c];
    return s->class_methods + s->class_method_off[c];
}

/* lcom_normalized_over, metrics.hpp:114-126:
 *   0 if attrs or methods empty, else 1 - hits / (A * M) with hits the summed
 *   |accesses(p) ∩ attrs(C)| — one division, as the reference does. */
double or_lcom_over(const mm_system* s, uint32_t cls, const uint32_t* methods, size_t n) {
    size_t na;
    const uint32_t* attrs = attrs_of(s, cls, &na);
    if (na == 0 || n == 0) return 0.0;
    uint64_t hits = 0;
    for (size_t i = 0; i < n; ++i) {
        size_t nacc;
        const uint32_t* acc = acc_row(s, methods[i], &nacc);
        hits += isect_count(acc, nacc, attrs, na);
    }
    const double denom = (double)na * (double)n;
    return 1.0 - (double)hits / denom;
}

/* lcom_ck_over, metrics.hpp:135-157: own-attribute sets by intersection
 * with attrs(C); pairs i<j sharing if their own sets intersect;
 * disjoint > sharing ? disjoint - sharing : 0; fewer than 2 methods -> 0. */
uint64_t or_lcom_ck_over(const mm_system* s, uint32_t cls, const uint32_t* methods, size_t n) {
    if (n < 2) return 0;
    size_t na;
    const uint32_t* attrs = attrs_of(s, cls, &na);
    uint32_t** own = (uint32_t**)calloc(n, sizeof(uint32_t*));
    size_t* nown = (size_t*)calloc(n, sizeof(size_t));
    for (size_t i = 0; i < n; ++i) {
        size_t nacc;
        const uint32_t* acc = acc_row(s, methods[i], &nacc);
        own[i] = (uint32_t*)malloc((nacc ? nacc : 1) * sizeof(uint32_t));
        size_t a = 0, b = 0, k = 0; /* set_intersection */
        while (a < nacc && b < na) {
            if (acc[a] < attrs[b]) ++a;
            else if (attrs[b] < acc[a]) ++b;
            else { own[i][k++] = acc[a]; ++a; ++b; }
        }
        nown[i] = k;
    }
    uint64_t disjoint = 0, sharing = 0;
    for (size_t i = 0; i < n; ++i)
        for (size_t j = i + 1; j < n; ++j) {
            if (isect_count(own[i], nown[i], own[j], nown[j]) > 0) ++sharing;
            else ++disjoint;
        }
    for (size_t i = 0; i < n; ++i) free(own[i]);
    free(own);
    free(nown);
    return disjoint > sharing ? disjoint - sharing : 0;
}

static int cmp_u32(const void* a, const void* b) {
    const uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
    return x < y ? -1 : x > y;
}

static size_t sort_unique_u32(uint32_t* v, size_t n) {
    if (n == 0) return 0;
    qsort(v, n, sizeof(uint32_t), cmp_u32);
    size_t k = 1;
    for (size_t i = 1; i < n; ++i)
        if (v[i] != v[k - 1]) v[k++] = v[i];
    return k;
}

/* cbo_over, metrics.hpp:167-185: distinct owners (≠ C) of everything the
 * methods call or access; push, sort, unique. */
uint32_t or_cbo_over(const mm_system* s, uint32_t cls, const uint32_t* methods, size_t n) {
    size_t cap = 0;
    for (size_t i = 0; i < n; ++i) {
        const uint32_t p = methods[i];
        cap += (s->call_off[p + 1] - s->call_off[p]) + (s->acc_off[p + 1] - s->acc_off[p]);
    }
    uint32_t* used = (uint32_t*)malloc((cap ? cap : 1) * sizeof(uint32_t));
    size_t k = 0;
    for (size_t i = 0; i < n; ++i) {
        size_t nc, nacc;
        const uint32_t* calls = call_row(s, methods[i], &nc);
        const uint32_t* acc = acc_row(s, methods[i], &nacc);
        for (size_t j = 0; j < nc; ++j) {
            const uint32_t o = s->method_owner[calls[j]];
            if (o != cls) used[k++] = o;
        }
        for (size_t j = 0; j < nacc; ++j) {
            const uint32_t o = s->attribute_owner[acc[j]];
            if (o != cls) used[k++] = o;
        }
    }
    const size_t u = sort_unique_u32(used, k);
    free(used);
    return (uint32_t)u;
}

/* fan_in, metrics.hpp:79-85: for every call list, ++in[t] per target;
 * fan_out, metrics.hpp:87-93: the call list's length */
int or_fan_metrics(const mm_system* s, uint32_t* fan_in, uint32_t* fan_out) {
    if (fan_in) {
        for (uint32_t p = 0; p < s->n_methods; ++p) fan_in[p] = 0;
        for (uint32_t q = 0; q < s->n_methods; ++q)
            for (uint32_t e = s->call_off[q]; e < s->call_off[q + 1]; ++e) ++fan_in[s->call_tgt[e]];
    }
    if (fan_out)
        for (uint32_t p = 0; p < s->n_methods; ++p) fan_out[p] = s->call_off[p + 1] - s->call_off[p];
    return MM_OK;
}

/* |a ∩ b| of two sorted unique lists, detail::intersection_count (metrics.hpp:15-25) */
static uint64_t isect(const uint32_t* a, uint32_t na, const uint32_t* b, uint32_t nb) {
    uint64_t n = 0;
    uint32_t i = 0, j = 0;
    while (i < na && j < nb) {
        if (a[i] < b[j]) ++i;
        else if (b[j] < a[i]) ++j;
        else { ++n; ++i; ++j; }
    }
    return n;
}

/* all_similarities, metrics.hpp:67-77 with similarity_if_nonzero (:47-55):
 * inter = shared calls + shared accesses, uni = |P_i| + |P_j| - inter,
 * value = (double)inter / (double)uni; pairs with inter == 0 not stored */
int or_similarities(const mm_system* s, mm_similarity* out, uint64_t cap, uint64_t* n_out) {
    uint64_t n = 0;
    for (uint32_t i = 0; i < s->n_methods; ++i) {
        const uint32_t ci = s->call_off[i], nci = s->call_off[i + 1] - ci;
        const uint32_t ai = s->acc_off[i], nai = s->acc_off[i + 1] - ai;
        for (uint32_t j = i + 1; j < s->n_methods; ++j) {
            const uint32_t cj = s->call_off[j], ncj = s->call_off[j + 1] - cj;
            const uint32_t aj = s->acc_off[j], naj = s->acc_off[j + 1] - aj;
            const uint64_t inter = isect(s->call_tgt + ci, nci, s->call_tgt + cj, ncj) +
                                   isect(s->acc_tgt + ai, nai, s->acc_tgt + aj, naj);
            if (inter == 0) continue;
            const uint64_t uni = (uint64_t)nci + nai + ncj + naj - inter;
            if (out && n < cap) {
                out[n].first = i;
                out[n].second = j;
                out[n].value = (double)inter / (double)uni;
            }
            ++n;
        }
    }
    *n_out = n;
    return (out && n > cap) ? MM_E_CAPACITY : MM_OK;
}

/* full_report class loop, metrics.hpp:253-261 */
int or_class_metrics(const mm_system* s, double* lcom, uint64_t* lcom_ck, uint32_t* cbo) {
    for (uint32_t c = 0; c < s->n_classes; ++c) {
        size_t n;
        const uint32_t* m = members_of(s, c, &n);
        if (lcom) lcom[c] = or_lcom_over(s, c, m, n);
        if (lcom_ck) lcom_ck[c] = or_lcom_ck_over(s, c, m, n);
        if (cbo) cbo[c] = or_cbo_over(s, c, m, n);
    }
    return MM_OK;
}

/* compute_thresholds, suggest.hpp:46-61: mean = sequential double sum / n,
 * 0 for empty input; an override replaces its mean; explicit_mode = any. */
int or_thresholds(const double* lcom, const uint32_t* cbo, uint64_t n_classes,
                  const double* similarity, uint64_t n_similarity,
                  const mm_overrides* ov, mm_thresholds* out) {
    double sl = 0.0, sc = 0.0, ss = 0.0;
    for (uint64_t i = 0; i < n_classes; ++i) sl += lcom[i];
    for (uint64_t i = 0; i < n_classes; ++i) sc += (double)cbo[i];
    for (uint64_t i = 0; i < n_similarity; ++i) ss += similarity[i];
    const double ml = n_classes ? sl / (double)n_classes : 0.0;
    const double mc = n_classes ? sc / (double)n_classes : 0.0;
    const double ms = n_similarity ? ss / (double)n_similarity : 0.0;
    mm_overrides none;
    memset(&none, 0, sizeof none);
    if (!ov) ov = &none;
    memset(out, 0, sizeof *out);
    out->similarity = ov->has_similarity ? ov->similarity : ms;
    out->lcom = ov->has_lcom ? ov->lcom : ml;
    out->cbo = ov->has_cbo ? ov->cbo : mc;
    out->explicit_mode = (uint8_t)(ov->has_similarity || ov->has_lcom || ov->has_cbo);
    return MM_OK;
}

static int member_of(const mm_system* s, uint32_t c, uint32_t method) {
    size_t n;
    const uint32_t* m = members_of(s, c, &n);
    size_t lo = 0, hi = n; /* std::binary_search */
    while (lo < hi) {
        const size_t mid = (lo + hi) / 2;
        if (m[mid] < method) lo = mid + 1;
        else hi = mid;
    }
    return lo < n && m[lo] == method;
}

/* what_if_move, suggest.hpp:87-122: recompute origin/destination metrics
 * over the moved membership, ownership frozen. */
int or_what_if(const mm_system* s, uint32_t method, uint32_t origin, uint32_t destination,
               mm_whatif* out) {
    if (origin >= s->n_classes || destination >= s->n_classes) return MM_E_RANGE; /* :89-90 */
    if (origin == destination) return MM_E_ARG;                                    /* :91-92 */
    if (!member_of(s, origin, method)) return MM_E_ARG;                            /* :93-96 */
    size_t no, nd;
    const uint32_t* om = members_of(s, origin, &no);
    const uint32_t* dm = members_of(s, destination, &nd);
    uint32_t* oa = (uint32_t*)malloc((no ? no : 1) * sizeof(uint32_t));
    uint32_t* da = (uint32_t*)malloc((nd + 1) * sizeof(uint32_t));
    size_t k = 0;
    for (size_t i = 0; i < no; ++i)
        if (om[i] != method) oa[k++] = om[i];
    size_t j = 0, w = 0; /* sorted insert (lower_bound) */
    while (j < nd && dm[j] < method) da[w++] = dm[j++];
    da[w++] = method;
    while (j < nd) da[w++] = dm[j++];
    memset(out, 0, sizeof *out);
    out->lcom_origin_before = or_lcom_over(s, origin, om, no);
    out->lcom_origin_after = or_lcom_over(s, origin, oa, k);
    out->lcom_dest_before = or_lcom_over(s, destination, dm, nd);
    out->lcom_dest_after = or_lcom_over(s, destination, da, w);
    out->cbo_origin_before = or_cbo_over(s, origin, om, no);
    out->cbo_origin_after = or_cbo_over(s, origin, oa, k);
    out->cbo_dest_before = or_cbo_over(s, destination, dm, nd);
    out->cbo_dest_after = or_cbo_over(s, destination, da, w);
    size_t naa, nad;
    attrs_of(s, origin, &naa);
    attrs_of(s, destination, &nad);
    out->origin_degenerate_after = (uint8_t)(k == 0 || naa == 0);
    out->dest_degenerate_after = (uint8_t)(nad == 0);
    free(oa);
    free(da);
    return MM_OK;
}

/* ---- suggestion sweep ------------------------------------------------- */

typedef struct {
    mm_suggestion* v;
    size_t n, cap;
} rec_vec;

static void push(rec_vec* r, const mm_suggestion* s) {
    if (r->n == r->cap) {
        r->cap = r->cap ? 2 * r->cap : 64;
        r->v = (mm_suggestion*)realloc(r->v, r->cap * sizeof(mm_suggestion));
    }
    r->v[r->n++] = *s;
}

/* used_classes, suggest.hpp:152-159: sorted-unique owners of calls ∪
 * accesses, minus the origin. Returns count; *out malloc'ed. */
static size_t used_classes(const mm_system* s, uint32_t u, uint32_t origin, uint32_t** out) {
    size_t nc, na;
    const uint32_t* calls = call_row(s, u, &nc);
    const uint32_t* acc = acc_row(s, u, &na);
    uint32_t* d = (uint32_t*)malloc((nc + na + 1) * sizeof(uint32_t));
    size_t k = 0;
    for (size_t i = 0; i < nc; ++i) {
        const uint32_t o = s->method_owner[calls[i]];
        if (o != origin) d[k++] = o;
    }
    for (size_t i = 0; i < na; ++i) {
        const uint32_t o = s->attribute_owner[acc[i]];
        if (o != origin) d[k++] = o;
    }
    *out = d;
    return sort_unique_u32(d, k);
}

/* lcom_improves / lcom_key, suggest.hpp:189-196; coupling predicate/key :285-290 */
static int passes(uint32_t crit, const mm_whatif* w) {
    if (crit == MM_CRIT_COHESION)
        return w->lcom_origin_after < w->lcom_origin_before && w->lcom_dest_after < w->lcom_dest_before;
    return w->cbo_origin_after < w->cbo_origin_before && w->cbo_dest_after <= w->cbo_dest_before;
}
static double key_of(uint32_t crit, const mm_whatif* w) {
    if (crit == MM_CRIT_COHESION) return w->lcom_origin_after + w->lcom_dest_after;
    return (double)w->cbo_dest_after;
}

static void fill(mm_suggestion* r, uint32_t u, uint32_t o, uint32_t d, uint32_t crit, const mm_whatif* w) {
    memset(r, 0, sizeof *r);
    r->method = u;
    r->origin = o;
    r->destination = d;
    r->criteria = (uint8_t)crit;
    r->lcom_origin_before = w->lcom_origin_before;
    r->lcom_origin_after = w->lcom_origin_after;
    r->lcom_dest_before = w->lcom_dest_before;
    r->lcom_dest_after = w->lcom_dest_after;
    r->cbo_origin_before = w->cbo_origin_before;
    r->cbo_origin_after = w->cbo_origin_after;
    r->cbo_dest_before = w->cbo_dest_before;
    r->cbo_dest_after = w->cbo_dest_after;
    r->origin_degenerate_after = w->origin_degenerate_after;
    r->dest_degenerate_after = w->dest_degenerate_after;
}

/* emit_for_method, suggest.hpp:165-187, generalised to keep the k smallest
 * (key, d) (k = 1 is the reference's best-only argmin, strict < so the first
 * minimum — lowest d — wins; k = SIZE_MAX is all_candidates in d order). */
static void emit_for_method(const mm_system* s, uint32_t u, uint32_t o, uint32_t crit, size_t k,
                            rec_vec* out) {
    uint32_t* dests;
    const size_t nd = used_classes(s, u, o, &dests);
    mm_suggestion* keep = (mm_suggestion*)malloc((nd ? nd : 1) * sizeof(mm_suggestion));
    double* keys = (double*)malloc((nd ? nd : 1) * sizeof(double));
    size_t nk = 0;
    for (size_t i = 0; i < nd; ++i) {
        mm_whatif w;
        or_what_if(s, u, o, dests[i], &w);
        if (!passes(crit, &w)) continue;
        fill(&keep[nk], u, o, dests[i], crit, &w);
        keys[nk++] = key_of(crit, &w);
    }
    if (k >= nk) {
        for (size_t i = 0; i < nk; ++i) push(out, &keep[i]);
    } else {
        /* select the k smallest (key, d); candidates are in ascending d, so a
         * stable selection on key alone yields the lexicographic order */
        unsigned char* taken = (unsigned char*)calloc(nk, 1);
        for (size_t r = 0; r < k; ++r) {
            size_t best = nk;
            for (size_t i = 0; i < nk; ++i)
                if (!taken[i] && (best == nk || keys[i] < keys[best])) best = i;
            taken[best] = 1;
        }
        for (size_t i = 0; i < nk; ++i)
            if (taken[i]) push(out, &keep[i]);
        free(taken);
    }
    free(keep);
    free(keys);
    free(dests);
}

static int cmp_method_dest(const void* a, const void* b) {
    const mm_suggestion* x = (const mm_suggestion*)a;
    const mm_suggestion* y = (const mm_suggestion*)b;
    if (x->method != y->method) return x->method < y->method ? -1 : 1;
    if (x->destination != y->destination) return x->destination < y->destination ? -1 : 1;
    return x->criteria < y->criteria ? -1 : x->criteria > y->criteria;
}
static int cmp_origin_method_dest(const void* a, const void* b) {
    const mm_suggestion* x = (const mm_suggestion*)a;
    const mm_suggestion* y = (const mm_suggestion*)b;
    if (x->origin != y->origin) return x->origin < y->origin ? -1 : 1;
    if (x->method != y->method) return x->method < y->method ? -1 : 1;
    return x->destination < y->destination ? -1 : x->destination > y->destination;
}

/* suggest_by_cohesion :239-259 / suggest_by_coupling :266-294 gated per
 * class, merged as suggest_all :303-350 (map keyed (method, dest), tags
 * unioned, intersection keeps all-tag entries, final (origin, method, dest)
 * sort). Per-criterion emission order inside a class (fan_out / fan_in+out,
 * :248-251, :275-280) does not affect the merged list and is not restated. */
int or_suggest(const mm_system* s, const double* lcom_gate, const uint32_t* cbo_gate,
               const mm_sweep_params* p, mm_suggestion* out, uint64_t cap, uint64_t* n_out) {
    const uint32_t sel = p->criteria & (MM_CRIT_SIMILARITY | MM_CRIT_COHESION | MM_CRIT_COUPLING);
    if (sel == 0) return MM_E_ARG; /* :313 */
    if (sel & MM_CRIT_SIMILARITY) return MM_E_UNSUPPORTED;
    const uint32_t cb = p->class_begin;
    const uint32_t ce = p->class_end ? p->class_end : s->n_classes;
    if (cb > ce || ce > s->n_classes) return MM_E_RANGE;
    const size_t k = p->all_candidates ? (size_t)-1 : (p->top_k > 1 ? p->top_k : 1);
    rec_vec all = {0, 0, 0};
    static const uint32_t order[2] = {MM_CRIT_COHESION, MM_CRIT_COUPLING};
    for (int ci = 0; ci < 2; ++ci) {
        const uint32_t crit = order[ci];
        if (!(sel & crit)) continue;
        for (uint32_t c = cb; c < ce; ++c) {
            const int gated = crit == MM_CRIT_COHESION ? lcom_gate[c] > p->thr_lcom
                                                       : (double)cbo_gate[c] > p->thr_cbo;
            if (!gated) continue;
            size_t n;
            const uint32_t* m = members_of(s, c, &n);
            for (size_t i = 0; i < n; ++i) emit_for_method(s, m[i], c, crit, k, &all);
        }
    }
    /* merge by (method, destination) */
    if (all.n) qsort(all.v, all.n, sizeof(mm_suggestion), cmp_method_dest);
    size_t w = 0;
    for (size_t i = 0; i < all.n; ++i) {
        if (w && all.v[w - 1].method == all.v[i].method && all.v[w - 1].destination == all.v[i].destination)
            all.v[w - 1].criteria |= all.v[i].criteria;
        else
            all.v[w++] = all.v[i];
    }
    size_t kept = 0;
    for (size_t i = 0; i < w; ++i) {
        if (p->combine == MM_COMBINE_INTERSECTION && all.v[i].criteria != sel) continue;
        all.v[kept++] = all.v[i];
    }
    if (kept) qsort(all.v, kept, sizeof(mm_suggestion), cmp_origin_method_dest);
    *n_out = kept;
    int rc = MM_OK;
    if (out && cap >= kept) memcpy(out, all.v, kept * sizeof(mm_suggestion));
    else if (kept) rc = MM_E_CAPACITY;
    free(all.v);
    return rc;
}
