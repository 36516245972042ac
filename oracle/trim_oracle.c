/*
 * trim_oracle.c — TEST INFRASTRUCTURE ONLY (see trim_oracle.h).
 *
 * A plain-C restatement of the reference's candidate-filtering path. Every
 * function cites the reference lines it follows (paths relative to
 * /root/reference/proj/include/trimsearch). Build with -ffp-contract=off and
 * no -march flag: the reference binary has no FMA, so every
 * fp32 multiply and add here is individually rounded, in the same order.
 */
#include "trim_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static __thread char g_err[512];

static int fail(int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
    return code;
}

const char* or_last_error(void) { return g_err; }

void or_free(void* p) { free(p); }

/* core/distance.hpp:11-29 — four interleaved accumulators over blocks of 4,
 * remainder into acc0, result (acc0+acc1)+(acc2+acc3). */
float or_euclidean_sq(const float* a, const float* b, size_t dim) {
    float acc0 = 0.0f, acc1 = 0.0f, acc2 = 0.0f, acc3 = 0.0f;
    size_t i = 0;
    for (; i + 4 <= dim; i += 4) {
        const float d0 = a[i] - b[i];
        const float d1 = a[i + 1] - b[i + 1];
        const float d2 = a[i + 2] - b[i + 2];
        const float d3 = a[i + 3] - b[i + 3];
        acc0 += d0 * d0;
        acc1 += d1 * d1;
        acc2 += d2 * d2;
        acc3 += d3 * d3;
    }
    for (; i < dim; ++i) {
        const float d = a[i] - b[i];
        acc0 += d * d;
    }
    return (acc0 + acc1) + (acc2 + acc3);
}

/* trim/lower_bound.hpp:9-14 */
float or_strict_lb(float gl_q, float gl_x) {
    const float d = gl_q - gl_x;
    return d * d;
}

/* trim/lower_bound.hpp:18-22: strict_lb + 2.0f*gamma*gl_q*gl_x, evaluated
 * left to right: ((2*gamma)*gl_q)*gl_x. */
float or_relaxed_lb(float gl_q, float gl_x, float gamma) {
    return or_strict_lb(gl_q, gl_x) + 2.0f * gamma * gl_q * gl_x;
}

static const float* centroid(const or_index* ix, uint32_t j, uint32_t c) {
    return ix->centroids + (size_t)ix->ksub * ix->sub_offsets[j] + (size_t)c * ix->sub_dims[j];
}

/* pq/pq.hpp:158-172 */
void or_build_distance_table(const or_index* ix, const float* q, float* table) {
    for (uint32_t j = 0; j < ix->m; ++j) {
        const float* qs = q + ix->sub_offsets[j];
        float* row = table + (size_t)j * ix->ksub;
        for (uint32_t c = 0; c < ix->ksub; ++c)
            row[c] = or_euclidean_sq(qs, centroid(ix, j, c), ix->sub_dims[j]);
    }
}

/* pq/pq.hpp:186-192 — sequential sum from 0.0f over j = 0..m-1. */
float or_adc_lookup(const float* table, uint32_t m, uint32_t ksub, const uint8_t* code) {
    float acc = 0.0f;
    for (uint32_t j = 0; j < m; ++j)
        acc += table[(size_t)j * ksub + code[j]];
    return acc;
}

/* ScoredId ordering, core/ground_truth.hpp:39-50: by dist_sq, ties by id. */
typedef struct {
    float d;
    uint32_t id;
} scored;

static int scored_less(scored a, scored b) {
    if (a.d != b.d)
        return a.d < b.d;
    return a.id < b.id;
}

static int scored_cmp(const void* pa, const void* pb) {
    const scored a = *(const scored*)pa, b = *(const scored*)pb;
    if (scored_less(a, b))
        return -1;
    if (scored_less(b, a))
        return 1;
    return 0;
}

/* ivf/ivf.hpp:173-187 — all nlist coarse distances, full sort, first nprobe. */
uint32_t or_probe_order(const or_index* ix, const float* q, uint32_t nprobe, uint32_t* order,
                        uint64_t* coarse_dc) {
    scored* s = (scored*)malloc(sizeof(scored) * ix->nlist);
    for (uint32_t c = 0; c < ix->nlist; ++c) {
        s[c].d = or_euclidean_sq(q, ix->coarse + (size_t)c * ix->dim, ix->dim);
        s[c].id = c;
    }
    *coarse_dc += ix->nlist;
    qsort(s, ix->nlist, sizeof(scored), scored_cmp);
    const uint32_t np = nprobe < ix->nlist ? nprobe : ix->nlist;
    for (uint32_t i = 0; i < np; ++i)
        order[i] = s[i].id;
    free(s);
    return np;
}

/* pq/kmeans.hpp:27-41 — strict < keeps the lowest index on ties. */
uint32_t or_nearest_centroid(const float* x, const float* centroids, uint32_t k, uint32_t dim) {
    uint32_t best = 0;
    float best_d = 3.402823466e+38f; /* std::numeric_limits<float>::max() */
    for (uint32_t c = 0; c < k; ++c) {
        const float d = or_euclidean_sq(x, centroids + (size_t)c * dim, dim);
        if (d < best_d) {
            best_d = d;
            best = c;
        }
    }
    return best;
}

/* pq/pq.hpp:116-134 */
void or_pq_encode(const or_index* ix, const float* x, uint8_t* code) {
    for (uint32_t j = 0; j < ix->m; ++j) {
        const float* xs = x + ix->sub_offsets[j];
        uint32_t best = 0;
        float best_d = 3.402823466e+38f;
        for (uint32_t c = 0; c < ix->ksub; ++c) {
            const float d = or_euclidean_sq(xs, centroid(ix, j, c), ix->sub_dims[j]);
            if (d < best_d) {
                best_d = d;
                best = c;
            }
        }
        code[j] = (uint8_t)best;
    }
}

/* trim/landmarks.hpp:66-70 with pq::decode (pq.hpp:137-148): the landmark is
 * the concatenation of the selected centroids. */
float or_landmark_dist(const or_index* ix, const float* x, const uint8_t* code) {
    float* l = (float*)malloc(sizeof(float) * ix->dim);
    for (uint32_t j = 0; j < ix->m; ++j)
        memcpy(l + ix->sub_offsets[j], centroid(ix, j, code[j]), sizeof(float) * ix->sub_dims[j]);
    const float r = sqrtf(or_euclidean_sq(x, l, ix->dim));
    free(l);
    return r;
}

/* ---- max-heap on ScoredId (std::priority_queue<ScoredId>, worst on top) ---- */
static void heap_push(scored* h, uint32_t* n, scored v) {
    uint32_t i = (*n)++;
    h[i] = v;
    while (i > 0) {
        const uint32_t p = (i - 1) / 2;
        if (!scored_less(h[p], h[i]))
            break;
        scored t = h[p];
        h[p] = h[i];
        h[i] = t;
        i = p;
    }
}

static void heap_replace_top(scored* h, uint32_t n, scored v) {
    uint32_t i = 0;
    h[0] = v;
    for (;;) {
        const uint32_t l = 2 * i + 1, r = l + 1;
        uint32_t big = i;
        if (l < n && scored_less(h[big], h[l]))
            big = l;
        if (r < n && scored_less(h[big], h[r]))
            big = r;
        if (big == i)
            break;
        scored t = h[big];
        h[big] = h[i];
        h[i] = t;
        i = big;
    }
}

static const float* row_of(const or_index* ix, uint32_t id) {
    return ix->vectors + (size_t)id * ix->dim;
}

/* ivf/ivf.hpp:243-304 — single pass; first k entries of the probe stream are
 * exact-evaluated unconditionally (dc, no edc, :264-271); then evaluate iff
 * relaxed_lb < max_dis (prune on tie, :275), replace top iff (d,id) < top. */
int or_search_trim_knn(const or_index* ix, const float* q, uint32_t k, uint32_t nprobe,
                       float gamma, uint32_t* ids_out, float* dist_out, or_counters* ct,
                       uint64_t* coarse_dc) {
    if (k == 0)
        return fail(OR_EINVAL, "search_trim_ivf_knn: k must be positive");
    if (!(gamma >= 0.0f))
        return fail(OR_EINVAL, "search_trim_ivf_knn: uncalibrated pruning profile");
    memset(ct, 0, sizeof *ct);
    *coarse_dc = 0;
    uint32_t* order = (uint32_t*)malloc(sizeof(uint32_t) * (ix->nlist ? ix->nlist : 1));
    const uint32_t np = or_probe_order(ix, q, nprobe, order, coarse_dc);
    float* table = (float*)malloc(sizeof(float) * (size_t)ix->m * ix->ksub);
    or_build_distance_table(ix, q, table);
    scored* heap = (scored*)malloc(sizeof(scored) * k);
    uint32_t hn = 0;
    float max_dis = INFINITY;
    for (uint32_t pi = 0; pi < np; ++pi) {
        const uint32_t c = order[pi];
        for (uint64_t e = ix->list_offsets[c]; e < ix->list_offsets[c + 1]; ++e) {
            ++ct->evaluated;
            const uint32_t id = ix->list_ids[e];
            if (hn < k) {
                const float d = or_euclidean_sq(q, row_of(ix, id), ix->dim);
                ++ct->dc;
                scored v = {d, id};
                heap_push(heap, &hn, v);
                if (hn == k)
                    max_dis = heap[0].d;
                continue;
            }
            const float glq =
                sqrtf(or_adc_lookup(table, ix->m, ix->ksub, ix->list_codes + e * ix->code_stride));
            ++ct->edc;
            const float est = or_relaxed_lb(glq, ix->list_lx[e], gamma);
            if (est < max_dis) {
                const float d = or_euclidean_sq(q, row_of(ix, id), ix->dim);
                ++ct->dc;
                scored v = {d, id};
                if (scored_less(v, heap[0])) {
                    heap_replace_top(heap, hn, v);
                    max_dis = heap[0].d;
                }
            } else {
                ++ct->pruned;
            }
        }
    }
    int rc = OR_OK;
    if (hn < k) {
        rc = fail(OR_EINVAL, "search_trim_ivf_knn: k exceeds probed vectors");
    } else {
        qsort(heap, hn, sizeof(scored), scored_cmp);
        for (uint32_t i = 0; i < hn; ++i) {
            ids_out[i] = heap[i].id;
            dist_out[i] = heap[i].d;
        }
    }
    free(heap);
    free(table);
    free(order);
    return rc;
}

/* ivf/ivf.hpp:308-347 — evaluate iff est <= r^2, member iff d <= r^2, sort. */
int or_search_trim_range(const or_index* ix, const float* q, float radius, uint32_t nprobe,
                         float gamma, uint32_t** ids_out, float** dist_out, uint64_t* count,
                         or_counters* ct, uint64_t* coarse_dc) {
    *ids_out = NULL;
    *dist_out = NULL;
    *count = 0;
    if (radius < 0.0f)
        return fail(OR_EINVAL, "search_trim_ivf_range: negative radius");
    if (!(gamma >= 0.0f))
        return fail(OR_EINVAL, "search_trim_ivf_range: uncalibrated pruning profile");
    const float radius_sq = radius * radius;
    memset(ct, 0, sizeof *ct);
    *coarse_dc = 0;
    uint32_t* order = (uint32_t*)malloc(sizeof(uint32_t) * (ix->nlist ? ix->nlist : 1));
    const uint32_t np = or_probe_order(ix, q, nprobe, order, coarse_dc);
    float* table = (float*)malloc(sizeof(float) * (size_t)ix->m * ix->ksub);
    or_build_distance_table(ix, q, table);
    uint64_t cap = 64, n = 0;
    scored* res = (scored*)malloc(sizeof(scored) * cap);
    for (uint32_t pi = 0; pi < np; ++pi) {
        const uint32_t c = order[pi];
        for (uint64_t e = ix->list_offsets[c]; e < ix->list_offsets[c + 1]; ++e) {
            ++ct->evaluated;
            const float glq =
                sqrtf(or_adc_lookup(table, ix->m, ix->ksub, ix->list_codes + e * ix->code_stride));
            ++ct->edc;
            const float est = or_relaxed_lb(glq, ix->list_lx[e], gamma);
            if (est <= radius_sq) {
                const uint32_t id = ix->list_ids[e];
                const float d = or_euclidean_sq(q, row_of(ix, id), ix->dim);
                ++ct->dc;
                if (d <= radius_sq) {
                    if (n == cap) {
                        cap *= 2;
                        res = (scored*)realloc(res, sizeof(scored) * cap);
                    }
                    res[n].d = d;
                    res[n].id = id;
                    ++n;
                }
            } else {
                ++ct->pruned;
            }
        }
    }
    qsort(res, n, sizeof(scored), scored_cmp);
    uint32_t* ids = (uint32_t*)malloc(sizeof(uint32_t) * (n ? n : 1));
    float* ds = (float*)malloc(sizeof(float) * (n ? n : 1));
    for (uint64_t i = 0; i < n; ++i) {
        ids[i] = res[i].id;
        ds[i] = res[i].d;
    }
    *ids_out = ids;
    *dist_out = ds;
    *count = n;
    free(res);
    free(table);
    free(order);
    return OR_OK;
}

/* ivf/ivf.hpp:193-237 — ADC for every probed entry, the k' smallest by
 * (est,id) (std::partial_sort), exact refine, sort by (d,id), first k. */
int or_search_baseline_ivfpq(const or_index* ix, const float* q, uint32_t k, uint32_t nprobe,
                             uint32_t k_prime, uint32_t* ids_out, float* dist_out,
                             uint64_t* nres, or_counters* ct, uint64_t* coarse_dc) {
    *nres = 0;
    if (k == 0 || k > k_prime)
        return fail(OR_EINVAL, "search_baseline_ivfpq: need 1 <= k <= k_prime");
    if (nprobe == 0)
        return fail(OR_EINVAL, "search_baseline_ivfpq: nprobe must be positive");
    memset(ct, 0, sizeof *ct);
    *coarse_dc = 0;
    uint32_t* order = (uint32_t*)malloc(sizeof(uint32_t) * (ix->nlist ? ix->nlist : 1));
    const uint32_t np = or_probe_order(ix, q, nprobe, order, coarse_dc);
    float* table = (float*)malloc(sizeof(float) * (size_t)ix->m * ix->ksub);
    or_build_distance_table(ix, q, table);
    uint64_t total = 0;
    for (uint32_t pi = 0; pi < np; ++pi)
        total += ix->list_offsets[order[pi] + 1] - ix->list_offsets[order[pi]];
    scored* cand = (scored*)malloc(sizeof(scored) * (total ? total : 1));
    uint64_t n = 0;
    for (uint32_t pi = 0; pi < np; ++pi) {
        const uint32_t c = order[pi];
        for (uint64_t e = ix->list_offsets[c]; e < ix->list_offsets[c + 1]; ++e) {
            cand[n].d = or_adc_lookup(table, ix->m, ix->ksub, ix->list_codes + e * ix->code_stride);
            cand[n].id = ix->list_ids[e];
            ++n;
            ++ct->edc;
            ++ct->evaluated;
        }
    }
    int rc = OR_OK;
    if (k > n) {
        rc = fail(OR_EINVAL, "search_baseline_ivfpq: k exceeds probed vectors");
    } else {
        const uint64_t refine_n = k_prime < n ? k_prime : n;
        /* the set of the refine_n smallest (est,id) is unique; a full sort
         * selects the same prefix as std::partial_sort */
        qsort(cand, n, sizeof(scored), scored_cmp);
        scored* refined = (scored*)malloc(sizeof(scored) * (refine_n ? refine_n : 1));
        for (uint64_t i = 0; i < refine_n; ++i) {
            refined[i].d = or_euclidean_sq(q, row_of(ix, cand[i].id), ix->dim);
            refined[i].id = cand[i].id;
            ++ct->dc;
        }
        ct->pruned = ct->evaluated - ct->dc;
        qsort(refined, refine_n, sizeof(scored), scored_cmp);
        const uint64_t out = k < refine_n ? k : refine_n;
        for (uint64_t i = 0; i < out; ++i) {
            ids_out[i] = refined[i].id;
            dist_out[i] = refined[i].d;
        }
        *nres = out;
        free(refined);
    }
    free(cand);
    free(table);
    free(order);
    return rc;
}


/* ======================= HNSW graph search (graph/search.hpp) ============= */
/* A growable binary heap of ScoredId; max-heap when `maxh`, else min-heap
 * (std::priority_queue<ScoredId> / <..., std::greater<ScoredId>>). */
typedef struct {
    scored* h;
    uint64_t n, cap;
    int maxh;
} gheap;

static int gh_above(const gheap* q, scored a, scored b) { /* a belongs above b */
    return q->maxh ? scored_less(b, a) : scored_less(a, b);
}
static int gh_push(gheap* q, scored v) {
    if (q->n == q->cap) {
        uint64_t nc = q->cap ? 2 * q->cap : 64;
        scored* nh = (scored*)realloc(q->h, sizeof(scored) * nc);
        if (!nh)
            return fail(OR_ENOMEM, "graph search: heap allocation failed");
        q->h = nh;
        q->cap = nc;
    }
    uint64_t i = q->n++;
    q->h[i] = v;
    while (i > 0) {
        const uint64_t p = (i - 1) / 2;
        if (!gh_above(q, q->h[i], q->h[p]))
            break;
        scored t = q->h[p];
        q->h[p] = q->h[i];
        q->h[i] = t;
        i = p;
    }
    return OR_OK;
}
static scored gh_pop(gheap* q) {
    const scored top = q->h[0];
    q->h[0] = q->h[--q->n];
    uint64_t i = 0;
    for (;;) {
        const uint64_t l = 2 * i + 1, r = l + 1;
        uint64_t b = i;
        if (l < q->n && gh_above(q, q->h[l], q->h[b]))
            b = l;
        if (r < q->n && gh_above(q, q->h[r], q->h[b]))
            b = r;
        if (b == i)
            break;
        scored t = q->h[b];
        q->h[b] = q->h[i];
        q->h[i] = t;
        i = b;
    }
    return top;
}

static uint32_t g_adj(const or_graph* g, uint32_t lvl, uint32_t v, const uint32_t** nb) {
    const uint64_t* o = g->offsets + (size_t)lvl * (g->n + 1);
    *nb = g->nbrs + g->nbr_base[lvl] + o[v];
    return (uint32_t)(o[v + 1] - o[v]);
}

/* detail_search::descend_to_level0 (search.hpp:37-58). */
static scored g_descend(const or_graph* g, const or_index* lm, const float* q, or_counters* c) {
    uint32_t cur = g->entry;
    float cur_d = or_euclidean_sq(q, row_of(lm, cur), lm->dim);
    ++c->dc;
    ++c->evaluated;
    for (uint32_t lvl = g->levels - 1; lvl > 0; --lvl) {
        int changed = 1;
        while (changed) {
            changed = 0;
            const uint32_t* nb;
            const uint32_t deg = g_adj(g, lvl, cur, &nb);
            for (uint32_t i = 0; i < deg; ++i) {
                const uint32_t v = nb[i];
                const float d = or_euclidean_sq(q, row_of(lm, v), lm->dim);
                ++c->dc;
                ++c->evaluated;
                if (d < cur_d || (d == cur_d && v < cur)) {
                    cur_d = d;
                    cur = v;
                    changed = 1;
                }
            }
        }
    }
    scored r = {cur_d, cur};
    return r;
}

static float g_plb(const or_index* lm, const float* table, uint32_t v, float gamma) {
    const float glq = sqrtf(or_adc_lookup(table, lm->m, lm->ksub, lm->list_codes + (size_t)v * lm->code_stride));
    return or_relaxed_lb(glq, lm->list_lx[v], gamma);
}

/* The shared walk of search_trim_knn (range = 0, search.hpp:188-264) and
 * search_trim_range (range = 1, :267-347). kNN results in `res` (max-heap,
 * capacity k); range results appended to *rout. */
static int g_walk(const or_graph* g, const or_index* lm, const float* q, uint32_t k, uint32_t ef, float gamma,
                  int range, float radius_sq, gheap* res, gheap* rout, or_counters* ct) {
    const float kInf = INFINITY;
    float* table = (float*)malloc(sizeof(float) * lm->m * lm->ksub);
    char* visited = (char*)calloc(g->n, 1);
    gheap sq = {NULL, 0, 0, 0}, cand = {NULL, 0, 0, 1};
    int rc = OR_OK;
    if (!table || !visited) {
        rc = fail(OR_ENOMEM, "graph search: allocation failed");
        goto out;
    }
    or_build_distance_table(lm, q, table);
    const scored entry = g_descend(g, lm, q, ct);
    visited[entry.id] = 1;
    const float eplb = g_plb(lm, table, entry.id, gamma);
    ++ct->edc;
    scored se = {eplb, entry.id};
    if ((rc = gh_push(&sq, se)) || (rc = gh_push(&cand, entry)))
        goto out;
    if (!range) {
        if ((rc = gh_push(res, entry)))
            goto out;
    } else if (entry.d <= radius_sq) {
        if ((rc = gh_push(rout, entry)))
            goto out;
    }
    float max_dis = (!range && res->n == k) ? res->h[0].d : kInf;
    float max_can_dis = cand.n == ef ? cand.h[0].d : kInf;
    while (sq.n > 0) {
        const scored cur = gh_pop(&sq);
        if (cand.n == ef && cur.d > max_can_dis)
            break;
        ++ct->hops;
        const uint32_t* nb;
        const uint32_t deg = g_adj(g, 0, cur.id, &nb);
        for (uint32_t i = 0; i < deg; ++i) {
            const uint32_t v = nb[i];
            if (visited[v])
                continue;
            visited[v] = 1;
            ++ct->evaluated;
            const float plb = g_plb(lm, table, v, gamma);
            ++ct->edc;
            if (cand.n < ef || (range ? plb <= radius_sq : plb < max_dis)) {
                const float d = or_euclidean_sq(q, row_of(lm, v), lm->dim);
                ++ct->dc;
                scored sd = {d, v}, sp = {plb, v};
                if (range && d <= radius_sq && (rc = gh_push(rout, sd)))
                    goto out;
                if ((rc = gh_push(&sq, sp)) || (rc = gh_push(&cand, sd)))
                    goto out;
                if (cand.n > ef)
                    gh_pop(&cand);
                if (cand.n == ef)
                    max_can_dis = cand.h[0].d;
                if (!range) {
                    if ((rc = gh_push(res, sd)))
                        goto out;
                    if (res->n > k)
                        gh_pop(res);
                    if (res->n == k)
                        max_dis = res->h[0].d;
                }
            } else {
                ++ct->pruned;
                if (plb < max_can_dis) {
                    scored sp = {plb, v};
                    if ((rc = gh_push(&sq, sp)) || (rc = gh_push(&cand, sp)))
                        goto out;
                    if (cand.n > ef)
                        gh_pop(&cand);
                    if (cand.n == ef)
                        max_can_dis = cand.h[0].d;
                }
            }
        }
    }
out:
    free(table);
    free(visited);
    free(sq.h);
    free(cand.h);
    return rc;
}

int or_graph_search_trim_knn(const or_graph* g, const or_index* lm, const float* q, uint32_t k, uint32_t ef,
                             float gamma, uint32_t* ids, float* dist, uint64_t* nres, or_counters* ct) {
    if (k == 0 || k > ef)
        return fail(OR_EINVAL, "search_trim_knn: need 1 <= k <= ef");
    if (gamma < 0.0f)
        return fail(OR_EINVAL, "search_trim_knn: uncalibrated pruning profile");
    memset(ct, 0, sizeof *ct);
    gheap res = {NULL, 0, 0, 1};
    int rc = g_walk(g, lm, q, k, ef, gamma, 0, 0.0f, &res, NULL, ct);
    if (rc == OR_OK) { /* collect_sorted (search.hpp:62-80) */
        qsort(res.h, res.n, sizeof(scored), scored_cmp);
        for (uint64_t i = 0; i < res.n; ++i) {
            ids[i] = res.h[i].id;
            dist[i] = res.h[i].d;
        }
        *nres = res.n;
    }
    free(res.h);
    return rc;
}

int or_graph_search_trim_range(const or_graph* g, const or_index* lm, const float* q, float radius, uint32_t ef,
                               float gamma, uint32_t** ids, float** dist, uint64_t* count, or_counters* ct) {
    if (radius < 0.0f)
        return fail(OR_EINVAL, "search_trim_range: negative radius");
    if (gamma < 0.0f)
        return fail(OR_EINVAL, "search_trim_range: uncalibrated pruning profile");
    memset(ct, 0, sizeof *ct);
    gheap out = {NULL, 0, 0, 1};
    int rc = g_walk(g, lm, q, 0, ef, gamma, 1, radius * radius, NULL, &out, ct);
    *ids = NULL;
    *dist = NULL;
    *count = 0;
    if (rc == OR_OK) { /* std::sort(results) (search.hpp:336) */
        qsort(out.h, out.n, sizeof(scored), scored_cmp);
        *ids = (uint32_t*)malloc(sizeof(uint32_t) * (out.n ? out.n : 1));
        *dist = (float*)malloc(sizeof(float) * (out.n ? out.n : 1));
        for (uint64_t i = 0; i < out.n; ++i) {
            (*ids)[i] = out.h[i].id;
            (*dist)[i] = out.h[i].d;
        }
        *count = out.n;
    }
    free(out.h);
    return rc;
}

/* ---- query batches: static contiguous chunks per worker (parallel.hpp:31-56) ---- */
typedef struct {
    int kind;
    const or_index* ix;
    const float* qs;
    uint64_t begin, end;
    uint32_t k, nprobe, k_prime;
    float gamma;
    const float* radius;
    uint32_t* ids;
    float* dist;
    or_counters* ct;
    uint64_t* coarse_dc;
    /* range */
    uint32_t** rids;
    float** rdist;
    uint64_t* rcount;
    /* brute force */
    const float* data;
    uint64_t n;
    uint32_t dim;
    /* landmarks */
    uint8_t* codes;
    uint32_t code_stride;
    float* lx;
    /* graph */
    const or_graph* g;
    uint32_t ef;
    int rc;
    char err[512];
} job;

enum { J_KNN, J_RANGE, J_BASE, J_BF, J_LM, J_GKNN, J_GRANGE };

static int bf_knn(const float* data, uint64_t n, uint32_t dim, const float* q, uint32_t k,
                  uint32_t* ids, float* dist) {
    if (k == 0 || k > n)
        return fail(OR_EINVAL, "brute_force_knn: k out of range");
    scored* h = (scored*)malloc(sizeof(scored) * k);
    uint32_t hn = 0;
    for (uint64_t i = 0; i < n; ++i) {
        scored v = {or_euclidean_sq(q, data + i * dim, dim), (uint32_t)i};
        if (hn < k)
            heap_push(h, &hn, v);
        else if (scored_less(v, h[0]))
            heap_replace_top(h, hn, v);
    }
    qsort(h, hn, sizeof(scored), scored_cmp);
    for (uint32_t i = 0; i < hn; ++i) {
        ids[i] = h[i].id;
        dist[i] = h[i].d;
    }
    free(h);
    return OR_OK;
}

static void* run_job(void* arg) {
    job* j = (job*)arg;
    j->rc = OR_OK;
    for (uint64_t i = j->begin; i < j->end && j->rc == OR_OK; ++i) {
        const float* q = j->qs ? j->qs + i * (j->ix ? j->ix->dim : j->dim) : NULL;
        switch (j->kind) {
        case J_KNN:
            j->rc = or_search_trim_knn(j->ix, q, j->k, j->nprobe, j->gamma, j->ids + i * j->k,
                                       j->dist + i * j->k, j->ct + i, j->coarse_dc + i);
            break;
        case J_RANGE:
            j->rc = or_search_trim_range(j->ix, q, j->radius[i], j->nprobe, j->gamma, j->rids + i,
                                         j->rdist + i, j->rcount + i, j->ct + i,
                                         j->coarse_dc + i);
            break;
        case J_BASE: {
            uint64_t nres;
            j->rc = or_search_baseline_ivfpq(j->ix, q, j->k, j->nprobe, j->k_prime,
                                             j->ids + i * j->k, j->dist + i * j->k, &nres,
                                             j->ct + i, j->coarse_dc + i);
            break;
        }
        case J_BF:
            j->rc = bf_knn(j->data, j->n, j->dim, q, j->k, j->ids + i * j->k, j->dist + i * j->k);
            break;
        case J_GKNN: {
            uint64_t nres = 0;
            j->rc = or_graph_search_trim_knn(j->g, j->ix, q, j->k, j->ef, j->gamma, j->ids + i * j->k,
                                             j->dist + i * j->k, &nres, j->ct + i);
            for (uint64_t r = nres; r < j->k; ++r) {
                j->ids[i * j->k + r] = 0xFFFFFFFFu;
                j->dist[i * j->k + r] = INFINITY;
            }
            break;
        }
        case J_GRANGE:
            j->rc = or_graph_search_trim_range(j->g, j->ix, q, j->radius[i], j->ef, j->gamma, j->rids + i,
                                               j->rdist + i, j->rcount + i, j->ct + i);
            break;
        case J_LM:
            or_pq_encode(j->ix, j->data + i * j->ix->dim, j->codes + i * j->code_stride);
            j->lx[i] = or_landmark_dist(j->ix, j->data + i * j->ix->dim,
                                        j->codes + i * j->code_stride);
            break;
        }
    }
    if (j->rc != OR_OK)
        snprintf(j->err, sizeof j->err, "%s", g_err);
    return NULL;
}

static int run_parallel(job* proto, uint64_t n, int threads) {
    if (n == 0)
        return OR_OK;
    if (threads < 1)
        threads = 1;
    if ((uint64_t)threads > n)
        threads = (int)n;
    job* jobs = (job*)calloc((size_t)threads, sizeof(job));
    pthread_t* tids = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
    const uint64_t chunk = (n + (uint64_t)threads - 1) / (uint64_t)threads;
    int used = 0;
    for (int w = 0; w < threads; ++w) {
        const uint64_t b = (uint64_t)w * chunk;
        const uint64_t e = b + chunk < n ? b + chunk : n;
        if (b >= e)
            break;
        jobs[w] = *proto;
        jobs[w].begin = b;
        jobs[w].end = e;
        if (threads == 1)
            run_job(&jobs[w]);
        else
            pthread_create(&tids[w], NULL, run_job, &jobs[w]);
        ++used;
    }
    int rc = OR_OK;
    for (int w = 0; w < used; ++w) {
        if (threads != 1)
            pthread_join(tids[w], NULL);
        if (jobs[w].rc != OR_OK && rc == OR_OK) {
            rc = jobs[w].rc;
            snprintf(g_err, sizeof g_err, "%s", jobs[w].err);
        }
    }
    free(jobs);
    free(tids);
    return rc;
}

int or_search_trim_knn_batch(const or_index* ix, const float* qs, uint64_t nq, uint32_t k,
                             uint32_t nprobe, float gamma, uint32_t* ids_out, float* dist_out,
                             or_counters* counters, uint64_t* coarse_dc, int threads) {
    job p;
    memset(&p, 0, sizeof p);
    p.kind = J_KNN;
    p.ix = ix;
    p.qs = qs;
    p.k = k;
    p.nprobe = nprobe;
    p.gamma = gamma;
    p.ids = ids_out;
    p.dist = dist_out;
    p.ct = counters;
    p.coarse_dc = coarse_dc;
    return run_parallel(&p, nq, threads);
}

int or_search_trim_range_batch(const or_index* ix, const float* qs, uint64_t nq,
                               const float* radius, uint32_t nprobe, float gamma,
                               uint64_t* offsets_out, uint32_t** ids_out, float** dist_out,
                               or_counters* counters, uint64_t* coarse_dc, int threads) {
    uint32_t** rids = (uint32_t**)calloc(nq ? nq : 1, sizeof(uint32_t*));
    float** rdist = (float**)calloc(nq ? nq : 1, sizeof(float*));
    uint64_t* rcount = (uint64_t*)calloc(nq ? nq : 1, sizeof(uint64_t));
    job p;
    memset(&p, 0, sizeof p);
    p.kind = J_RANGE;
    p.ix = ix;
    p.qs = qs;
    p.nprobe = nprobe;
    p.gamma = gamma;
    p.radius = radius;
    p.ct = counters;
    p.coarse_dc = coarse_dc;
    p.rids = rids;
    p.rdist = rdist;
    p.rcount = rcount;
    int rc = run_parallel(&p, nq, threads);
    if (rc == OR_OK) {
        uint64_t tot = 0;
        offsets_out[0] = 0;
        for (uint64_t i = 0; i < nq; ++i) {
            tot += rcount[i];
            offsets_out[i + 1] = tot;
        }
        uint32_t* ids = (uint32_t*)malloc(sizeof(uint32_t) * (tot ? tot : 1));
        float* ds = (float*)malloc(sizeof(float) * (tot ? tot : 1));
        for (uint64_t i = 0; i < nq; ++i) {
            memcpy(ids + offsets_out[i], rids[i], sizeof(uint32_t) * rcount[i]);
            memcpy(ds + offsets_out[i], rdist[i], sizeof(float) * rcount[i]);
        }
        *ids_out = ids;
        *dist_out = ds;
    }
    for (uint64_t i = 0; i < nq; ++i) {
        free(rids[i]);
        free(rdist[i]);
    }
    free(rids);
    free(rdist);
    free(rcount);
    return rc;
}

int or_search_baseline_ivfpq_batch(const or_index* ix, const float* qs, uint64_t nq, uint32_t k,
                                   uint32_t nprobe, uint32_t k_prime, uint32_t* ids_out,
                                   float* dist_out, or_counters* counters, uint64_t* coarse_dc,
                                   int threads) {
    job p;
    memset(&p, 0, sizeof p);
    p.kind = J_BASE;
    p.ix = ix;
    p.qs = qs;
    p.k = k;
    p.nprobe = nprobe;
    p.k_prime = k_prime;
    p.ids = ids_out;
    p.dist = dist_out;
    p.ct = counters;
    p.coarse_dc = coarse_dc;
    return run_parallel(&p, nq, threads);
}

int or_build_landmarks(const or_index* ix, const float* data, uint64_t n, uint8_t* codes,
                       uint32_t code_stride, float* lx, int threads) {
    job p;
    memset(&p, 0, sizeof p);
    p.kind = J_LM;
    p.ix = ix;
    p.data = data;
    p.codes = codes;
    p.code_stride = code_stride;
    p.lx = lx;
    return run_parallel(&p, n, threads);
}

int or_brute_force_knn_batch(const float* data, uint64_t n, uint32_t dim, const float* qs,
                             uint64_t nq, uint32_t k, uint32_t* ids_out, float* dist_out,
                             int threads) {
    job p;
    memset(&p, 0, sizeof p);
    p.kind = J_BF;
    p.qs = qs;
    p.data = data;
    p.n = n;
    p.dim = dim;
    p.k = k;
    p.ids = ids_out;
    p.dist = dist_out;
    return run_parallel(&p, nq, threads);
}

int or_graph_search_trim_knn_batch(const or_graph* g, const or_index* lm, const float* qs, uint64_t nq,
                                   uint32_t k, uint32_t ef, float gamma, uint32_t* ids_out, float* dist_out,
                                   or_counters* counters, int threads) {
    job p;
    memset(&p, 0, sizeof p);
    p.kind = J_GKNN;
    p.g = g;
    p.ix = lm;
    p.qs = qs;
    p.k = k;
    p.ef = ef;
    p.gamma = gamma;
    p.ids = ids_out;
    p.dist = dist_out;
    p.ct = counters;
    return run_parallel(&p, nq, threads);
}

int or_graph_search_trim_range_batch(const or_graph* g, const or_index* lm, const float* qs, uint64_t nq,
                                     const float* radius, uint32_t ef, float gamma, uint64_t* offsets_out,
                                     uint32_t** ids_out, float** dist_out, or_counters* counters, int threads) {
    uint32_t** rids = (uint32_t**)calloc(nq ? nq : 1, sizeof(uint32_t*));
    float** rdist = (float**)calloc(nq ? nq : 1, sizeof(float*));
    uint64_t* rcount = (uint64_t*)calloc(nq ? nq : 1, sizeof(uint64_t));
    job p;
    memset(&p, 0, sizeof p);
    p.kind = J_GRANGE;
    p.g = g;
    p.ix = lm;
    p.qs = qs;
    p.ef = ef;
    p.gamma = gamma;
    p.radius = radius;
    p.ct = counters;
    p.rids = rids;
    p.rdist = rdist;
    p.rcount = rcount;
    int rc = run_parallel(&p, nq, threads);
    uint64_t tot = 0;
    offsets_out[0] = 0;
    for (uint64_t i = 0; i < nq; ++i) {
        tot += rcount[i];
        offsets_out[i + 1] = tot;
    }
    *ids_out = (uint32_t*)malloc(sizeof(uint32_t) * (tot ? tot : 1));
    *dist_out = (float*)malloc(sizeof(float) * (tot ? tot : 1));
    for (uint64_t i = 0; i < nq; ++i) {
        if (rcount[i]) {
            memcpy(*ids_out + offsets_out[i], rids[i], sizeof(uint32_t) * rcount[i]);
            memcpy(*dist_out + offsets_out[i], rdist[i], sizeof(float) * rcount[i]);
        }
        free(rids[i]);
        free(rdist[i]);
    }
    free(rids);
    free(rdist);
    free(rcount);
    return rc;
}
