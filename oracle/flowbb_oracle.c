/*
 * flowbb_oracle.c -- CPU restatement of the reference flowbb hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see flowbb_oracle.h).  Plain C, single thread,
 * written for clarity, not speed: each function follows the cited reference
 * function step by step, including std::stable_sort's order in Johnson's rule.
 * Citations are relative to the reference's proj/include/flowbb/.
 */
#include "flowbb_oracle.h"

#include <limits.h>
#include <stdlib.h>
#include <string.h>

#define W_OF(n) (((n) + 63) / 64)

static int mask_test(const uint64_t* mask, int j) { return (int)((mask[j >> 6] >> (j & 63)) & 1u); }
static void mask_set(uint64_t* mask, int j) { mask[j >> 6] |= (uint64_t)1 << (j & 63); }

/* instance.hpp:227-265: Lehmer LCG (16807, 2^31-1) with Schrage's split, the
 * draw low + (int)(u * (high-low+1)) with u = state / m in double. */
int orc_generate_instance(int n, int m, int32_t seed, int32_t* p_out) {
    if (seed <= 0 || seed >= 2147483647) return -1;
    int64_t state = seed;
    const int64_t M = 2147483647, A = 16807, Q = 127773, R = 2836;
    for (int k = 0; k < m; ++k) {
        for (int j = 0; j < n; ++j) {
            int64_t kq = state / Q;
            state = A * (state % Q) - R * kq;
            if (state < 0) state += M;
            double u = (double)state / (double)M;
            p_out[(int64_t)j * m + k] = 1 + (int32_t)(u * 99.0);
        }
    }
    return 0;
}

/* instance.hpp:38-45 */
void orc_tails(int n, int m, const int32_t* p, int32_t* tails) {
    for (int j = 0; j < n; ++j) {
        int32_t acc = 0;
        for (int k = m - 1; k >= 0; --k) {
            tails[j * m + k] = acc;
            acc += p[j * m + k];
        }
    }
}

/* instance.hpp:81-89: r'[k] = max(r'[k-1], r[k]) + p[job][k]. */
void orc_child_heads(int n, int m, const int32_t* p, const int32_t* heads, int job,
                     int32_t* out) {
    (void)n;
    int32_t prev = 0;
    for (int k = 0; k < m; ++k) {
        int32_t h = heads[k] > prev ? heads[k] : prev;
        prev = h + p[job * m + k];
        out[k] = prev;
    }
}

/* instance.hpp:92-96 */
int32_t orc_makespan(int n, int m, const int32_t* p, const int32_t* perm, int len) {
    int32_t* h = (int32_t*)calloc((size_t)m, sizeof(int32_t));
    int32_t* t = (int32_t*)malloc((size_t)m * sizeof(int32_t));
    for (int i = 0; i < len; ++i) {
        orc_child_heads(n, m, p, h, perm[i], t);
        memcpy(h, t, (size_t)m * sizeof(int32_t));
    }
    int32_t v = h[m - 1];
    free(h);
    free(t);
    return v;
}

/* bound.hpp:27-44.  std::stable_sort with the comparator
 *   first-group (a+lag < lag+b) before second; first group ascending a+lag;
 *   second group descending lag+b; ties keep input order
 * is restated as a sort on the key (group, key, input index), which is the
 * same total order a stable sort produces.  Insertion sort keeps it obvious. */
int32_t orc_johnson_two_machine(const int32_t* a, const int32_t* lag, const int32_t* b,
                                int count, int32_t release_a, int32_t release_b) {
    int order_buf[1024];
    int* order = count <= 1024 ? order_buf : (int*)malloc((size_t)count * sizeof(int));
    for (int i = 0; i < count; ++i) order[i] = i;
#define IN_FIRST(i) (a[i] + lag[i] < lag[i] + b[i])
#define BEFORE(i, j)                                                                   \
    (IN_FIRST(i) != IN_FIRST(j) ? IN_FIRST(i)                                          \
     : IN_FIRST(i)              ? (a[i] + lag[i] < a[j] + lag[j])                      \
                                : (lag[i] + b[i] > lag[j] + b[j]))
    for (int s = 1; s < count; ++s) {
        int v = order[s];
        int t = s - 1;
        /* move v left past every element it strictly precedes (stability) */
        while (t >= 0 && BEFORE(v, order[t])) {
            order[t + 1] = order[t];
            --t;
        }
        order[t + 1] = v;
    }
#undef BEFORE
#undef IN_FIRST
    int32_t t_a = release_a, t_b = release_b;
    for (int s = 0; s < count; ++s) {
        int i = order[s];
        t_a += a[i];
        int32_t x = t_a + lag[i];
        t_b = (t_b > x ? t_b : x) + b[i];
    }
    if (order != order_buf) free(order);
    return t_b;
}

/* bound.hpp:61-74 (tails precomputed once, as Instance does) */
static int32_t lb_one_machine_t(int n, int m, const int32_t* p, const int32_t* tails,
                                const uint64_t* mask, const int32_t* heads) {
    int32_t best = 0;
    for (int k = 0; k < m; ++k) {
        int32_t load = 0, min_tail = INT_MAX;
        for (int j = 0; j < n; ++j) {
            if (mask_test(mask, j)) continue; /* unscheduled_jobs, bound.hpp:49-55 */
            load += p[j * m + k];
            if (tails[j * m + k] < min_tail) min_tail = tails[j * m + k];
        }
        int32_t v = heads[k] + load + min_tail;
        if (v > best) best = v;
    }
    return best;
}

/* bound.hpp:79-90 (scratch: 3n ints) */
static int32_t lb_machine_pair_t(int n, int m, const int32_t* p, const int32_t* tails,
                                 const uint64_t* mask, const int32_t* heads, int k, int l,
                                 int32_t* scratch) {
    int32_t* a = scratch;
    int32_t* lag = scratch + n;
    int32_t* b = scratch + 2 * n;
    int cnt = 0;
    int32_t min_tail = INT_MAX;
    for (int j = 0; j < n; ++j) {
        if (mask_test(mask, j)) continue;
        a[cnt] = p[j * m + k];
        lag[cnt] = tails[j * m + k] - p[j * m + l] - tails[j * m + l];
        b[cnt] = p[j * m + l];
        ++cnt;
        if (tails[j * m + l] < min_tail) min_tail = tails[j * m + l];
    }
    return orc_johnson_two_machine(a, lag, b, cnt, heads[k], heads[l]) + min_tail;
}

/* bound.hpp:94-101 */
static int32_t lower_bound_t(int n, int m, const int32_t* p, const int32_t* tails,
                             const uint64_t* mask, const int32_t* heads, int depth,
                             int32_t* scratch) {
    if (depth == n) return heads[m - 1];
    int32_t best = lb_one_machine_t(n, m, p, tails, mask, heads);
    for (int k = 0; k < m; ++k)
        for (int l = k + 1; l < m; ++l) {
            int32_t v = lb_machine_pair_t(n, m, p, tails, mask, heads, k, l, scratch);
            if (v > best) best = v;
        }
    return best;
}

int32_t orc_lb_one_machine(int n, int m, const int32_t* p, const uint64_t* mask,
                           const int32_t* heads) {
    int32_t* tails = (int32_t*)malloc((size_t)n * m * sizeof(int32_t));
    orc_tails(n, m, p, tails);
    int32_t v = lb_one_machine_t(n, m, p, tails, mask, heads);
    free(tails);
    return v;
}

int32_t orc_lb_machine_pair(int n, int m, const int32_t* p, const uint64_t* mask,
                            const int32_t* heads, int k, int l) {
    int32_t* tails = (int32_t*)malloc((size_t)n * m * sizeof(int32_t));
    int32_t* scratch = (int32_t*)malloc((size_t)3 * n * sizeof(int32_t));
    orc_tails(n, m, p, tails);
    int32_t v = lb_machine_pair_t(n, m, p, tails, mask, heads, k, l, scratch);
    free(scratch);
    free(tails);
    return v;
}

int32_t orc_lower_bound(int n, int m, const int32_t* p, const uint64_t* mask,
                        const int32_t* heads, int depth) {
    int32_t* tails = (int32_t*)malloc((size_t)n * m * sizeof(int32_t));
    int32_t* scratch = (int32_t*)malloc((size_t)3 * n * sizeof(int32_t));
    orc_tails(n, m, p, tails);
    int32_t v = lower_bound_t(n, m, p, tails, mask, heads, depth, scratch);
    free(scratch);
    free(tails);
    return v;
}

/* bound.hpp:104-109 */
void orc_evaluate_batch(int n, int m, const int32_t* p, int64_t count, const uint64_t* masks,
                        const int32_t* heads, const int32_t* depth, int32_t* lb_out) {
    const int W = W_OF(n);
    int32_t* tails = (int32_t*)malloc((size_t)n * m * sizeof(int32_t));
    int32_t* scratch = (int32_t*)malloc((size_t)3 * n * sizeof(int32_t));
    orc_tails(n, m, p, tails);
    for (int64_t i = 0; i < count; ++i)
        lb_out[i] = lower_bound_t(n, m, p, tails, masks + i * W, heads + i * m, depth[i], scratch);
    free(scratch);
    free(tails);
}

/* node.hpp:37-52: root, then child() per prefix entry. */
void orc_node_from_prefix(int n, int m, const int32_t* p, const int32_t* prefix, int depth,
                          uint64_t* mask, int32_t* heads) {
    const int W = W_OF(n);
    memset(mask, 0, (size_t)W * sizeof(uint64_t));
    memset(heads, 0, (size_t)m * sizeof(int32_t));
    int32_t* t = (int32_t*)malloc((size_t)m * sizeof(int32_t));
    for (int i = 0; i < depth; ++i) {
        mask_set(mask, prefix[i]);
        orc_child_heads(n, m, p, heads, prefix[i], t);
        memcpy(heads, t, (size_t)m * sizeof(int32_t));
    }
    free(t);
}

/* search.hpp:40-59 */
int orc_branch(int n, int m, const int32_t* p, const int32_t* prefix, int depth,
               int32_t* cprefix, uint64_t* cmask, int32_t* cheads, int32_t* cdepth) {
    if (depth >= n) return -1;
    const int W = W_OF(n);
    uint64_t* mask = (uint64_t*)malloc((size_t)W * sizeof(uint64_t));
    int32_t* heads = (int32_t*)malloc((size_t)m * sizeof(int32_t));
    orc_node_from_prefix(n, m, p, prefix, depth, mask, heads);
    int c = 0;
    for (int j = 0; j < n; ++j) {
        if (mask_test(mask, j)) continue;
        int32_t* pr = cprefix + (int64_t)c * n;
        uint64_t* mk = cmask + (int64_t)c * W;
        int32_t* hd = cheads + (int64_t)c * m;
        memcpy(pr, prefix, (size_t)depth * sizeof(int32_t));
        memcpy(mk, mask, (size_t)W * sizeof(uint64_t));
        pr[depth] = j;
        mask_set(mk, j);
        orc_child_heads(n, m, p, heads, j, hd);
        int d = depth + 1;
        if (d == n - 1) { /* auto-complete with the unique remaining job */
            for (int last = 0; last < n; ++last) {
                if (!mask_test(mk, last)) {
                    int32_t* t = (int32_t*)malloc((size_t)m * sizeof(int32_t));
                    orc_child_heads(n, m, p, hd, last, t);
                    memcpy(hd, t, (size_t)m * sizeof(int32_t));
                    free(t);
                    pr[d] = last;
                    mask_set(mk, last);
                    ++d;
                    break;
                }
            }
        }
        cdepth[c] = d;
        ++c;
    }
    free(mask);
    free(heads);
    return c;
}

/* ---------------------------------------------------------------------------
 * Explorer restatement: PendingTree (pending.hpp:13-56), fill_buffer
 * (search.hpp:64-73), integrate (search.hpp:84-107), solve (search.hpp:124-174)
 * and the frozen resolve loop (bench.hpp:63-114).
 * ------------------------------------------------------------------------- */

typedef struct {
    int n, m, W;
    int32_t* prefix; /* cap x n */
    uint64_t* mask;  /* cap x W */
    int32_t* heads;  /* cap x m */
    int64_t size, cap;
} nodevec;

static void nv_init(nodevec* v, int n, int m) {
    memset(v, 0, sizeof(*v));
    v->n = n;
    v->m = m;
    v->W = W_OF(n);
}
static void nv_free(nodevec* v) {
    free(v->prefix);
    free(v->mask);
    free(v->heads);
    memset(v, 0, sizeof(*v));
}
static void nv_reserve(nodevec* v, int64_t cap) {
    if (cap <= v->cap) return;
    int64_t c = v->cap ? v->cap : 16;
    while (c < cap) c *= 2;
    v->prefix = (int32_t*)realloc(v->prefix, (size_t)c * v->n * sizeof(int32_t));
    v->mask = (uint64_t*)realloc(v->mask, (size_t)c * v->W * sizeof(uint64_t));
    v->heads = (int32_t*)realloc(v->heads, (size_t)c * v->m * sizeof(int32_t));
    v->cap = c;
}
static void nv_push(nodevec* v, const int32_t* prefix, const uint64_t* mask,
                    const int32_t* heads) {
    nv_reserve(v, v->size + 1);
    memcpy(v->prefix + v->size * v->n, prefix, (size_t)v->n * sizeof(int32_t));
    memcpy(v->mask + v->size * v->W, mask, (size_t)v->W * sizeof(uint64_t));
    memcpy(v->heads + v->size * v->m, heads, (size_t)v->m * sizeof(int32_t));
    v->size++;
}

/* pending.hpp:13-50: buckets by depth, deepest first, LIFO within a bucket. */
typedef struct {
    int maxd;
    nodevec* b;
    int64_t count;
    int deepest;
} pendtree;

static void pt_init(pendtree* t, int n, int m) {
    t->maxd = n;
    t->b = (nodevec*)malloc((size_t)(n + 1) * sizeof(nodevec));
    for (int d = 0; d <= n; ++d) nv_init(&t->b[d], n, m);
    t->count = 0;
    t->deepest = 0;
}
static void pt_free(pendtree* t) {
    for (int d = 0; d <= t->maxd; ++d) nv_free(&t->b[d]);
    free(t->b);
}
static void pt_push(pendtree* t, int depth, const int32_t* prefix, const uint64_t* mask,
                    const int32_t* heads) {
    nv_push(&t->b[depth], prefix, mask, heads);
    if (depth > t->deepest) t->deepest = depth;
    t->count++;
}
/* pop into out (prefix n ints); returns depth. */
static int pt_pop(pendtree* t, int32_t* prefix) {
    while (t->b[t->deepest].size == 0) --t->deepest;
    nodevec* v = &t->b[t->deepest];
    v->size--;
    memcpy(prefix, v->prefix + v->size * v->n, (size_t)v->n * sizeof(int32_t));
    t->count--;
    return t->deepest;
}

/* search.hpp:64-73: pop deepest and branch until size >= target. */
static int64_t fill_buffer(int n, int m, const int32_t* p, pendtree* pend, int64_t target,
                           nodevec* batch, int32_t** bdepth, int64_t* bdepth_cap,
                           int64_t* branched) {
    const int W = W_OF(n);
    batch->size = 0;
    int32_t* pr = (int32_t*)malloc((size_t)n * sizeof(int32_t));
    int32_t* cpre = (int32_t*)malloc((size_t)n * n * sizeof(int32_t));
    uint64_t* cmask = (uint64_t*)malloc((size_t)n * W * sizeof(uint64_t));
    int32_t* chead = (int32_t*)malloc((size_t)n * m * sizeof(int32_t));
    int32_t* cdep = (int32_t*)malloc((size_t)n * sizeof(int32_t));
    while (batch->size < target && pend->count > 0) {
        int d = pt_pop(pend, pr);
        ++*branched;
        int c = orc_branch(n, m, p, pr, d, cpre, cmask, chead, cdep);
        for (int i = 0; i < c; ++i) {
            if (batch->size + 1 > *bdepth_cap) {
                *bdepth_cap = (*bdepth_cap ? *bdepth_cap : 16) * 2;
                *bdepth = (int32_t*)realloc(*bdepth, (size_t)*bdepth_cap * sizeof(int32_t));
            }
            (*bdepth)[batch->size] = cdep[i];
            nv_push(batch, cpre + (int64_t)i * n, cmask + (int64_t)i * W, chead + (int64_t)i * m);
        }
    }
    free(pr);
    free(cpre);
    free(cmask);
    free(chead);
    free(cdep);
    return batch->size;
}

static int64_t target_at(const int64_t* targets, int ntargets, int64_t r) {
    if (ntargets <= 0) return 1;
    return targets[r < ntargets ? r : ntargets - 1];
}

static void trace_put(orc_round* trace, int64_t max_trace, int64_t r, const orc_round* rec) {
    if (trace && r < max_trace) trace[r] = *rec;
}

/* search.hpp:124-174 (with search.hpp:84-107 integrate inlined) */
int orc_solve(int n, int m, const int32_t* p, int32_t initial_ub, const int64_t* targets,
              int ntargets, int64_t budget, orc_result* res, int32_t* schedule_out,
              orc_round* trace, int64_t max_trace) {
    const int W = W_OF(n);
    memset(res, 0, sizeof(*res));
    int32_t* tails = (int32_t*)malloc((size_t)n * m * sizeof(int32_t));
    int32_t* scratch = (int32_t*)malloc((size_t)3 * n * sizeof(int32_t));
    orc_tails(n, m, p, tails);
    int32_t inc;
    int found = 0;
    if (initial_ub >= 0) {
        inc = initial_ub;
    } else { /* identity permutation, search.hpp:131-137 */
        int32_t* id = (int32_t*)malloc((size_t)n * sizeof(int32_t));
        for (int j = 0; j < n; ++j) id[j] = j;
        inc = orc_makespan(n, m, p, id, n);
        if (schedule_out) memcpy(schedule_out, id, (size_t)n * sizeof(int32_t));
        found = 1;
        free(id);
    }
    pendtree pend;
    pt_init(&pend, n, m);
    nodevec batch;
    nv_init(&batch, n, m);
    int32_t* bdepth = NULL;
    int64_t bdcap = 0;
    /* batch = {root} */
    {
        int32_t* pr = (int32_t*)calloc((size_t)n, sizeof(int32_t));
        uint64_t* mk = (uint64_t*)calloc((size_t)W, sizeof(uint64_t));
        int32_t* hd = (int32_t*)calloc((size_t)m, sizeof(int32_t));
        nv_push(&batch, pr, mk, hd);
        bdcap = 16;
        bdepth = (int32_t*)malloc((size_t)bdcap * sizeof(int32_t));
        bdepth[0] = 0;
        free(pr);
        free(mk);
        free(hd);
    }
    int64_t r = 0, target = 0, branched_round = 0;
    while (batch.size > 0) {
        orc_round rec;
        memset(&rec, 0, sizeof(rec));
        rec.target = target;
        rec.branched = branched_round;
        rec.bounded = batch.size;
        res->bounded += batch.size;
        for (int64_t i = 0; i < batch.size; ++i) {
            const uint64_t* mk = batch.mask + i * W;
            const int32_t* hd = batch.heads + i * m;
            int32_t lb = lower_bound_t(n, m, p, tails, mk, hd, bdepth[i], scratch);
            if (bdepth[i] == n) {
                rec.leaves++;
                if (lb < inc) {
                    inc = lb;
                    found = 1;
                    if (schedule_out)
                        memcpy(schedule_out, batch.prefix + i * n, (size_t)n * sizeof(int32_t));
                }
            } else if (lb < inc) {
                rec.inserted++;
                pt_push(&pend, bdepth[i], batch.prefix + i * n, mk, hd);
            } else {
                rec.pruned++;
            }
        }
        res->pruned += rec.pruned;
        res->leaves += rec.leaves;
        rec.incumbent = inc;
        rec.pending = pend.count;
        trace_put(trace, max_trace, r, &rec);
        ++r;
        if (pend.count == 0) break;
        if (budget > 0 && res->bounded >= budget) break;
        target = target_at(targets, ntargets, r - 1);
        int64_t before = res->branched;
        fill_buffer(n, m, p, &pend, target, &batch, &bdepth, &bdcap, &res->branched);
        branched_round = res->branched - before;
    }
    res->rounds = r;
    res->optimum = inc;
    res->found = found;
    res->pending = pend.count;
    free(bdepth);
    nv_free(&batch);
    pt_free(&pend);
    free(tails);
    free(scratch);
    return 0;
}

/* bench.hpp:63-114 (frozen incumbent; warm-up evaluate has no effect on the
 * explored set and is omitted) */
int orc_resolve(int n, int m, const int32_t* p, int32_t ub, int64_t nroots,
                const int32_t* roots_prefix, const int32_t* roots_depth, const int64_t* targets,
                int ntargets, int64_t budget, orc_result* res, orc_round* trace,
                int64_t max_trace) {
    const int W = W_OF(n);
    memset(res, 0, sizeof(*res));
    res->optimum = -1;
    int32_t* tails = (int32_t*)malloc((size_t)n * m * sizeof(int32_t));
    int32_t* scratch = (int32_t*)malloc((size_t)3 * n * sizeof(int32_t));
    orc_tails(n, m, p, tails);
    pendtree pend;
    pt_init(&pend, n, m);
    uint64_t* mk = (uint64_t*)malloc((size_t)W * sizeof(uint64_t));
    int32_t* hd = (int32_t*)malloc((size_t)m * sizeof(int32_t));
    for (int64_t i = 0; i < nroots; ++i) {
        orc_node_from_prefix(n, m, p, roots_prefix + i * n, roots_depth[i], mk, hd);
        pt_push(&pend, roots_depth[i], roots_prefix + i * n, mk, hd);
    }
    free(mk);
    free(hd);
    nodevec batch;
    nv_init(&batch, n, m);
    int32_t* bdepth = NULL;
    int64_t bdcap = 0;
    int64_t r = 0;
    while (pend.count > 0) {
        orc_round rec;
        memset(&rec, 0, sizeof(rec));
        int64_t target = target_at(targets, ntargets, r);
        rec.target = target;
        int64_t before = res->branched;
        fill_buffer(n, m, p, &pend, target, &batch, &bdepth, &bdcap, &res->branched);
        rec.branched = res->branched - before;
        rec.bounded = batch.size;
        res->bounded += batch.size;
        for (int64_t i = 0; i < batch.size; ++i) {
            const uint64_t* bm = batch.mask + i * W;
            const int32_t* bh = batch.heads + i * m;
            int32_t lb = lower_bound_t(n, m, p, tails, bm, bh, bdepth[i], scratch);
            if (bdepth[i] == n) {
                rec.leaves++;
                if (lb < ub && (!res->found || lb < res->optimum)) {
                    res->optimum = lb;
                    res->found = 1;
                }
            } else if (lb < ub) {
                rec.inserted++;
                pt_push(&pend, bdepth[i], batch.prefix + i * n, bm, bh);
            } else {
                rec.pruned++;
            }
        }
        res->pruned += rec.pruned;
        res->leaves += rec.leaves;
        rec.incumbent = res->found ? res->optimum : ub;
        rec.pending = pend.count;
        trace_put(trace, max_trace, r, &rec);
        ++r;
        if (budget > 0 && res->bounded >= budget) break;
    }
    res->rounds = r;
    res->pending = pend.count;
    free(bdepth);
    nv_free(&batch);
    pt_free(&pend);
    free(tails);
    free(scratch);
    return 0;
}
