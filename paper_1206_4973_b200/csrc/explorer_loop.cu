// explorer_loop.cu -- the explorer round planned and closed on the device, so that a
// batch of rounds runs back to back without the host (fbb_explorer_run).
//
//   step  (1 warp)     closes the previous round, then plans this one:
//   plan               fill_buffer (search.hpp:64-73) on the bucket sizes: pop the
//                      deepest bucket tops, LIFO, until the children reach the target;
//                      lay out segments and chunks exactly as the host planner does
//                      (capi.cu layout_pool); point each segment at its source and
//                      destination buckets; reset the round state.
//   round              leaves, leaf schedule, K2, place (expand_kernel.cu)
//   close              integrate / frozen prune bookkeeping (search.hpp:84-107,
//                      bench.hpp:96-106): bucket sizes, incumbent and schedule, the
//                      round's counters, stop conditions (empty tree, node budget).
// A round whose destination bucket is too small is not started: the batch stops with
// stop = 3 and the host grows that bucket and resumes, so device buckets never
// reallocate inside a batch.
#include "fbb_internal.h"

namespace fbb {

namespace {

__device__ __forceinline__ unsigned long long loop_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// plan of round `round` (thread 0; cnt = the block's shared copy of the bucket sizes)
__device__ void plan_round(const DevTables& t, LoopState* ls, Pool* pool, RoundState* rs, int round,
                           const int64_t* cnt) {
    if (round < kLoopMax) ls->rec[round].t0 = loop_ns();
    const int n = t.n;
    pool->nseg = 0;
    pool->nchunks = 0;
    pool->nchildren = 0;
    rs->leaf_inv = 0ull;
    rs->found = 0;
    rs->ticket = 0u;
    rs->total = 0;
    rs->place_done = 0u;
    rs->arrived = 0u;
    rs->k2_t0_inv = 0ull;
    rs->k2_t1 = 0ull;
    pool->ub = ls->incumbent;
    pool->frozen = ls->frozen;
    pool->first_internal = 0;
    if (ls->stop || round >= ls->nrounds) return;
    const int64_t target = ls->targets[round] < 1 ? 1 : ls->targets[round];
    // fill_buffer on the sizes (deepest bucket first, LIFO, until >= target)
    int64_t have = 0;
    int nseg = 0;
    for (int d = n; d >= 0 && have < target; --d) {
        const int64_t c = cnt[d];
        if (c == 0) continue;
        const int r = n - d;
        const int64_t k = min(c, (target - have + r - 1) / r);
        Segment& sg = pool->seg[nseg++];
        sg.src = ls->bucket[d];
        sg.first = c - 1;
        sg.step = -1;
        sg.count = k;
        sg.depth = d;
        sg.pad = 0;
        sg.dst_lb = nullptr;
        have += k * r;
    }
    if (nseg == 0) {
        ls->stop = 1;
        return;
    }
    // destinations: bucket d+1 after this round's pops; all sizes checked first
    for (int s = 0; s < nseg; ++s) {
        Segment& sg = pool->seg[s];
        const int d = sg.depth;
        if (d >= n - 2) {
            sg.dst = NodeStore{nullptr, nullptr, nullptr};
            sg.dst_base = 0;
            continue;
        }
        int64_t after = cnt[d + 1];
        for (int s2 = 0; s2 < s; ++s2)
            if (pool->seg[s2].depth == d + 1) after -= pool->seg[s2].count;
        const int64_t worst = after + sg.count * (n - d);
        if (worst > ls->cap[d + 1]) {
            ls->stop = 3;
            ls->need_depth = d + 1;
            ls->need_rows = worst;
            return;  // nseg stays 0: nothing of this round runs
        }
        sg.dst = ls->bucket[d + 1];
        sg.dst_base = after;
    }
    // chunk layout (capi.cu layout_pool)
    const int cmax = ls->cmax;
    int64_t child = 0, chunk = 0;
    int first_internal = nseg;
    const int ppc_lim = spread_ppc(pool->seg, nseg, n, cmax, ls->ppc_cap, ls->spread_blocks);
    const int cap = round_ppc_cap(ls->ppc_cap, ppc_lim);
    for (int s = 0; s < nseg; ++s) {
        Segment& sg = pool->seg[s];
        const int r = n - sg.depth;
        sg.child_base = child;
        child += sg.count * r;
        sg.chunk_base = chunk;
        if (sg.depth >= n - 2) continue;
        if (first_internal == nseg) first_internal = s;
        const int ppc = parents_per_chunk(n, sg.depth, cmax, cap);
        chunk += (sg.count + ppc - 1) / ppc;
    }
    if (chunk > ls->chunk_cap) {  // the host sized staging for the worst case: never taken
        ls->stop = 5;
        return;  // nseg stays 0: nothing of this round runs
    }
    for (int s = 0; s < nseg; ++s) rs->seg_surv[s] = 0;
    pool->first_internal = first_internal;
    pool->nchunks = chunk;
    pool->nchildren = child;
    pool->pad = 0;
    pool->host_dst = ls->host_dst;
    // single-wave pools: K2 places the survivors itself (capi.cu run_pool, same rule)
    pool->direct = (ls->direct_cap > 0 && chunk > 0 && chunk <= ls->direct_cap) ? 1 : 0;
    pool->ppc_lim = ppc_lim;
    pool->summary = nullptr;
    pool->nseg = nseg;
}

// integrate bookkeeping of round `round` (thread 0; updates the shared bucket sizes)
__device__ void close_round(const DevTables& t, LoopState* ls, const Pool* pool, const RoundState* rs,
                            int round, int64_t* cnt) {
    const int n = t.n;
    LoopRecord& rec = ls->rec[round];
    rec.valid = 0;
    if (pool->nseg == 0) return;  // stopped before this round
    rec.k2_t0 = rs->k2_t0_inv ? ~rs->k2_t0_inv : 0ull;
    rec.k2_t1 = rs->k2_t1;
    if (rs->found < 0) {          // corrupt pending node (leaf kernel's check)
        ls->stop = 4;
        return;
    }
    int64_t branched = 0, internal = 0, leaves = 0;
    for (int s = 0; s < pool->nseg; ++s) {
        const Segment& sg = pool->seg[s];
        const int64_t kids = sg.count * (n - sg.depth);
        branched += sg.count;
        cnt[sg.depth] -= sg.count;  // pops (the bucket tops)
        if (sg.depth >= n - 2) leaves += kids;
        else internal += kids;
    }
    for (int s = 0; s < pool->nseg; ++s) {  // pushes, batch order
        const Segment& sg = pool->seg[s];
        if (sg.depth < n - 2) cnt[sg.depth + 1] += rs->seg_surv[s];
    }
    if (leaves > 0 && rs->leaf_inv != 0ull) {
        const int32_t v = (int32_t)((~rs->leaf_inv) >> 32);
        if (ls->frozen) {
            if (v < ls->incumbent && (!ls->found || v < ls->best)) {  // bench.hpp:99-102
                ls->best = v;
                ls->found = 1;
            }
        } else if (v < ls->incumbent) {  // search.hpp:93-99
            ls->incumbent = v;
            ls->best = v;
            ls->found = 1;
            if (rs->found > 0)
                for (int i = 0; i < n; ++i) ls->schedule[i] = rs->schedule[i];
        }
    }
    int64_t pending = 0;
    for (int d = 0; d <= n; ++d) pending += cnt[d];
    rec.target = ls->targets[round];
    rec.branched = branched;
    rec.bounded = internal + leaves;
    rec.inserted = rs->total;
    rec.pruned = internal - rs->total;
    rec.leaves = leaves;
    rec.pending = pending;
    rec.incumbent = ls->frozen ? (ls->found ? ls->best : ls->incumbent) : ls->incumbent;
    rec.valid = 1;
    ls->tot_bounded += internal + leaves;
    if (pending == 0) ls->stop = 1;
    else if (ls->budget > 0 && ls->tot_bounded >= ls->budget) ls->stop = 2;
    rec.t1 = loop_ns();
}


// One kernel between two rounds of a batch: the integrate bookkeeping of round - 1 and the
// plan of round (either may be absent: round 0 has nothing to close, round == nrounds
// nothing to plan).  One warp: the bucket sizes move to shared memory with parallel
// loads, thread 0 runs the sequential parts over that copy, the warp writes it back.
__global__ void loop_step_kernel(DevTables t, LoopState* ls, Pool* pool, RoundState* rs, int round,
                                 int last) {
    // a programmatic dependent of the previous round's place kernel (or of the batch's
    // state upload): wait for it before reading anything, then let the leaf kernel be
    // scheduled
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;");
    __shared__ int64_t s_cnt[kMaxJobs + 1];
    const int n = t.n, lane = threadIdx.x;
    for (int d = lane; d <= n; d += 32) s_cnt[d] = ls->cnt[d];
    // a batch starts with every record invalid (rounds it never reaches stay so; the
    // host uploads only the state head)
    if (round == 0)
        for (int i = lane; i < kLoopMax; i += 32) ls->rec[i].valid = 0;
    __syncwarp();
    if (lane == 0) {
        if (round > 0) close_round(t, ls, pool, rs, round - 1, s_cnt);
        if (!last) plan_round(t, ls, pool, rs, round, s_cnt);
    }
    __syncwarp();
    for (int d = lane; d <= n; d += 32) ls->cnt[d] = s_cnt[d];
}

// The step of a batch driven by a conditional WHILE node of the batch graph, run first in
// the loop body: it closes the round run by the previous iteration, plans the next one
// and sets both conditions -- the WHILE node's (another iteration after this one: a round
// was planned) and the body's IF node around the leaf kernels (the planned pool has leaf
// segments).  The round index lives in the loop state (ls->cur_round), so one graph
// serves every batch length; an iteration that plans nothing runs K2 / place as no-ops and
// ends the loop.
__global__ void loop_step_dyn_kernel(DevTables t, LoopState* ls, Pool* pool, RoundState* rs,
                                     cudaGraphConditionalHandle loop_cond,
                                     cudaGraphConditionalHandle leaf_cond) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;");
    __shared__ int64_t s_cnt[kMaxJobs + 1];
    const int n = t.n, lane = threadIdx.x;
    for (int d = lane; d <= n; d += 32) s_cnt[d] = ls->cnt[d];
    if (ls->cur_round == 0)  // a batch starts with every record invalid (see loop_step_kernel)
        for (int i = lane; i < kLoopMax; i += 32) ls->rec[i].valid = 0;
    __syncwarp();
    if (lane == 0) {
        const int round = ls->cur_round;
        if (round > 0) close_round(t, ls, pool, rs, round - 1, s_cnt);
        plan_round(t, ls, pool, rs, round, s_cnt);  // nothing planned past nrounds or a stop
        ls->cur_round = round + 1;
        const bool planned = pool->nseg > 0;
        cudaGraphSetConditional(leaf_cond, planned && pool->seg[0].depth >= n - 2 ? 1u : 0u);
        cudaGraphSetConditional(loop_cond, planned ? 1u : 0u);
    }
    __syncwarp();
    for (int d = lane; d <= n; d += 32) ls->cnt[d] = s_cnt[d];
}

}  // namespace

// Loads the loop kernels now (CUDA loads kernels lazily, at first launch -- which would
// otherwise land inside the first batch's graph capture).
void preload_loop_kernels() {
    cudaFuncAttributes a;
    cudaFuncGetAttributes(&a, loop_step_kernel);
    cudaFuncGetAttributes(&a, loop_step_dyn_kernel);
}

cudaError_t launch_loop_step_dyn(const DevTables& t, LoopState* ls, Pool* pool, RoundState* rs,
                                 cudaGraphConditionalHandle loop_cond, cudaGraphConditionalHandle leaf_cond,
                                 cudaStream_t stream, bool pdl) {
    return launch_pdl(loop_step_dyn_kernel, dim3(1), dim3(32), 0, stream, pdl, t, ls, pool, rs, loop_cond,
                      leaf_cond);
}

cudaError_t launch_loop_step(const DevTables& t, LoopState* ls, Pool* pool, RoundState* rs, int round,
                             bool last, cudaStream_t stream, bool pdl) {
    return launch_pdl(loop_step_kernel, dim3(1), dim3(32), 0, stream, pdl, t, ls, pool, rs, round,
                      last ? 1 : 0);
}

}  // namespace fbb
