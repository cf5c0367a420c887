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
#include "loop_plan.cuh"

namespace fbb {

namespace {

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
    __shared__ __align__(16) unsigned char s_pool_raw[sizeof(Pool)];
    Pool* s_pool = reinterpret_cast<Pool*>(s_pool_raw);
    const int n = t.n, lane = threadIdx.x;
    for (int d = lane; d <= n; d += 32) s_cnt[d] = ls->cnt[d];
    // a batch starts with every record invalid (rounds it never reaches stay so; the
    // host uploads only the state head)
    if (round == 0)
        for (int i = lane; i < kLoopMax; i += 32) ls->rec[i].valid = 0;
    // the last round's plan (closed here) into shared memory; the new plan is built there
    if (round > 0) pool_load(s_pool, pool, __ldcg(&pool->nseg), lane, 32);
    __syncwarp();
    __shared__ NodeStore s_bucket[kMaxJobs + 1];
    __shared__ int64_t s_cap[kMaxJobs + 1];
    stage_buckets(ls, s_bucket, s_cap, n, lane, 32);
    __syncwarp();
    if (round > 0) close_round(t, ls, s_pool, rs, round - 1, s_cnt, lane);
    __syncwarp();
    if (!last) plan_round(t, ls, s_pool, rs, round, s_cnt, LoopBuckets{s_bucket, s_cap}, lane);
    if (!last) pool_store(pool, s_pool, s_pool->nseg, lane, 32);
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
    __shared__ __align__(16) unsigned char s_pool_raw[sizeof(Pool)];
    Pool* s_pool = reinterpret_cast<Pool*>(s_pool_raw);
    const int n = t.n, lane = threadIdx.x;
    for (int d = lane; d <= n; d += 32) s_cnt[d] = ls->cnt[d];
    const int round = ls->cur_round;
    if (round == 0)  // a batch starts with every record invalid (see loop_step_kernel)
        for (int i = lane; i < kLoopMax; i += 32) ls->rec[i].valid = 0;
    if (round > 0) pool_load(s_pool, pool, __ldcg(&pool->nseg), lane, 32);  // (see loop_step_kernel)
    __syncwarp();
    __shared__ NodeStore s_bucket[kMaxJobs + 1];
    __shared__ int64_t s_cap[kMaxJobs + 1];
    stage_buckets(ls, s_bucket, s_cap, n, lane, 32);
    __syncwarp();
    if (round > 0) close_round(t, ls, s_pool, rs, round - 1, s_cnt, lane);
    __syncwarp();
    plan_round(t, ls, s_pool, rs, round, s_cnt, LoopBuckets{s_bucket, s_cap}, lane);  // nothing planned past nrounds or a stop
    if (lane == 0) {
        ls->cur_round = round + 1;
        const bool planned = s_pool->nseg > 0;
        cudaGraphSetConditional(leaf_cond, planned && s_pool->seg[0].depth >= n - 2 ? 1u : 0u);
        cudaGraphSetConditional(loop_cond, planned ? 1u : 0u);
    }
    __syncwarp();
    pool_store(pool, s_pool, s_pool->nseg, lane, 32);
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
