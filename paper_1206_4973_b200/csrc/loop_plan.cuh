// loop_plan.cuh -- plan and close of one explorer round on the device (thread 0 of one
// CTA over a shared-memory copy of the bucket sizes): used by the batch step kernels
// (explorer_loop.cu) and by the persistent batch kernel (expand_v2.cu).
//   plan    fill_buffer (search.hpp:64-73) on the bucket sizes: pop the deepest bucket
//           tops, LIFO, until the children reach the target; lay out segments and chunks
//           exactly as the host planner does (capi.cu layout_pool); point each segment at
//           its source and destination buckets; reset the round state.
//   close   integrate / frozen prune bookkeeping (search.hpp:84-107, bench.hpp:96-106):
//           bucket sizes, incumbent and schedule, the round's counters, stop conditions.
#pragma once

#include "fbb_internal.h"

namespace fbb {

__device__ __forceinline__ unsigned long long loop_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// A pool's head and its first nseg segments, in 64-bit words over the calling threads:
// global -> shared (L2 reads: the plan was written during this kernel or the last one) and
// shared -> global.
__device__ __forceinline__ int pool_words(int nseg) {
    return (int)((offsetof(Pool, seg) + (size_t)nseg * sizeof(Segment)) / 8);
}
__device__ __forceinline__ void pool_load(Pool* __restrict__ s_dst, const Pool* __restrict__ g_src, int nseg,
                                          int tid, int nthreads) {
    const unsigned long long* src = reinterpret_cast<const unsigned long long*>(g_src);
    unsigned long long* dst = reinterpret_cast<unsigned long long*>(s_dst);
    for (int i = tid; i < pool_words(nseg); i += nthreads) dst[i] = __ldcg(src + i);
}
__device__ __forceinline__ void pool_store(Pool* __restrict__ g_dst, const Pool* __restrict__ s_src, int nseg,
                                           int tid, int nthreads) {
    const unsigned long long* src = reinterpret_cast<const unsigned long long*>(s_src);
    unsigned long long* dst = reinterpret_cast<unsigned long long*>(g_dst);
    for (int i = tid; i < pool_words(nseg); i += nthreads) dst[i] = src[i];
}

// Warp sums / exclusive scans over the segments of a plan (lanes = segments, in passes of 32).
__device__ __forceinline__ int64_t warp_sum64(int64_t v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
    return v;
}
__device__ __forceinline__ int64_t warp_excl64(int64_t v, int lane) {
    int64_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int64_t y = __shfl_up_sync(0xFFFFFFFFu, x, o);
        if (lane >= o) x += y;
    }
    return x - v;
}

// Chunks of the plan's internal segments with at most `cap` parents per chunk (warp sum).
__device__ __forceinline__ int64_t warp_chunks(const Pool* __restrict__ pool, int nseg, int n, int cmax, int cap,
                                               int lane) {
    int64_t c = 0;
    for (int s = lane; s < nseg; s += 32) {
        const Segment& sg = pool->seg[s];
        if (sg.depth < n - 2) c += ceil_div(sg.count, parents_per_chunk(n, sg.depth, cmax, cap));
    }
    return warp_sum64(c);
}

// plan of round `round`, by the 32 lanes of one warp (cnt = the block's shared copy of the
// bucket sizes; pool = a SHARED-memory pool the caller copies out).  Lane 0 runs
// fill_buffer and the destination checks; the chunk layout and the small-pool spread
// (spread_ppc) run with a lane per segment -- one thread doing it all took ~10 us per
// round (integer divisions and shared-memory loads in dependent chains, O(segments) each).
// LoopBuckets: the batch-constant bucket storage and capacities, staged in shared memory
// by the caller (the lane-0 loops read them per segment: global loads there were a chain
// of L2 round trips).
struct LoopBuckets {
    const NodeStore* __restrict__ bucket;
    const int64_t* __restrict__ cap;
};
__device__ __forceinline__ void stage_buckets(const LoopState* __restrict__ ls, NodeStore* s_bucket, int64_t* s_cap,
                                              int n, int tid, int nthreads) {
    for (int d = tid; d <= n; d += nthreads) {
        s_bucket[d] = ls->bucket[d];
        s_cap[d] = ls->cap[d];
    }
}

__device__ __forceinline__ void plan_round(const DevTables& t, LoopState* __restrict__ ls, Pool* __restrict__ pool,
                                           RoundState* __restrict__ rs, int round,
                                           const int64_t* __restrict__ cnt, LoopBuckets bk, int lane) {
    const int n = t.n;
    int nseg = 0;
    int64_t target = 0;
    if (lane == 0) {
        if (round < kLoopMax) ls->rec[round].t0 = loop_ns();
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
        if (!ls->stop && round < ls->nrounds) target = ls->targets[round] < 1 ? 1 : ls->targets[round];
    }
    target = __shfl_sync(0xFFFFFFFFu, target, 0);
    if (target == 0) return;  // stopped, or past the batch's rounds
    // fill_buffer on the sizes (deepest bucket first, LIFO, until >= target), a lane per
    // bucket in passes of 32 (i = n - d, deepest first): bucket i is popped iff it is
    // non-empty and the full contents of the deeper buckets, prefix_i = sum_{j<i} c_j r_j,
    // stay below the target (then every deeper one was popped whole); it gives k_i =
    // min(c_i, ceil((target - prefix_i) / r_i)) parents.  Destinations: bucket d+1 after
    // the pops (only bucket i-1 = d+1 can have been popped) must hold the worst case.
    int64_t have = 0, k_prev = 0;
    int fail = -1;  // first segment whose destination is too small
    int64_t fail_rows = 0;
    for (int i0 = 0; i0 <= n && have < target; i0 += 32) {
        const int i = i0 + lane, d = n - i;
        const bool lane_ok = i <= n;
        const int64_t c = lane_ok ? cnt[d] : 0;
        const int r = i;
        const int64_t capc = c * r;
        const int64_t prefix = have + warp_excl64(capc, lane);
        const bool take = lane_ok && c > 0 && prefix < target;
        const int64_t k = take ? (r > 0 ? min(c, ceil_div(target - prefix, r)) : c) : 0;
        const unsigned tk = __ballot_sync(0xFFFFFFFFu, take);
        const int s = nseg + __popc(tk & ((1u << lane) - 1u));
        int64_t kp = __shfl_up_sync(0xFFFFFFFFu, k, 1);  // bucket d+1's pops
        if (lane == 0) kp = k_prev;
        bool bad = false;
        int64_t worst = 0;
        if (take) {
            Segment& sg = pool->seg[s];
            sg.src = bk.bucket[d];
            sg.first = c - 1;
            sg.step = -1;
            sg.count = k;
            sg.depth = d;
            sg.pad = 0;
            sg.dst_lb = nullptr;
            if (d >= n - 2) {
                sg.dst = NodeStore{nullptr, nullptr, nullptr};
                sg.dst_base = 0;
            } else {
                const int64_t after = cnt[d + 1] - kp;
                worst = after + k * r;
                bad = worst > bk.cap[d + 1];
                sg.dst = bk.bucket[d + 1];
                sg.dst_base = after;
            }
        }
        const unsigned badm = __ballot_sync(0xFFFFFFFFu, bad);
        if (badm && fail < 0) {
            const int src = __ffs(badm) - 1;
            fail_rows = __shfl_sync(0xFFFFFFFFu, worst, src);
            fail = n - (i0 + src) + 1;  // the bucket that must grow: depth d + 1
        }
        nseg += __popc(tk);
        have += warp_sum64(take ? k * r : 0);
        k_prev = __shfl_sync(0xFFFFFFFFu, k, 31);
    }
    if (lane == 0) {
        if (nseg == 0) ls->stop = 1;
        else if (fail >= 0) {
            ls->stop = 3;
            ls->need_depth = fail;
            ls->need_rows = fail_rows;
        }
    }
    if (fail >= 0) nseg = 0;  // nothing of this round runs
    nseg = __shfl_sync(0xFFFFFFFFu, nseg, 0);
    __syncwarp();
    if (nseg == 0) return;
    // chunk layout (capi.cu layout_pool): small pools spread over the K2 wave (spread_ppc,
    // the same result: the smallest cap that fits, by binary search on warp sums)
    const int cmax = ls->cmax, ppc_cap = ls->ppc_cap, blocks = ls->spread_blocks;
    int ppc_lim = 0;
    if (blocks > 0) {
        int64_t parents = 0, nint = 0;
        int ppc_max = 0;
        for (int s = lane; s < nseg; s += 32) {
            const Segment& sg = pool->seg[s];
            if (sg.depth >= n - 2) continue;
            parents += sg.count;
            ++nint;
            ppc_max = max(ppc_max, parents_per_chunk(n, sg.depth, cmax, ppc_cap));
        }
        parents = warp_sum64(parents);
        nint = warp_sum64(nint);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) ppc_max = max(ppc_max, __shfl_xor_sync(0xFFFFFFFFu, ppc_max, o));
        if (nint > 0 && blocks > nint && warp_chunks(pool, nseg, n, cmax, ppc_cap, lane) < blocks) {
            int64_t lo = ceil_div(parents, blocks - nint), hi = ppc_max;
            if (lo < 1) lo = 1;
            if (lo < hi && warp_chunks(pool, nseg, n, cmax, (int)lo, lane) <= blocks) hi = lo;  // usual case
            while (lo < hi) {
                const int64_t mid = (lo + hi) >> 1;
                if (warp_chunks(pool, nseg, n, cmax, (int)mid, lane) > blocks) lo = mid + 1;
                else hi = mid;
            }
            ppc_lim = lo < ppc_max ? (int)lo : 0;
        }
    }
    const int cap = round_ppc_cap(ppc_cap, ppc_lim);
    int64_t child = 0, chunk = 0;
    int first_internal = nseg;
    for (int s0 = 0; s0 < nseg; s0 += 32) {
        const int s = s0 + lane;
        int64_t kids = 0, chunks = 0;
        bool internal = false;
        if (s < nseg) {
            const Segment& sg = pool->seg[s];
            kids = sg.count * (n - sg.depth);
            internal = sg.depth < n - 2;
            if (internal) chunks = ceil_div(sg.count, parents_per_chunk(n, sg.depth, cmax, cap));
        }
        const int64_t cb = child + warp_excl64(kids, lane), kb = chunk + warp_excl64(chunks, lane);
        if (s < nseg) {
            pool->seg[s].child_base = cb;
            pool->seg[s].chunk_base = kb;
            rs->seg_surv[s] = 0;
        }
        const unsigned in = __ballot_sync(0xFFFFFFFFu, internal);
        if (first_internal == nseg && in) first_internal = s0 + __ffs(in) - 1;
        child += warp_sum64(kids);
        chunk += warp_sum64(chunks);
    }
    if (lane == 0) {
        if (chunk > ls->chunk_cap) {  // the host sized staging for the worst case: never taken
            ls->stop = 5;
            return;  // nseg stays 0: nothing of this round runs
        }
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
    __syncwarp();
}

// integrate bookkeeping of round `round`, by the 32 lanes of one warp (updates the shared
// bucket sizes): per-segment pops, pushes and counts a lane per segment, the rest lane 0
__device__ __forceinline__ void close_round(const DevTables& t, LoopState* __restrict__ ls, const Pool* __restrict__ pool,
                                            const RoundState* rs, int round, int64_t* __restrict__ cnt, int lane) {
    // (rs: written by other CTAs during the persistent kernel -- never the read-only path)
    const int n = t.n;
    LoopRecord& rec = ls->rec[round];
    const int nseg = pool->nseg;
    if (nseg == 0) {  // stopped before this round
        if (lane == 0) rec.valid = 0;
        return;
    }
    if (rs->found < 0) {  // corrupt pending node (leaf kernel's check)
        if (lane == 0) {
            rec.valid = 0;
            ls->stop = 4;
        }
        return;
    }
    int64_t branched = 0, internal = 0, leaves = 0;
    for (int s = lane; s < nseg; s += 32) {  // pops (the bucket tops); depths are distinct
        const Segment& sg = pool->seg[s];
        const int64_t kids = sg.count * (n - sg.depth);
        branched += sg.count;
        cnt[sg.depth] -= sg.count;
        if (sg.depth >= n - 2) leaves += kids;
        else internal += kids;
    }
    __syncwarp();
    for (int s = lane; s < nseg; s += 32) {  // pushes
        const Segment& sg = pool->seg[s];
        if (sg.depth < n - 2) cnt[sg.depth + 1] += rs->seg_surv[s];
    }
    branched = warp_sum64(branched);
    internal = warp_sum64(internal);
    leaves = warp_sum64(leaves);
    __syncwarp();
    int64_t pending = 0;
    for (int d = lane; d <= n; d += 32) pending += cnt[d];
    pending = warp_sum64(pending);
    if (lane != 0) return;
    rec.k2_t0 = rs->k2_t0_inv ? ~rs->k2_t0_inv : 0ull;
    rec.k2_t1 = rs->k2_t1;
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

}  // namespace fbb
