// k2_common.cuh -- pieces shared by the K2 kernels: chunk claiming, segment
// lookup and the leaf key.
//
// Output ordering.  A pool's children are processed in chunks (runs of parents
// of one segment, claimed in increasing order from an atomic ticket for load
// balance).  Each chunk compacts its survivors (stable, batch order) into its
// own staging slot and records the count and its segment; place_kernel derives
// every chunk's destination row from the counts and moves the survivors to their
// final, batch-ordered positions (the reference's push order, search.hpp:100-102).
// No chunk ever waits on another: an in-kernel decoupled look-back cost ~30 % of
// K2 in barrier stalls, and a last-CTA scan inside K2 needs a gpu-scope release
// per CTA, which doubled K2's time on B200.
#pragma once

#include "fbb_internal.h"

namespace fbb {

__device__ __forceinline__ int find_segment_lb(const Pool* __restrict__ pool, int lo, int64_t chunk) {
    int hi = pool->nseg - 1;
    while (lo < hi) {  // last segment with chunk_base <= chunk
        int mid = (lo + hi + 1) >> 1;
        if (pool->seg[mid].chunk_base <= chunk) lo = mid; else hi = mid - 1;
    }
    return lo;
}

// K2's span on the device clock (%globaltimer, ns): with place_kernel launched as its
// programmatic dependent no CUDA event can sit between the two kernels, so the K2 time
// of a round is the first CTA start .. last CTA end recorded here.
__device__ __forceinline__ unsigned long long global_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ void k2_stamp_begin(RoundState* rs) {
    if (threadIdx.x == 0) atomicMax(&rs->k2_t0_inv, ~global_ns());
}
__device__ __forceinline__ void k2_stamp_end(RoundState* rs) {
    __syncthreads();
    if (threadIdx.x == 0) atomicMax(&rs->k2_t1, global_ns());
}

// Claims the next chunk for the CTA (all threads return the same value).
__device__ inline int64_t claim_chunk(RoundState* rs, int64_t c_begin, int64_t* s_slot) {
    __syncthreads();  // previous chunk fully consumed
    if (threadIdx.x == 0) *s_slot = c_begin + (int64_t)atomicAdd(&rs->ticket, 1u);
    __syncthreads();
    return *s_slot;
}

// Compact pending rows (the host-resident tree stores prefixes only, see capi.cu): a
// parent's heads are child_heads (instance.hpp:81-89) folded over its prefix.  One
// thread per parent, the M heads in registers; pj(j, k) = p[j][k].
template <int M, class PJ>
__device__ __forceinline__ void heads_from_prefix(const uint8_t* pre, int depth, PJ pj, int32_t (&h)[M]) {
#pragma unroll
    for (int k = 0; k < M; ++k) h[k] = 0;
    for (int i = 0; i < depth; ++i) {
        const int j = pre[i];
        int32_t prev = 0;
#pragma unroll
        for (int k = 0; k < M; ++k) {
            prev = max(prev, h[k]) + pj(j, k);
            h[k] = prev;
        }
    }
}

// A survivor's staged row written with the widest stores its alignment allows (one
// thread per survivor, so narrow stores scatter): heads as 16- or 8-byte vectors, the
// prefix -- the parent's staged prefix (smem, 4-byte aligned rows) with the child's
// job at `depth` -- as 4-byte words when rows are word aligned (n % 4 == 0).
template <int M>
__device__ __forceinline__ void store_heads(int32_t* dst, const int32_t (&R)[M]) {
    if constexpr (M % 4 == 0) {
#pragma unroll
        for (int k = 0; k < M / 4; ++k)
            reinterpret_cast<uint4*>(dst)[k] = make_uint4(R[4 * k], R[4 * k + 1], R[4 * k + 2], R[4 * k + 3]);
    } else if constexpr (M % 2 == 0) {
#pragma unroll
        for (int k = 0; k < M / 2; ++k) reinterpret_cast<uint2*>(dst)[k] = make_uint2(R[2 * k], R[2 * k + 1]);
    } else {
#pragma unroll
        for (int k = 0; k < M; ++k) dst[k] = R[k];
    }
}
__device__ __forceinline__ void store_prefix(uint8_t* dp, const uint8_t* sp, int depth, int x, int n) {
    if ((n & 3) == 0) {
        const uint32_t* s32 = reinterpret_cast<const uint32_t*>(sp);
        uint32_t* d32 = reinterpret_cast<uint32_t*>(dp);
        for (int w = 0; w <= (depth >> 2); ++w) {
            uint32_t v = s32[w];
            if (w == (depth >> 2)) {
                const int sh = (depth & 3) * 8;
                v = (v & ~(0xFFu << sh)) | ((uint32_t)x << sh);
            }
            d32[w] = v;
        }
    } else {
        for (int i = 0; i < depth; ++i) dp[i] = sp[i];
        dp[depth] = (uint8_t)x;
    }
}

// Direct placement (Pool::direct): the grid-wide arrival of every chunk's counts.  Thread
// 0 of each CTA adds its chunk's survivors to the segment / pool totals, releases them
// (gpu-scope fence) and counts itself in; then waits until all `nchunks` chunks are in.
// Every CTA of the grid is resident (the host enables the mode only for single-wave pools,
// and K2 triggers its programmatic dependents only after this barrier), so the spin ends.
__device__ __forceinline__ void direct_arrive(RoundState* rs, int s, int tot, int64_t nchunks) {
    if (threadIdx.x == 0) {
        if (tot) {
            atomicAdd((unsigned long long*)&rs->seg_surv[s], (unsigned long long)tot);
            atomicAdd((unsigned long long*)&rs->total, (unsigned long long)tot);
        }
        __threadfence();
        atomicAdd(&rs->arrived, 1u);
        uint32_t v;
        for (;;) {
            asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(v) : "l"(&rs->arrived) : "memory");
            if ((int64_t)v >= nchunks) break;
            __nanosleep(64);
        }
    }
    __syncthreads();
}

// Survivors of chunks [lo, hi) (their counts are final after direct_arrive): a block-wide
// sum of L2 reads; every thread gets the result.
__device__ __forceinline__ int64_t direct_prefix(const int32_t* count, int64_t lo, int64_t hi,
                                                 int64_t* s_red) {
    int64_t v = 0;
    for (int64_t c = lo + threadIdx.x; c < hi; c += blockDim.x) v += __ldcg(count + c);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
    if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = v;
    __syncthreads();
    int64_t t = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += s_red[w];
    return t;
}

// Direct placement, at the end of a CTA's chunk (after its K2 end stamp): the last CTA
// publishes the round summary into the mapped host RoundState, as place_kernel's last CTA
// does in the staged form.
__device__ __forceinline__ void direct_finish(const Pool* pool, RoundState* rs, int n, int64_t nchunks) {
    __shared__ int s_last;
    if (threadIdx.x == 0) {
        __threadfence();
        s_last = (int64_t)atomicAdd(&rs->place_done, 1u) == nchunks - 1;
    }
    __syncthreads();
    RoundState* summary = pool->summary;
    if (!s_last || summary == nullptr) return;
    __threadfence();
    const int words = (int)((offsetof(RoundState, seg_surv) + (size_t)pool->nseg * 8) / 8);
    const unsigned long long* src = reinterpret_cast<const unsigned long long*>(rs);
    unsigned long long* dst = reinterpret_cast<unsigned long long*>(summary);
    for (int i = threadIdx.x; i < words; i += blockDim.x) dst[i] = __ldcg(src + i);
    for (int i = threadIdx.x; i < n; i += blockDim.x) summary->schedule[i] = __ldcg(rs->schedule + i);
}

__device__ __forceinline__ void leaf_offer(RoundState* rs, int32_t value, int64_t pos) {
    // min over (value, position) == max over its complement; 0 means "none yet"
    unsigned long long key = ((unsigned long long)(uint32_t)value << 32) | (uint32_t)pos;
    atomicMax(&rs->leaf_inv, ~key);
}

// Children of parents at depth >= n-2 are complete schedules: bound = makespan
// (bound.hpp:95).  Thread per child; batch-minimum (value, position) by atomicMin.
// A pool has at most two leaf segments, both ahead of every internal one (segments
// are depth-descending): parents at depth n-1 (children complete at once) and at
// depth n-2 (children auto-completed, search.hpp:48-55).  Pending trees built by the
// search itself never hold depth n-1 nodes, but fbb_explorer_reset / push and
// fbb_expand_bound_prune accept them.
__device__ __forceinline__ int leaf_segments(const Pool* __restrict__ pool, int n) {
    int k = 0;
    while (k < 2 && k < pool->nseg && pool->seg[k].depth >= n - 2) ++k;
    return k;
}

// The leaf children of a pool, one per thread (grid-stride): makespan of the completion,
// batch minimum (value, first position) by atomicMin.
__device__ __forceinline__ void leaf_children(const DevTables& t, const Pool* __restrict__ pool, RoundState* rs,
                                              int nls) {
    const int n = t.n, m = t.m, W = t.W;
    const int64_t nc0 = pool->seg[0].count * (n - pool->seg[0].depth);
    const int64_t nct = nc0 + (nls > 1 ? pool->seg[1].count * (n - pool->seg[1].depth) : 0);
    for (int64_t cc = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; cc < nct;
         cc += (int64_t)gridDim.x * blockDim.x) {
        const int si = cc < nc0 ? 0 : 1;
        const Segment& sg = pool->seg[si];
        const int64_t c = si == 0 ? cc : cc - nc0;
        const int depth = sg.depth;
        const int r = n - depth;
        int64_t pp = c / r;
        int rk = (int)(c - pp * r);
        int64_t node = sg.first + sg.step * pp;
        // the unscheduled jobs in ascending order: x = rk-th, y = the other
        int u[2] = {-1, -1}, cnt = 0;
        int32_t prev = 0, h[kMaxMachines];
        if (sg.src.heads) {
            const uint64_t* mk = sg.src.masks + node * W;
            for (int j = 0; j < n && cnt < 2; ++j)
                if (!((mk[j >> 6] >> (j & 63)) & 1ull)) u[cnt++] = j;
            for (int k = 0; k < m; ++k) h[k] = sg.src.heads[node * m + k];
        } else {  // compact rows: heads and unscheduled jobs from the prefix
            const uint8_t* pre = sg.src.prefix + node * n;
            uint64_t sm[kMaxWords] = {0, 0, 0, 0};
            for (int k = 0; k < m; ++k) h[k] = 0;
            for (int i = 0; i < depth; ++i) {  // child_heads, instance.hpp:81-89
                const int j = pre[i];
                sm[j >> 6] |= 1ull << (j & 63);
                prev = 0;
                for (int k = 0; k < m; ++k) {
                    prev = max(prev, h[k]) + t.p[j * m + k];
                    h[k] = prev;
                }
            }
            for (int j = 0; j < n && cnt < 2; ++j)
                if (!((sm[j >> 6] >> (j & 63)) & 1ull)) u[cnt++] = j;
        }
        if (cnt < r) {  // a pending node must have exactly r unscheduled jobs
            atomicExch(&rs->found, -1);
            continue;
        }
        int x = u[rk], y = (r == 2) ? u[1 - rk] : -1;
        prev = 0;
        for (int k = 0; k < m; ++k) {
            prev = max(prev, h[k]) + t.p[x * m + k];
            h[k] = prev;
        }
        if (y >= 0) {
            prev = 0;
            for (int k = 0; k < m; ++k) {
                prev = max(prev, h[k]) + t.p[y * m + k];
                h[k] = prev;
            }
        }
        leaf_offer(rs, h[m - 1], sg.child_base + c);
    }
}

// Writes the schedule of the batch's best leaf (if it beats the pool's bound) before the
// parents' storage is recycled by the push.  A
// corrupt-node flag (found < 0, set by the leaf kernel) is kept for the host to report.
__device__ inline void write_leaf_schedule(const DevTables& t, const Pool* __restrict__ pool, RoundState* rs) {
    if (rs->found < 0) return;
    const int32_t ub = pool->ub;
    const int n = t.n;
    const int nls = leaf_segments(pool, n);
    unsigned long long inv = rs->leaf_inv;
    unsigned long long key = ~inv;
    int32_t* schedule = rs->schedule;
    int32_t* found = &rs->found;
    if (nls == 0 || inv == 0ull || (int32_t)(key >> 32) >= ub) {  // no (improving) leaf
        *found = 0;
        return;
    }
    int64_t pos = (int64_t)(key & 0xFFFFFFFFull);
    // the leaf's segment: the first or (depth n-2 behind depth n-1) the second one
    const int si = nls > 1 && pos >= pool->seg[1].child_base ? 1 : 0;
    const Segment& sg = pool->seg[si];
    const int r = n - sg.depth;
    int64_t c = pos - sg.child_base;
    int64_t pp = c / r;
    int rk = (int)(c - pp * r);
    int64_t node = sg.first + sg.step * pp;
    const uint8_t* pre = sg.src.prefix + node * n;
    uint64_t sm[kMaxWords] = {0, 0, 0, 0};  // scheduled jobs, from the prefix
    for (int i = 0; i < sg.depth; ++i) {
        schedule[i] = pre[i];
        sm[pre[i] >> 6] |= 1ull << (pre[i] & 63);
    }
    int u[2] = {-1, -1}, cnt = 0;
    for (int j = 0; j < n && cnt < 2; ++j)
        if (!((sm[j >> 6] >> (j & 63)) & 1ull)) u[cnt++] = j;
    schedule[sg.depth] = u[rk];
    if (r == 2) schedule[sg.depth + 1] = u[1 - rk];
    *found = 1;
}

}  // namespace fbb
