// k2_common.cuh -- pieces shared by the K2 kernels: chunk claiming, segment
// lookup and the leaf key.
//
// Output ordering.  A pool's children are processed in chunks (runs of parents
// of one segment, claimed in increasing order from an atomic ticket for load
// balance).  Each chunk compacts its survivors (stable, batch order) into its
// own staging slot and records the count and its segment.  The last CTA of the
// launch to finish (k2_finish) scans the counts into every chunk's destination
// row; place_kernel then moves the survivors to their final, batch-ordered
// positions (the reference's push order, search.hpp:100-102).  No chunk ever
// waits on another: an in-kernel decoupled look-back was tried and cost ~30 % of
// K2 in barrier stalls.
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

// Claims the next chunk for the CTA (all threads return the same value).
__device__ inline int64_t claim_chunk(RoundState* rs, int64_t c_begin, int64_t* s_slot) {
    __syncthreads();  // previous chunk fully consumed
    if (threadIdx.x == 0) *s_slot = c_begin + (int64_t)atomicAdd(&rs->ticket, 1u);
    __syncthreads();
    return *s_slot;
}

__device__ __forceinline__ void leaf_offer(RoundState* rs, int32_t value, int64_t pos) {
    // min over (value, position) == max over its complement; 0 means "none yet"
    unsigned long long key = ((unsigned long long)(uint32_t)value << 32) | (uint32_t)pos;
    atomicMax(&rs->leaf_inv, ~key);
}

// Scratch (shared memory, reused after the chunk loop) that k2_finish needs.
constexpr int kFinishPer = 16;  // chunks per thread per scan pass
constexpr size_t kFinishScratch = (size_t)(4 * kMaxSegments + 34) * 8;

// Called by every CTA of a K2 launch after its last chunk.  The last CTA to
// arrive turns the per-chunk survivor counts into destination rows (exclusive
// scan in batch order, rebased per segment onto dst_base) and the per-segment
// and pool totals of `rs`.  Each thread scans kFinishPer consecutive chunks, so
// a pass covers blockDim * kFinishPer chunks (one pass for a 256K-child pool).
__device__ inline void k2_finish(const Pool* __restrict__ pool, RoundState* rs, ChunkOut out,
                                 unsigned char* scratch) {
    int64_t* s_cb = (int64_t*)scratch;            // chunk_base per segment
    int64_t* s_db = s_cb + kMaxSegments;          // dst_base per segment
    int64_t* s_segoff = s_db + kMaxSegments;      // exclusive offset of the segment's first chunk
    unsigned long long* s_tot = (unsigned long long*)(s_segoff + kMaxSegments);
    int64_t* s_warp = (int64_t*)(s_tot + kMaxSegments);  // 32
    int* s_last = (int*)(s_warp + 32);
    __threadfence();  // this CTA's counts and staging rows before its arrival
    __syncthreads();
    if (threadIdx.x == 0) *s_last = atomicAdd(&rs->done, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!*s_last) return;
    __threadfence();
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
    const int64_t nchunks = pool->nchunks;
    const int nseg = pool->nseg;
    for (int s = tid; s < nseg; s += blockDim.x) {
        s_cb[s] = pool->seg[s].chunk_base;
        s_db[s] = pool->seg[s].dst_base;
        s_tot[s] = 0ull;
    }
    __syncthreads();
    int64_t carry = 0;
    for (int64_t base = 0; base < nchunks; base += (int64_t)blockDim.x * kFinishPer) {
        const int64_t i0 = base + (int64_t)tid * kFinishPer;
        int v[kFinishPer];
        int64_t sum = 0;
#pragma unroll
        for (int u = 0; u < kFinishPer; ++u) {
            v[u] = i0 + u < nchunks ? __ldcg(out.count + i0 + u) : 0;
            sum += v[u];
        }
        int64_t incl = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int64_t x = __shfl_up_sync(0xFFFFFFFFu, incl, o);
            if (lane >= o) incl += x;
        }
        if (lane == 31) s_warp[warp] = incl;
        __syncthreads();
        int64_t woff = 0, tot = 0;
        for (int w = 0; w < nw; ++w) {
            if (w < warp) woff += s_warp[w];
            tot += s_warp[w];
        }
        const int64_t excl0 = carry + woff + incl - sum;
        // segment of chunk i0 (last with chunk_base <= i0); segments start at
        // increasing chunks, a chunk-less (leaf) segment shares its successor's
        int s0 = 0;
        {
            int lo = 0, hi = nseg - 1;
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if (s_cb[mid] <= i0) lo = mid; else hi = mid - 1;
            }
            s0 = lo;
        }
        int s = s0;
        int64_t e = excl0;
#pragma unroll
        for (int u = 0; u < kFinishPer; ++u) {
            const int64_t i = i0 + u;
            if (i < nchunks) {
                while (s + 1 < nseg && s_cb[s + 1] <= i) ++s;
                if (i == s_cb[s]) s_segoff[s] = e;
                if (v[u]) atomicAdd(&s_tot[s], (unsigned long long)v[u]);
                e += v[u];
            }
        }
        __syncthreads();
        s = s0;
        e = excl0;
#pragma unroll
        for (int u = 0; u < kFinishPer; ++u) {
            const int64_t i = i0 + u;
            if (i < nchunks) {
                while (s + 1 < nseg && s_cb[s + 1] <= i) ++s;
                out.dst_row[i] = s_db[s] < 0 ? e : s_db[s] + e - s_segoff[s];
                e += v[u];
            }
        }
        carry += tot;
        __syncthreads();
    }
    for (int s = tid; s < nseg; s += blockDim.x) rs->seg_surv[s] = (int64_t)s_tot[s];
    if (tid == 0) rs->total = carry;
}

}  // namespace fbb
