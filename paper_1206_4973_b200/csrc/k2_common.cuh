// k2_common.cuh -- pieces shared by the K2 kernels: chunk claiming, the
// decoupled look-back that orders survivors across chunks, and the leaf key.
//
// Output ordering.  A pool's children are processed in chunks (runs of
// parents of one segment).  Survivors must land in batch order (that is the
// reference's push order, search.hpp:100-102), so chunk c needs the number of
// survivors of chunks < c.  Chunks are CLAIMED in increasing order from an
// atomic ticket; each chunk publishes its survivor count (aggregate), walks
// back to the nearest published inclusive prefix, then publishes its own
// inclusive prefix (Merrill & Garland's decoupled look-back).  Because a chunk
// only waits on chunks claimed before it by running CTAs, this cannot deadlock
// whatever the residency.  A chunk publishes only after it has read all of its
// parents (prefixes staged in shared memory), which makes writing survivors
// straight into bucket depth+1 -- whose popped region holds the parents of the
// previous segment, all in earlier chunks -- race-free.
#pragma once

#include <cuda/atomic>

#include "fbb_internal.h"

namespace fbb {

constexpr uint64_t kFlagAggregate = 1ull << 46;
constexpr uint64_t kFlagInclusive = 2ull << 46;
constexpr uint64_t kFlagValueMask = (1ull << 46) - 1;

__device__ __forceinline__ uint64_t flag_pack(uint32_t epoch, uint64_t state, int64_t value) {
    return ((uint64_t)(epoch & 0xFFFFu) << 48) | state | ((uint64_t)value & kFlagValueMask);
}

__device__ __forceinline__ int find_segment_lb(const Pool* __restrict__ pool, int lo, int64_t chunk) {
    int hi = pool->nseg - 1;
    while (lo < hi) {  // last segment with chunk_base <= chunk
        int mid = (lo + hi + 1) >> 1;
        if (pool->seg[mid].chunk_base <= chunk) lo = mid; else hi = mid - 1;
    }
    return lo;
}

// Thread 0 of the CTA: publish `tot`, look back, publish the inclusive prefix;
// returns the exclusive prefix (survivors of all chunks before `chunk`).
__device__ inline int64_t lookback(uint64_t* flags, uint32_t epoch, int64_t c_begin, int64_t chunk,
                                   int64_t tot) {
    cuda::atomic_ref<uint64_t, cuda::thread_scope_device> mine(flags[chunk]);
    if (chunk == c_begin) {
        mine.store(flag_pack(epoch, kFlagInclusive, tot), cuda::memory_order_release);
        return 0;
    }
    mine.store(flag_pack(epoch, kFlagAggregate, tot), cuda::memory_order_release);
    int64_t excl = 0;
    for (int64_t j = chunk - 1; j >= c_begin; --j) {
        cuda::atomic_ref<uint64_t, cuda::thread_scope_device> f(flags[j]);
        uint64_t v;
        do {
            v = f.load(cuda::memory_order_acquire);
        } while ((uint32_t)(v >> 48) != (epoch & 0xFFFFu));
        excl += (int64_t)(v & kFlagValueMask);
        if (v & kFlagInclusive) break;
    }
    mine.store(flag_pack(epoch, kFlagInclusive, excl + tot), cuda::memory_order_release);
    return excl;
}

// Warp 0 of the CTA (all 32 lanes): the same, examining 32 predecessors per
// step -- the nearest inclusive prefix ends the walk (lowest lane = closest).
__device__ inline int64_t lookback_warp(uint64_t* flags, uint32_t epoch, int64_t c_begin,
                                        int64_t chunk, int64_t tot) {
    const int lane = threadIdx.x & 31;
    cuda::atomic_ref<uint64_t, cuda::thread_scope_device> mine(flags[chunk]);
    if (chunk == c_begin) {
        if (lane == 0) mine.store(flag_pack(epoch, kFlagInclusive, tot), cuda::memory_order_release);
        return 0;
    }
    if (lane == 0) mine.store(flag_pack(epoch, kFlagAggregate, tot), cuda::memory_order_release);
    const uint32_t ep = epoch & 0xFFFFu;
    int64_t excl = 0;
    for (int64_t base = chunk - 1;; base -= 32) {
        const int64_t idx = base - lane;
        uint64_t v = 0;
        bool inc = true;  // before the first chunk: an inclusive zero
        if (idx >= c_begin) {
            cuda::atomic_ref<uint64_t, cuda::thread_scope_device> f(flags[idx]);
            do {
                v = f.load(cuda::memory_order_acquire);
            } while ((uint32_t)(v >> 48) != ep);
            inc = (v & kFlagInclusive) != 0;
        }
        const unsigned m = __ballot_sync(0xFFFFFFFFu, inc);
        const int first = m ? __ffs(m) - 1 : 32;
        int64_t val = lane <= first ? (int64_t)(v & kFlagValueMask) : 0;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) val += __shfl_down_sync(0xFFFFFFFFu, val, off);
        excl += __shfl_sync(0xFFFFFFFFu, val, 0);
        if (m) break;
    }
    if (lane == 0) mine.store(flag_pack(epoch, kFlagInclusive, excl + tot), cuda::memory_order_release);
    return excl;
}

// Inclusive prefix published by `chunk` (spins until it is).
__device__ inline int64_t inclusive_of(uint64_t* flags, uint32_t epoch, int64_t chunk) {
    cuda::atomic_ref<uint64_t, cuda::thread_scope_device> f(flags[chunk]);
    uint64_t v;
    do {
        v = f.load(cuda::memory_order_acquire);
    } while ((uint32_t)(v >> 48) != (epoch & 0xFFFFu) || !(v & kFlagInclusive));
    return (int64_t)(v & kFlagValueMask);
}

// Output base for `chunk` of segment `sg` (thread 0), and the per-segment /
// total survivor counts from the last chunks.
__device__ inline int64_t chunk_output_base(const Pool* __restrict__ pool, int s, int64_t chunk,
                                            int64_t c_begin, int64_t nch_seg, int64_t excl,
                                            int64_t tot, uint64_t* flags, uint32_t epoch,
                                            RoundState* rs) {
    const Segment& sg = pool->seg[s];
    int64_t before_seg = sg.chunk_base > c_begin ? inclusive_of(flags, epoch, sg.chunk_base - 1) : 0;
    if (chunk == sg.chunk_base + nch_seg - 1) rs->seg_surv[s] = excl + tot - before_seg;
    if (chunk == pool->nchunks - 1) rs->total = excl + tot;
    return sg.dst_base < 0 ? excl : sg.dst_base + (excl - before_seg);
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

}  // namespace fbb
