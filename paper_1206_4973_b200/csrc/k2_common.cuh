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

}  // namespace fbb
