// expand_kernel.cu -- K2: fused expand + bound + prune + compact of a pool.
//
// One round of the reference explorer for a list of parents in pop order:
//   branch           search.hpp:40-59   children in ascending job order,
//                                       depth n-1 children auto-completed
//   evaluate         bound.hpp:94-109   every child's lower bound
//   integrate/prune  search.hpp:84-107, bench.hpp:96-106
// fused so that children never exist in memory unless they survive.
//
// Sibling bound (SURVEY finding 3).  For parent U (unscheduled set, r jobs)
// and pair q = (k,l) let V_i = D_<i + c_i over the Johnson order of U.  The
// child that schedules x (position i_x) has M'_x = max(prefmax_{<i_x},
// sufmax_{>i_x} - d_x), so ONE forward and ONE backward scan of the pair row
// give M' for all r children: O(P*n) per parent instead of O(P*n) per child.
// Child bound for pair q: Lc'_l(x) + max(R'_l(x), R'_k(x) + M'_x) with R' the
// child heads (instance.hpp:81-89) and Lc'_l(x) = load_l(U) - p[x][l] +
// min_{U\x} tail_l (min1/min2 per machine).
//
// Work layout per CTA and chunk (a run of parents of one depth whose
// children fit `cmax`):
//   stage     parents' unscheduled bits and heads -> smem
//   per parent: rank of each job in U; per (parent, machine) load/min1/min2
//   Phase A   items (parent, pair): forward+backward scan, M' -> smem Mq[child][pair]
//   Phase B   items child: heads, one-machine term, max over pairs -> lb
//   compact   block scan of (lb < UB) in batch order -> staging[chunk]
// Leaves (parents at depth >= n-2) are evaluated by their own kernel, which
// also produces the batch leaf minimum that non-frozen pruning needs
// (integrate lowers the incumbent mid-batch; leaves precede every internal
// child in a pool because the leaf-producing bucket is the deepest one).
#include <climits>
#include <type_traits>

#include "k2_common.cuh"

namespace fbb {

namespace {

constexpr int32_t kNeg = -(1 << 20);

__host__ __device__ inline size_t a16(size_t x) { return (x + 15) & ~size_t(15); }

struct K2Layout {
    size_t jm, pk, p, tl, um, R, rank, ujob, load, min1, min2, amin, Mq, cR, cL, pre, wsum, total;
    int ppc_max, pst, mst;
};

// mq_bytes: 2 (int16 M', the safe16 instances) or 4 (kWide: int32 M')
__host__ __device__ inline K2Layout k2_layout(int n, int m, int P, int cmax, int threads,
                                              bool jm_in_smem, int mq_bytes = 2) {
    K2Layout L;
    int W32 = (n + 31) / 32;
    L.ppc_max = cmax / 3 > 0 ? cmax / 3 : 1;
    L.pst = P + 1;             // Mq row stride (elements); odd -> conflict-free rows
    L.mst = m + 1;             // child row stride for cR / cL
    size_t o = 0;
    L.jm = o;   o = a16(o + (jm_in_smem ? (size_t)n * P * 4 : 0));
    L.pk = o;   o = a16(o + (size_t)P * 4);
    L.p = o;    o = a16(o + (size_t)n * m * 4);
    L.tl = o;   o = a16(o + (size_t)n * m * 4);
    L.um = o;   o = a16(o + (size_t)L.ppc_max * W32 * 4);
    L.R = o;    o = a16(o + (size_t)L.ppc_max * m * 4);
    L.rank = o; o = a16(o + (size_t)L.ppc_max * n);
    L.ujob = o; o = a16(o + (size_t)L.ppc_max * n);
    L.load = o; o = a16(o + (size_t)L.ppc_max * m * 4);
    L.min1 = o; o = a16(o + (size_t)L.ppc_max * m * 4);
    L.min2 = o; o = a16(o + (size_t)L.ppc_max * m * 4);
    L.amin = o; o = a16(o + (size_t)L.ppc_max * m * 4);
    L.Mq = o;   o = a16(o + (size_t)cmax * L.pst * mq_bytes);
    L.cR = o;   o = a16(o + (size_t)cmax * L.mst * 4);
    L.cL = o;   o = a16(o + (size_t)cmax * L.mst * 4);
    L.pre = o;  o = a16(o + (size_t)L.ppc_max * n);
    L.wsum = o; o = a16(o + (size_t)(threads / 32 + 2) * 8);
    L.total = o;
    return L;
}

__device__ inline int find_segment(const Pool* __restrict__ pool, int lo, int64_t chunk) {
    int hi = pool->nseg - 1;
    while (lo < hi) {  // last segment with chunk_base <= chunk
        int mid = (lo + hi + 1) >> 1;
        if (pool->seg[mid].chunk_base <= chunk) lo = mid; else hi = mid - 1;
    }
    return lo;
}

__device__ inline bool um_test(const uint32_t* um, int j) { return (um[j >> 5] >> (j & 31)) & 1u; }

// kJmSmem: the Johnson table is staged in shared memory (n*P*4 bytes); for the
// largest instances (200x20: 152 KB) it is read through L1/L2 instead.
// kWide: instances outside the packed / 16-bit ranges (DevTables::safe16): the unpacked
// rows (DevTables::jw) and int32 M' -- the reference's plain int arithmetic
// (bound.hpp:27-44, 79-90) for any instance whose total processing time fits int32.
template <bool kJmSmem, bool kWide>
__global__ void __launch_bounds__(128) k2_internal_kernel(DevTables t, const Pool* __restrict__ pool,
                                                         int first_seg, int cmax, int32_t ub,
                                                         int frozen, RoundState* rs,
                                                         ChunkOut out) {
    asm volatile("griddepcontrol.launch_dependents;");  // place_kernel may be scheduled early
    extern __shared__ __align__(16) unsigned char smem[];
    const int n = t.n, m = t.m, P = t.P, W = t.W;
    const int W32 = (n + 31) / 32;
    using MqT = typename std::conditional<kWide, int32_t, int16_t>::type;
    constexpr int32_t kNegA = kWide ? -(1 << 29) : kNeg;  // -inf: |D|, c <= 2^30 (total check)
    const K2Layout L = k2_layout(n, m, P, cmax, blockDim.x, kJmSmem && !kWide, (int)sizeof(MqT));
    const uint32_t* s_jm = (kJmSmem && !kWide) ? (const uint32_t*)(smem + L.jm) : t.jm;
    int32_t* s_pk = (int32_t*)(smem + L.pk);
    int32_t* s_p = (int32_t*)(smem + L.p);
    int32_t* s_tl = (int32_t*)(smem + L.tl);
    uint32_t* s_um = (uint32_t*)(smem + L.um);
    int32_t* s_R = (int32_t*)(smem + L.R);
    uint8_t* s_rank = (uint8_t*)(smem + L.rank);
    uint8_t* s_ujob = (uint8_t*)(smem + L.ujob);
    int32_t* s_load = (int32_t*)(smem + L.load);
    int32_t* s_min1 = (int32_t*)(smem + L.min1);
    int32_t* s_min2 = (int32_t*)(smem + L.min2);
    int32_t* s_amin = (int32_t*)(smem + L.amin);
    MqT* s_Mq = (MqT*)(smem + L.Mq);
    int32_t* s_cR = (int32_t*)(smem + L.cR);
    int32_t* s_cL = (int32_t*)(smem + L.cL);
    uint8_t* s_pre = (uint8_t*)(smem + L.pre);
    int64_t* s_slot = (int64_t*)(smem + L.wsum);
    int32_t* s_wsum = (int32_t*)(smem + L.wsum + 16);
    const int tid = threadIdx.x, bd = blockDim.x, lane = tid & 31, warp = tid >> 5;
    const int nwarps = bd >> 5;

    if (kJmSmem && !kWide)
        for (int x = tid; x < n * P; x += bd) ((uint32_t*)(smem + L.jm))[x] = t.jm[x];
    for (int x = tid; x < P; x += bd) s_pk[x] = (int32_t)t.pair_k[x] | ((int32_t)t.pair_l[x] << 16);
    for (int x = tid; x < n * m; x += bd) {
        s_p[x] = t.p[x];
        s_tl[x] = t.tails[x];
    }
    // Johnson row entry (job, d, c) of position i, pair q
    auto entry = [&](int i, int q, int& j, int32_t& d, int32_t& c) {
        if constexpr (kWide) {
            const int4 w = __ldg(t.jw + (size_t)i * P + q);
            j = w.x;
            d = w.y;
            c = w.z;
        } else {
            const uint32_t e = s_jm[i * P + q];
            j = entry_job(e);
            d = entry_d(e);
            c = entry_c(e);
        }
    };
    // incumbent for internal children: min(UB, batch leaf minimum) unless frozen
    // the round's bound, semantics and first internal segment come from the pool
    // (written by the host, or by the device-side planner of the batched explorer loop)
    asm volatile("griddepcontrol.wait;" ::: "memory");  // the pool upload kernel (PDL)
    k2_stamp_begin(rs);
    ub = pool->ub;
    frozen = pool->frozen;
    first_seg = pool->first_internal;
    if (first_seg >= pool->nseg) return;
    int32_t ub_eff = ub;
    if (!frozen) {
        unsigned long long inv = rs->leaf_inv;
        int32_t v = (int32_t)((~inv) >> 32);
        if (inv != 0ull && v < ub_eff) ub_eff = v;
    }

    const int64_t c_begin = pool->seg[first_seg].chunk_base;
    const int64_t c_end = pool->nchunks;
    for (int64_t chunk = claim_chunk(rs, c_begin, s_slot); chunk < c_end;
         chunk = claim_chunk(rs, c_begin, s_slot)) {
        const int s = find_segment(pool, first_seg, chunk);
        const Segment& sg = pool->seg[s];
        const int depth = sg.depth;
        const int r = n - depth;
        const int ppc = cmax / r;
        const int64_t p0 = (chunk - sg.chunk_base) * ppc;
        const int np = (int)(sg.count - p0 < ppc ? sg.count - p0 : ppc);
        const int nc = np * r;
        const NodeStore src = sg.src;
        const int64_t first = sg.first, step = sg.step;
        // ---- stage parents (all global parent reads happen before the look-back)
        for (int x = tid; x < np * depth; x += bd) {
            int pp = x / depth, i = x - pp * depth;
            s_pre[pp * n + i] = src.prefix[(first + step * (p0 + pp)) * n + i];
        }
        const bool compact = src.heads == nullptr;  // prefix-only rows (host-resident tree)
        for (int x = tid; x < np * W32 && !compact; x += bd) {
            int pp = x / W32, w = x - pp * W32;
            int64_t node = first + step * (p0 + pp);
            uint64_t word = src.masks[node * W + (w >> 1)];
            uint32_t half = (w & 1) ? (uint32_t)(word >> 32) : (uint32_t)word;
            int valid = min(32, n - w * 32);
            uint32_t vmask = valid >= 32 ? 0xFFFFFFFFu : ((1u << valid) - 1u);
            s_um[x] = ~half & vmask;
        }
        for (int x = tid; x < np * m && !compact; x += bd) {
            int pp = x / m, k = x - pp * m;
            int64_t node = first + step * (p0 + pp);
            s_R[x] = src.heads[node * m + k];
        }
        __syncthreads();
        if (compact) {  // heads and unscheduled set folded from the staged prefixes
            for (int pp = tid; pp < np; pp += bd) {
                const uint8_t* pre = s_pre + pp * n;
                int32_t* R = s_R + pp * m;
                for (int k = 0; k < m; ++k) R[k] = 0;
                for (int i = 0; i < depth; ++i) {  // child_heads, instance.hpp:81-89
                    const int j = pre[i];
                    int32_t prev = 0;
                    for (int k = 0; k < m; ++k) {
                        prev = max(prev, R[k]) + s_p[j * m + k];
                        R[k] = prev;
                    }
                }
                uint32_t* um = s_um + pp * W32;
                for (int w = 0; w < W32; ++w) {
                    const int valid = min(32, n - w * 32);
                    um[w] = valid >= 32 ? 0xFFFFFFFFu : ((1u << valid) - 1u);
                }
                for (int i = 0; i < depth; ++i) um[pre[i] >> 5] &= ~(1u << (pre[i] & 31));
            }
            __syncthreads();
        }
        // ---- per parent: rank of each unscheduled job, ascending job list
        for (int pp = tid; pp < np; pp += bd) {
            const uint32_t* um = s_um + pp * W32;
            int rk = 0;
            for (int j = 0; j < n; ++j) {
                if (um_test(um, j)) {
                    s_rank[pp * n + j] = (uint8_t)rk;
                    s_ujob[pp * n + rk] = (uint8_t)j;
                    ++rk;
                }
            }
        }
        // ---- per (parent, machine): load, smallest and second-smallest tail
        for (int x = tid; x < np * m; x += bd) {
            int pp = x / m, k = x - pp * m;
            const uint32_t* um = s_um + pp * W32;
            int32_t load = 0, m1 = INT_MAX, m2 = INT_MAX, am = -1;
            for (int j = 0; j < n; ++j) {
                if (um_test(um, j)) {
                    load += s_p[j * m + k];
                    int32_t tv = s_tl[j * m + k];
                    if (tv < m1) {
                        m2 = m1;
                        m1 = tv;
                        am = j;
                    } else if (tv < m2) {
                        m2 = tv;
                    }
                }
            }
            s_load[x] = load;
            s_min1[x] = m1;
            s_min2[x] = m2;
            s_amin[x] = am;
        }
        __syncthreads();
        // ---- Phase A: per (parent, pair) forward/backward Johnson scans
        for (int x = tid; x < np * P; x += bd) {
            int pp = x / P, q = x - pp * P;
            const uint32_t* um = s_um + pp * W32;
            const uint8_t* rank = s_rank + pp * n;
            MqT* Mq = s_Mq + (size_t)(pp * r) * L.pst + q;
            // int16 M' (safe16 instances: every M' fits; -inf clamps to -32768, which
            // loses to R_l since R_k <= R_l); int32 M' in the kWide form
            constexpr int32_t kLo = kWide ? INT_MIN : -32768;
            int32_t D = 0, PM = kNegA;
            for (int i = 0; i < n; ++i) {
                int j;
                int32_t dj, cj;
                entry(i, q, j, dj, cj);
                if (um_test(um, j)) {
                    Mq[rank[j] * L.pst] = (MqT)max(PM, kLo);  // exclusive prefix max
                    PM = max(PM, D + cj);
                    D += dj;
                }
            }
            int32_t SM = kNegA;
            for (int i = n - 1; i >= 0; --i) {
                int j;
                int32_t dj, cj;
                entry(i, q, j, dj, cj);
                if (um_test(um, j)) {
                    D -= dj;  // D_<i
                    MqT* slot = Mq + rank[j] * L.pst;
                    int32_t v = max((int32_t)*slot, SM - dj);
                    *slot = (MqT)max(v, kLo);
                    SM = max(SM, D + cj);
                }
            }
        }
        __syncthreads();
        // ---- Phase B: per child bound
        for (int c = tid; c < nc; c += bd) {
            int pp = c / r, rk = c - pp * r;
            int x = s_ujob[pp * n + rk];
            const int32_t* R = s_R + pp * m;
            int32_t* cR = s_cR + c * L.mst;
            int32_t* cL = s_cL + c * L.mst;
            int32_t prev = 0, lb = 0;
            for (int k = 0; k < m; ++k) {
                prev = max(prev, R[k]) + s_p[x * m + k];  // child_heads, instance.hpp:81-89
                cR[k] = prev;
                int pk = pp * m + k;
                int32_t mt = (x == s_amin[pk]) ? s_min2[pk] : s_min1[pk];
                int32_t lc = s_load[pk] - s_p[x * m + k] + mt;
                cL[k] = lc;
                lb = max(lb, prev + lc);  // one-machine term (bound.hpp:61-74)
            }
            const MqT* Mq = s_Mq + (size_t)c * L.pst;
            for (int q = 0; q < P; ++q) {
                int kl = s_pk[q];
                int k = kl & 0xFFFF, l = kl >> 16;
                int32_t v = cL[l] + max(cR[l], cR[k] + (int32_t)Mq[q]);
                lb = max(lb, v);
            }
            cR[m] = lb;  // stash the bound in the row's spare slot
        }
        __syncthreads();
        // ---- prune + stable compaction straight into the destination
        int base_off = 0;
        for (int c0 = 0; c0 < nc; c0 += bd) {  // survivor count first
            int c = c0 + tid;
            bool keep = c < nc && s_cR[c * L.mst + m] < ub_eff;
            unsigned ballot = __ballot_sync(0xFFFFFFFFu, keep);
            if (lane == 0) s_wsum[warp] = __popc(ballot);
            __syncthreads();
            int tot = 0;
            for (int w = 0; w < nwarps; ++w) tot += s_wsum[w];
            base_off += tot;
            __syncthreads();
        }
        if (tid == 0) {
            out.count[chunk] = base_off;
            out.seg[chunk] = s;
        }
        const int64_t out0 = chunk * (int64_t)cmax;
        const NodeStore dst = out.nodes;
        int run = 0;
        for (int c0 = 0; c0 < nc; c0 += bd) {
            int c = c0 + tid;
            int32_t lb = c < nc ? s_cR[c * L.mst + m] : 0;
            bool keep = c < nc && lb < ub_eff;
            unsigned ballot = __ballot_sync(0xFFFFFFFFu, keep);
            if (lane == 0) s_wsum[warp] = __popc(ballot);
            __syncthreads();
            int woff = 0, tot = 0;
            for (int w = 0; w < nwarps; ++w) {
                int v = s_wsum[w];
                if (w < warp) woff += v;
                tot += v;
            }
            if (keep) {
                const int64_t o = out0 + run + woff + __popc(ballot & ((1u << lane) - 1u));
                int pp = c / r, rk = c - pp * r;
                int xj = s_ujob[pp * n + rk];
                const int32_t* cR = s_cR + c * L.mst;
                for (int k = 0; k < m; ++k) dst.heads[o * m + k] = cR[k];
                const uint32_t* um = s_um + pp * W32;
                for (int w = 0; w < W; ++w) {
                    uint32_t lo = 2 * w < W32 ? um[2 * w] : 0u;
                    uint32_t hi = 2 * w + 1 < W32 ? um[2 * w + 1] : 0u;
                    int vlo = min(32, max(0, n - 64 * w));
                    int vhi = min(32, max(0, n - 64 * w - 32));
                    uint32_t mlo = vlo >= 32 ? 0xFFFFFFFFu : ((1u << vlo) - 1u);
                    uint32_t mhi = vhi >= 32 ? 0xFFFFFFFFu : ((1u << vhi) - 1u);
                    uint64_t sched = ((uint64_t)(~hi & mhi) << 32) | (uint64_t)(~lo & mlo);
                    if ((xj >> 6) == w) sched |= (uint64_t)1 << (xj & 63);
                    dst.masks[o * W + w] = sched;
                }
                uint8_t* dp = dst.prefix + o * n;
                for (int i = 0; i < depth; ++i) dp[i] = s_pre[pp * n + i];
                dp[depth] = (uint8_t)xj;
                out.lb[o] = lb;
            }
            run += tot;
            __syncthreads();
        }
    }
    k2_stamp_end(rs);
}


__global__ void k2_leaf_kernel(DevTables t, const Pool* __restrict__ pool, int /*unused*/,
                               RoundState* rs) {
    asm volatile("griddepcontrol.wait;" ::: "memory");  // the pool upload (PDL chain)
    asm volatile("griddepcontrol.launch_dependents;");
    const int n = t.n;
    const int nls = leaf_segments(pool, n);
    if (nls == 0) return;  // no leaves
    leaf_children(t, pool, rs, nls);
}

// The best leaf's schedule, after every leaf CTA's offer is in: a one-thread programmatic
// dependent of the leaf kernel.  (Having the leaf kernel's last CTA write it instead needs
// a gpu-scope release per CTA -- measured +10 us per Ta001 leaf round of ~1000 CTAs.)
__global__ void leaf_schedule_kernel(DevTables t, const Pool* __restrict__ pool, RoundState* rs) {
    asm volatile("griddepcontrol.wait;" ::: "memory");  // the leaf kernel (PDL chain)
    asm volatile("griddepcontrol.launch_dependents;");
    if (threadIdx.x == 0 && blockIdx.x == 0) write_leaf_schedule(t, pool, rs);
}

// Moves every chunk's survivors from its staging slot to its final, batch-ordered
// row: the segment's dst at dst_base + (survivors of the segment's earlier
// chunks), or the contiguous output at (survivors of all earlier chunks) when
// dst_base < 0; adds the per-segment and pool totals to `rs`.  One CTA per
// kPlaceChunks consecutive chunks derives its own offsets by summing the counts
// of all earlier chunks (a few thousand L2-resident ints, kPlaceBatch
// independent loads per thread), so no scan pass or grid-wide fence is needed.
// Rows are copied flat (one thread per 4-byte head, mask word or prefix byte).
#ifndef FBB_PLACE_CHUNKS
#define FBB_PLACE_CHUNKS 8
#endif
constexpr int kPlaceChunks = FBB_PLACE_CHUNKS;
constexpr int kPlaceThreads = 256;
constexpr int kPlaceBatch = 8;

// Copies rows x width elements: element f = (row, k) with row = f / width.  The thread's
// (row, k) advance by a fixed (kPlaceThreads / width, kPlaceThreads % width) step with one
// carry, so no integer division per element (the division emulation was most of the
// kernel's instructions).
template <int B, class Load, class Store>
__device__ __forceinline__ void copy_rows(int rows, int width, Load load, Store store) {
    const int total = rows * width;
    const int qs = kPlaceThreads / width, rs = kPlaceThreads - qs * width;
    int row = threadIdx.x / width, k = threadIdx.x - row * width;
    for (int base = threadIdx.x; base < total; base += B * kPlaceThreads) {
        decltype(load(0, 0)) v[B];
        int rr[B], kk[B];
#pragma unroll
        for (int u = 0; u < B; ++u) {
            rr[u] = row;
            kk[u] = k;
            if (base + u * kPlaceThreads < total) v[u] = load(row, k);
            row += qs;
            k += rs;
            if (k >= width) {
                k -= width;
                ++row;
            }
        }
#pragma unroll
        for (int u = 0; u < B; ++u)
            if (base + u * kPlaceThreads < total) store(rr[u], kk[u], v[u]);
    }
}

// kGridStride: a fixed grid strides over the chunk groups (the device-planned loop, whose
// pool size the host does not know); otherwise one group per CTA -- the plain form,
// measurably faster (19 vs 26 us per 262K-child round) when the host sizes the grid.
template <bool kGridStride>
// summary (non-null, one-group form only): the last CTA past the counting copies the
// round's counters (and the leaf schedule) into this mapped host RoundState, which
// replaces the summary download (one stream operation less per round).
__global__ void __launch_bounds__(kPlaceThreads) place_kernel(DevTables t, const Pool* __restrict__ pool,
                                                              int cmax, RoundState* rs, ChunkOut out,
                                                              RoundState* summary) {
    const int n = t.n, m = t.m, W = t.W;
    __shared__ int s_row0[kPlaceChunks + 1];  // CTA-local exclusive survivor offsets
    __shared__ int s_seg[kPlaceChunks];
    __shared__ int64_t s_dst[kPlaceChunks];
    __shared__ NodeStore s_store[kPlaceChunks];
    __shared__ int32_t* s_dlb[kPlaceChunks];
    __shared__ int64_t s_red[2][kPlaceThreads / 32];
    __shared__ int s_need;                     // prefix bytes that matter: max child depth
    extern __shared__ uint8_t s_rc[];          // chunk of each row (cmax * kPlaceChunks)
    // launched as a programmatic dependent of K2 (FBB_PDL=1): wait for its completion
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;");  // the device loop's close kernel
    if (pool->direct) return;  // K2 placed the survivors itself (single-wave pool)
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t nchunks = pool->nchunks;
    for (int64_t c0 = (int64_t)blockIdx.x * kPlaceChunks; c0 < nchunks;
         c0 += kGridStride ? (int64_t)gridDim.x * kPlaceChunks : nchunks) {
    if (kGridStride) __syncthreads();  // previous group's shared tables consumed
    const int nch = (int)(nchunks - c0 < kPlaceChunks ? nchunks - c0 : kPlaceChunks);
    const int s0 = out.seg[c0];
    const int64_t cb0 = pool->seg[s0].chunk_base;
    if (tid == 0) s_need = 0;
    if (tid < 32) {
        const int v = tid < nch ? out.count[c0 + tid] : 0;
        int incl = v;
        for (int o = 1; o < 32; o <<= 1) {
            const int u = __shfl_up_sync(0xFFFFFFFFu, incl, o);
            if (tid >= o) incl += u;
        }
        if (tid < nch) {
            s_row0[tid] = incl - v;
            s_seg[tid] = out.seg[c0 + tid];
        }
        if (tid == nch - 1) s_row0[nch] = incl;
    }
    // a = survivors of chunks [0, cb0), b = of [cb0, c0)
    int64_t a = 0, b = 0;
    for (int64_t base = tid; base < c0; base += (int64_t)kPlaceBatch * kPlaceThreads) {
        int v[kPlaceBatch];
#pragma unroll
        for (int u = 0; u < kPlaceBatch; ++u) {
            const int64_t i = base + (int64_t)u * kPlaceThreads;
            v[u] = i < c0 ? out.count[i] : 0;
        }
#pragma unroll
        for (int u = 0; u < kPlaceBatch; ++u) {
            const int64_t i = base + (int64_t)u * kPlaceThreads;
            if (i < cb0) a += v[u]; else b += v[u];
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        a += __shfl_xor_sync(0xFFFFFFFFu, a, o);
        b += __shfl_xor_sync(0xFFFFFFFFu, b, o);
    }
    if (lane == 0) {
        s_red[0][warp] = a;
        s_red[1][warp] = b;
    }
    __syncthreads();
    if (tid < nch) {
        int64_t A = 0, B = 0;
        for (int w = 0; w < kPlaceThreads / 32; ++w) {
            A += s_red[0][w];
            B += s_red[1][w];
        }
        const int s = s_seg[tid];
        const Segment& sg = pool->seg[s];
        const int64_t glob = A + B + s_row0[tid];
        const int64_t seg0 = s == s0 ? A : A + B + s_row0[sg.chunk_base - c0];
        s_dst[tid] = sg.dst_base < 0 ? glob : sg.dst_base + (glob - seg0);
        s_store[tid] = sg.dst;
        s_dlb[tid] = sg.dst_lb;
        const int cnt = s_row0[tid + 1] - s_row0[tid];
        if (cnt) atomicAdd((unsigned long long*)&rs->seg_surv[s], (unsigned long long)cnt);
        atomicMax(&s_need, sg.depth + 1);
    }
    const int R = s_row0[nch];
    if (tid == 0 && R) atomicAdd((unsigned long long*)&rs->total, (unsigned long long)R);
    if (!kGridStride && summary && tid < max(nch, 1)) __threadfence();  // this CTA's counts, device-wide
    for (int c = 0; c < nch; ++c)
        for (int row = s_row0[c] + tid; row < s_row0[c + 1]; row += kPlaceThreads) s_rc[row] = (uint8_t)c;
    __syncthreads();
    if (!kGridStride && summary) {
        __shared__ int s_last;
        if (tid == 0) s_last = atomicAdd(&rs->place_done, 1u) == gridDim.x - 1;
        __syncthreads();
        if (s_last) {  // every CTA's counts are in: publish the summary
            __threadfence();
            const int words = (int)((offsetof(RoundState, seg_surv) + (size_t)pool->nseg * 8) / 8);
            const unsigned long long* src = reinterpret_cast<const unsigned long long*>(rs);
            unsigned long long* dst = reinterpret_cast<unsigned long long*>(summary);
            for (int i = tid; i < words; i += kPlaceThreads) dst[i] = __ldcg(src + i);
            for (int i = tid; i < t.n; i += kPlaceThreads) summary->schedule[i] = __ldcg(rs->schedule + i);
        }
    }
    auto src_row = [&](int row) { const int c = s_rc[row]; return (c0 + c) * (int64_t)cmax + (row - s_row0[c]); };
    auto dst_row = [&](int row) { const int c = s_rc[row]; return s_dst[c] + (row - s_row0[c]); };
    // Each array moves row by row in the widest unit that divides its row size (rows of
    // one array start at multiples of the row size in both places): 16-byte units for
    // 20-machine heads, 4-byte units for 20/100/200-job prefixes.  Wide units matter
    // most when the destination is pinned host memory written over the host link.
    // Only the first `used_bytes` of a row are copied (prefix rows: the child depth).
    auto copy_array = [&](const void* src_base, int row_bytes, int used_bytes, auto dst_of) {
        auto go = [&](auto unit) {
            using T = decltype(unit);
            const int w = row_bytes / (int)sizeof(T);
            const int wu = min(w, (used_bytes + (int)sizeof(T) - 1) / (int)sizeof(T));
            const T* src = (const T*)src_base;
            copy_rows<kPlaceBatch>(R, wu, [&](int row, int k) { return __ldg(src + src_row(row) * w + k); },
                                   [&](int row, int k, T v) { ((T*)dst_of(row))[dst_row(row) * w + k] = v; });
        };
        if (row_bytes % 16 == 0) go(uint4{});
        else if (row_bytes % 8 == 0) go(uint2{});
        else if (row_bytes % 4 == 0) go(0u);
        else if (row_bytes % 2 == 0) go((unsigned short)0);
        else go((unsigned char)0);
    };
    // compact destinations (prefix-only rows, the host-resident tree) have no heads /
    // masks; all segments of a pool share one residency
    if (s_store[0].heads) {
        copy_array(out.nodes.heads, m * 4, m * 4, [&](int row) { return (void*)s_store[s_rc[row]].heads; });
        copy_array(out.nodes.masks, W * 8, W * 8, [&](int row) { return (void*)s_store[s_rc[row]].masks; });
    }
    // prefix rows up to the child depth (the bytes past it are don't-care in both places)
    if (2 * s_need <= n || !pool->host_dst) {
        copy_array(out.nodes.prefix, n, s_need, [&](int row) { return (void*)s_store[s_rc[row]].prefix; });
    } else {
        // host buckets, mostly-used rows: whole rows, in aligned 16-byte stores (the host
        // link takes ~2x more bytes/s from those than from 4-byte row-unit stores; in HBM
        // the row form is faster).  Consecutive chunks of one segment are contiguous in the
        // destination, so the CTA's chunks merge into runs (usually one): partial 16-byte
        // blocks -- written byte by byte, each a separate small write over the link -- occur
        // only at the two ends of a run, not at every chunk boundary.  The 16-byte blocks of
        // all runs form one flat index space.
        __shared__ int64_t s_blk[kPlaceChunks + 1];
        __shared__ int s_run_row[kPlaceChunks + 1];  // first CTA row of each run
        __shared__ uint8_t* s_run_dst[kPlaceChunks];
        __shared__ int s_nrun;
        if (tid == 0) {
            int nr = 0;
            for (int c = 0; c < nch; ++c) {
                uint8_t* d = s_store[c].prefix + s_dst[c] * n;
                if (nr > 0 && d == s_run_dst[nr - 1] + (int64_t)(s_row0[c] - s_run_row[nr - 1]) * n) continue;
                s_run_dst[nr] = d;
                s_run_row[nr] = s_row0[c];
                ++nr;
            }
            s_run_row[nr] = s_row0[nch];
            int64_t acc = 0;
            for (int k = 0; k < nr; ++k) {
                s_blk[k] = acc;
                const int64_t len = (int64_t)(s_run_row[k + 1] - s_run_row[k]) * n;
                const uintptr_t d0 = (uintptr_t)s_run_dst[k];
                acc += len ? (int64_t)((d0 + len - (d0 & ~(uintptr_t)15) + 15) >> 4) : 0;
            }
            s_blk[nr] = acc;
            s_nrun = nr;
        }
        __syncthreads();
        const int nr = s_nrun;
        for (int64_t b = tid; b < s_blk[nr]; b += kPlaceThreads) {
            int k = 0;
            while (b >= s_blk[k + 1]) ++k;
            const int64_t len = (int64_t)(s_run_row[k + 1] - s_run_row[k]) * n;
            uint8_t* dst = s_run_dst[k];
            const uintptr_t a0 = (uintptr_t)dst & ~(uintptr_t)15;
            const int64_t off = (int64_t)(a0 + 16 * (b - s_blk[k]) - (uintptr_t)dst);  // block in dst
            // the block's bytes from the staged rows (a run's rows are not contiguous there)
            const int64_t o0 = off < 0 ? 0 : off;
            int row = (int)(o0 / n), col = (int)(o0 - (int64_t)row * n);
            const uint8_t* sp = out.nodes.prefix + src_row(s_run_row[k] + row) * n;
            uint8_t v[16];
#pragma unroll
            for (int q = 0; q < 16; ++q) {
                const int64_t o = off + q;
                v[q] = 0;
                if (o >= o0 && o < len) {
                    v[q] = __ldg(sp + col);
                    if (++col == n) {
                        col = 0;
                        ++row;
                        if (o + 1 < len) sp = out.nodes.prefix + src_row(s_run_row[k] + row) * n;
                    }
                }
            }
            if (off >= 0 && off + 16 <= len) {
                uint32_t w[4];
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    w[q] = (uint32_t)v[4 * q] | ((uint32_t)v[4 * q + 1] << 8) | ((uint32_t)v[4 * q + 2] << 16) |
                           ((uint32_t)v[4 * q + 3] << 24);
                *(uint4*)(dst + off) = make_uint4(w[0], w[1], w[2], w[3]);
            } else {  // a partial block at either end of the run
#pragma unroll
                for (int q = 0; q < 16; ++q)
                    if (off + q >= 0 && off + q < len) dst[off + q] = v[q];
            }
        }
    }
    if (s_dlb[0])  // all segments of a pool share dst_lb (set or not)
        copy_rows<kPlaceBatch>(R, 1, [&](int row, int) { return __ldg(out.lb + src_row(row)); },
                               [&](int row, int, int32_t v) { s_dlb[s_rc[row]][dst_row(row)] = v; });
    }
}

}  // namespace

K2Config k2_config(const DevTables& t, int device) {
    K2Config c;
    c.threads = 128;
    int n = t.n;
    c.cmax = n <= 128 ? 128 : ((n + 31) / 32) * 32;
    c.wide = !(t.safe16 & kSafeM16);  // outside the packed / int16 ranges: int32 form
    int max_smem = 0;
    cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
    const int mqb = c.wide ? 4 : 2;
    c.smem = k2_layout(t.n, t.m, t.P, c.cmax, c.threads, !c.wide, mqb).total;
    c.jm_in_smem = !c.wide && c.smem <= (size_t)max_smem / 2;  // keep >= 2 CTAs per SM
    if (!c.jm_in_smem) c.smem = k2_layout(t.n, t.m, t.P, c.cmax, c.threads, false, mqb).total;
    int sms = 148, per_sm = 1;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    auto kern = c.wide ? k2_internal_kernel<false, true>
                       : (c.jm_in_smem ? k2_internal_kernel<true, false> : k2_internal_kernel<false, false>);
    // the attribute is per kernel, not per context: allow the device maximum once
    int optin = 0;
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, optin);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, c.threads, c.smem);
    if (per_sm < 1) per_sm = 1;
    c.blocks = sms * per_sm;
    return c;
}

cudaError_t launch_k2_leaves(const DevTables& t, const Pool* d_pool, const Pool& h_pool,
                             int seg_index, RoundState* rs, cudaStream_t stream, bool pdl) {
    int64_t nc = 0;  // children of every leaf segment (at most two, from the first)
    for (int s = 0; s < 2 && s < h_pool.nseg && h_pool.seg[s].depth >= t.n - 2; ++s)
        nc += h_pool.seg[s].count * (t.n - h_pool.seg[s].depth);
    (void)seg_index;
    if (nc <= 0) return cudaSuccess;
    int blocks = (int)((nc + 255) / 256);
    if (blocks > 4096) blocks = 4096;
    cudaError_t e = launch_pdl(k2_leaf_kernel, dim3(blocks), dim3(256), 0, stream, pdl, t, d_pool, seg_index, rs);
    if (e != cudaSuccess) return e;
    return launch_pdl(leaf_schedule_kernel, dim3(1), dim3(32), 0, stream, pdl, t, d_pool, rs);
}

cudaError_t launch_k2_internal(const DevTables& t, const K2Config& cfg, const Pool* d_pool,
                               const Pool& h_pool, int first_seg, int32_t ub, int frozen,
                               RoundState* rs, ChunkOut out, cudaStream_t stream, bool pdl) {
    if (first_seg >= h_pool.nseg) return cudaSuccess;
    int64_t nch = h_pool.nchunks - h_pool.seg[first_seg].chunk_base;
    if (nch <= 0) return cudaSuccess;
    int blocks = (int)(nch < cfg.blocks ? nch : cfg.blocks);
    if (cfg.variant >= 100000)
        return launch_k2_v3(t, cfg, d_pool, first_seg, blocks, ub, frozen, rs, out, stream, pdl);
    if (cfg.variant != 0)
        return launch_k2_v2(t, cfg, d_pool, first_seg, blocks, h_pool.direct ? 1 : 0, frozen, rs, out, stream,
                            pdl);
    return launch_pdl(cfg.wide ? k2_internal_kernel<false, true>
                               : (cfg.jm_in_smem ? k2_internal_kernel<true, false> : k2_internal_kernel<false, false>),
                      dim3(blocks),
                      dim3(cfg.threads), cfg.smem, stream, pdl, t, d_pool, first_seg, cfg.cmax, ub, frozen, rs,
                      out);
}

namespace {
__global__ void pool_upload_kernel(const volatile unsigned long long* __restrict__ src,
                                   unsigned long long* __restrict__ dst, int words) {
    asm volatile("griddepcontrol.launch_dependents;");  // K2 may start its prologue now
    for (int i = threadIdx.x; i < words; i += blockDim.x) dst[i] = src[i];
}
}  // namespace

cudaError_t launch_pool_upload(const void* h_src, void* d_dst, int words, cudaStream_t stream) {
    pool_upload_kernel<<<1, 256, 0, stream>>>((const volatile unsigned long long*)h_src,
                                              (unsigned long long*)d_dst, words);
    return cudaGetLastError();
}


}  // namespace fbb

namespace fbb {

cudaError_t launch_place(const DevTables& t, const K2Config& cfg, const Pool* d_pool,
                         const Pool& h_pool, RoundState* rs, ChunkOut out, cudaStream_t stream,
                         RoundState* summary) {
    if (h_pool.nchunks == 0) return cudaSuccess;
    const int64_t blocks = (h_pool.nchunks + kPlaceChunks - 1) / kPlaceChunks;
    static const bool pdl = [] { const char* e = getenv("FBB_PDL"); return !(e && e[0] == '0'); }();
    if (pdl) {
        cudaLaunchConfig_t lc = {};
        lc.gridDim = dim3((unsigned)blocks);
        lc.blockDim = dim3(kPlaceThreads);
        lc.dynamicSmemBytes = (size_t)cfg.cmax * kPlaceChunks;
        lc.stream = stream;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        lc.attrs = at;
        lc.numAttrs = 1;
        return cudaLaunchKernelEx(&lc, place_kernel<false>, t, d_pool, cfg.cmax, rs, out, summary);
    }
    place_kernel<false><<<(unsigned)blocks, kPlaceThreads, (size_t)cfg.cmax * kPlaceChunks, stream>>>(
        t, d_pool, cfg.cmax, rs, out, summary);
    return cudaGetLastError();
}

}  // namespace fbb

namespace fbb {

// One round of the batched (device-planned) explorer loop: every kernel reads the
// round's plan from the device Pool / RoundState and exits when it has nothing to do,
// so the grids are fixed and nothing here needs the host.
void preload_round_kernels() {
    cudaFuncAttributes a;
    cudaFuncGetAttributes(&a, k2_leaf_kernel);
    cudaFuncGetAttributes(&a, leaf_schedule_kernel);
    cudaFuncGetAttributes(&a, place_kernel<false>);
    cudaFuncGetAttributes(&a, place_kernel<true>);
    cudaFuncGetAttributes(&a, pool_upload_kernel);
}

cudaError_t launch_round_leaves(const DevTables& t, const Pool* d_pool, RoundState* rs, cudaStream_t stream,
                                bool pdl_first, bool pdl) {
    // a one-wave grid-stride grid (rounds without leaves exit at once)
    cudaError_t e = launch_pdl(k2_leaf_kernel, dim3(148), dim3(256), 0, stream, pdl_first, t, d_pool, 0, rs);
    if (e != cudaSuccess) return e;
    return launch_pdl(leaf_schedule_kernel, dim3(1), dim3(32), 0, stream, pdl, t, d_pool, rs);
}

cudaError_t launch_round_k2_place(const DevTables& t, const K2Config& cfg, const Pool* d_pool, RoundState* rs,
                                  ChunkOut out, cudaStream_t stream, bool pdl_k2, bool pdl, int64_t place_chunks) {
    cudaError_t e;
    if (cfg.variant >= 100000)
        e = launch_k2_v3(t, cfg, d_pool, 0, cfg.blocks, 0, 0, rs, out, stream, pdl_k2);
    else if (cfg.variant != 0)
        e = launch_k2_v2(t, cfg, d_pool, 0, cfg.blocks, -1, 0, rs, out, stream, pdl_k2);
    else
        e = launch_pdl(cfg.wide ? k2_internal_kernel<false, true>
                                : (cfg.jm_in_smem ? k2_internal_kernel<true, false> : k2_internal_kernel<false, false>),
                       dim3(cfg.blocks), dim3(cfg.threads), cfg.smem, stream, pdl_k2, t, d_pool, 0, cfg.cmax, 0, 0,
                       rs, out);
    if (e != cudaSuccess || place_chunks <= 0) return e;  // 0: every pool of the batch is placed by K2
    // one CTA per group of kPlaceChunks chunks of the largest pool the staging holds (groups
    // past a round's chunks exit at once): measured faster than a fixed grid striding over
    // the groups (Ta021 262 K: the grid-stride place cost ~7 us more per round)
    const int64_t blocks = (place_chunks + kPlaceChunks - 1) / kPlaceChunks;
    return launch_pdl(place_kernel<false>, dim3((unsigned)blocks), dim3(kPlaceThreads),
                      (size_t)cfg.cmax * kPlaceChunks, stream, pdl, t, d_pool, cfg.cmax, rs, out,
                      (RoundState*)nullptr);
}

cudaError_t launch_round_device(const DevTables& t, const K2Config& cfg, const Pool* d_pool,
                                RoundState* rs, ChunkOut out, cudaStream_t stream, bool pdl, int64_t place_chunks) {
    cudaError_t e = launch_round_leaves(t, d_pool, rs, stream, pdl, pdl);
    if (e != cudaSuccess) return e;
    return launch_round_k2_place(t, cfg, d_pool, rs, out, stream, pdl, pdl, place_chunks);
}

}  // namespace fbb

