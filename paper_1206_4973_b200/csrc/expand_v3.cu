// expand_v3.cu -- K2 for 64 < n <= 256 jobs and m in {5, 10, 20} (Taillard 100xm and
// 200xm: configs 4-5).  Same contract and output as k2_internal_kernel
// (expand_kernel.cu) and k2_v2_kernel (expand_v2.cu); a mapping that does not keep
// per-position state in registers, so it scales to n = 256:
//
//  * the repacked Johnson rows (DevTables::rowv3, [i][q]) are read from global memory
//    through L1 -- 76 KB at 100x20, 152 KB at 200x20, too large for shared memory next
//    to the per-child output rows -- lanes of a warp reading consecutive pairs of one
//    position (coalesced 128-byte rows);
//  * thread (g, q) owns machine pair q of parent lane g.  Per (parent, pair) the forward
//    pass writes every member's exclusive prefix max to its child's Mq slot, the
//    backward pass folds in the suffix max, max(slot, sufmax - d), by a read-modify-write
//    of the slot (SURVEY finding 3; bound.hpp:27-44 in max-plus form).  A per-parent
//    u16 table indexed by the job gives both the child's Mq row (or a dummy row) and
//    the membership mask, so the scans are branch-free;
//  * per (parent, machine) the load and the two smallest tails (lb_one_machine,
//    bound.hpp:61-74) by warp reductions over the unscheduled jobs;
//  * Phase B (one child per thread: child_heads, the one-machine term, max over the
//    pairs with 128-bit Mq row loads) and the stable per-chunk compaction as in v2.
#include <climits>
#include <cstdlib>

#include "k2_common.cuh"

namespace fbb {

namespace {

constexpr int32_t kNeg3 = -(1 << 20);
// takes a scheduled job's c out of every max (not a power of two: stays one IMAD)
constexpr int32_t kV3Off = 0x100003;
constexpr int kV3Ppc = 16;  // parents per chunk at most (per-parent tables are N bytes)

__host__ __device__ inline size_t c16(size_t x) { return (x + 15) & ~size_t(15); }

__host__ __device__ inline int v3_row_bytes(int P) {
    int b = (P * 2 + 15) / 16;  // 16-byte units
    if ((b & 1) == 0) b += 1;   // odd -> consecutive rows hit distinct bank groups
    return b * 16;
}

struct V3Layout {
    size_t u, rank, ujob, R, load, mins, amin, Mq, pre, wsum, total;
    int rowb;
};

__host__ __device__ inline V3Layout v3_layout(int m, int P, int cmax, int threads, int NW) {
    V3Layout L;
    const int N = 32 * NW;
    L.rowb = v3_row_bytes(P);
    size_t o = 0;
    L.u = o;    o = c16(o + (size_t)kV3Ppc * NW * 4);
    L.rank = o; o = c16(o + (size_t)kV3Ppc * N * 2);  // u16 slot table per parent
    L.ujob = o; o = c16(o + (size_t)kV3Ppc * N);
    L.R = o;    o = c16(o + (size_t)kV3Ppc * m * 4);
    L.load = o; o = c16(o + (size_t)kV3Ppc * m * 4);
    L.mins = o; o = c16(o + (size_t)kV3Ppc * m * 4);  // min1 | min2 << 16
    L.amin = o; o = c16(o + (size_t)kV3Ppc * m);
    // + dummy rows for scheduled jobs, one per parent lane (threads / P), so concurrent
    // read-modify-writes of garbage never share an address
    L.Mq = o;   o = c16(o + (size_t)(cmax + threads / P) * L.rowb);
    L.pre = o;  o = c16(o + (size_t)kV3Ppc * N);
    L.wsum = o; o = c16(o + (size_t)(threads / 32 + 2) * 8);
    L.total = o;
    return L;
}

__device__ __forceinline__ uint32_t v3_lds_u32(uint32_t addr) {
    uint32_t v;
    asm("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ uint32_t v3_lds_u16(uint32_t addr) {
    uint32_t v;
    asm("ld.shared.u16 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ uint32_t v3_lds_u8(uint32_t addr) {
    uint32_t v;
    asm("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ int32_t v3_lds_s16(uint32_t addr) {
    int16_t v;
    asm volatile("ld.shared.s16 %0, [%1];" : "=h"(v) : "r"(addr));
    return (int32_t)v;
}
__device__ __forceinline__ void v3_sts_u16(uint32_t addr, int32_t v) {
    asm volatile("st.shared.u16 [%0], %1;" ::"r"(addr), "h"((unsigned short)v));
}


// (min1, argmin, min2) of a set of tails, merged across lanes; ties keep the
// smallest job index as the argmin, as the ascending scan of v2 does.
struct Mins {
    int32_t m1, a1, m2;
};
__device__ __forceinline__ Mins mins_merge(Mins x, Mins y) {
    const bool xf = x.m1 < y.m1 || (x.m1 == y.m1 && x.a1 < y.a1);
    Mins r;
    r.m1 = xf ? x.m1 : y.m1;
    r.a1 = xf ? x.a1 : y.a1;
    r.m2 = xf ? min(x.m2, y.m1) : min(y.m2, x.m1);
    return r;
}

// 4 CTAs/SM at n <= 128 (80 registers; chunk = one parent's r <= n children, cmax = n, so
// the Mq rows fit 4 CTAs' shared memory), 2 at n <= 256
template <int NW, int M>
__global__ void __launch_bounds__(NW <= 4 ? 192 : 256, NW <= 4 ? 4 : 2)
    k2_v3_kernel(DevTables t, const Pool* __restrict__ pool, int first_seg, int cmax, int32_t ub,
                 int frozen, RoundState* rs, ChunkOut out) {
    asm volatile("griddepcontrol.launch_dependents;");  // place_kernel may be scheduled early
    constexpr int P = M * (M - 1) / 2;
    constexpr int N = 32 * NW;
    // scan unroll: 16 independent row / table loads in flight per thread (measured +2.4 %
    // at Ta081 and +3.6 % at Ta101 over 8)
    constexpr int kV3Unroll = 16;
    extern __shared__ __align__(16) unsigned char smem[];
    const int n = t.n, W = t.W;
    const V3Layout L = v3_layout(M, P, cmax, blockDim.x, NW);
    uint32_t* s_u = (uint32_t*)(smem + L.u);  // unscheduled jobs, NW words per parent
    // per parent and job: (child row offset in Mq / 16) | 0x8000 if the job is scheduled
    // (then the offset is the dummy row's)
    uint16_t* s_slot16 = (uint16_t*)(smem + L.rank);
    uint8_t* s_ujob = (uint8_t*)(smem + L.ujob);
    int32_t* s_R = (int32_t*)(smem + L.R);
    int32_t* s_load = (int32_t*)(smem + L.load);
    uint32_t* s_mins = (uint32_t*)(smem + L.mins);
    uint8_t* s_amin = (uint8_t*)(smem + L.amin);
    unsigned char* s_Mq = smem + L.Mq;
    uint8_t* s_pre = (uint8_t*)(smem + L.pre);
    int64_t* s_slot = (int64_t*)(smem + L.wsum);
    int32_t* s_wsum = (int32_t*)(smem + L.wsum + 16);
    const int tid = threadIdx.x, bd = blockDim.x, lane = tid & 31, warp = tid >> 5;
    const int nwarps = bd >> 5;
    const int G = bd / P;
    const int q = tid % P, g = tid / P;

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
        const int s = find_segment_lb(pool, first_seg, chunk);
        const Segment& sg = pool->seg[s];
        const int depth = sg.depth;
        const int r = n - depth;
        const int ppc = min(cmax / r, kV3Ppc);
        const int64_t p0 = (chunk - sg.chunk_base) * ppc;
        const int np = (int)(sg.count - p0 < ppc ? sg.count - p0 : ppc);
        const int nc = np * r;
        const NodeStore src = sg.src;
        const int64_t first = sg.first, step = sg.step;
        // ---- stage the parents
        for (int x = tid; x < np * depth; x += bd) {
            const int pp = x / depth, i = x - pp * depth;
            s_pre[pp * N + i] = src.prefix[(first + step * (p0 + pp)) * n + i];
        }
        const bool compact = src.heads == nullptr;  // prefix-only rows (host-resident tree)
        for (int x = tid; x < np * NW && !compact; x += bd) {
            const int pp = x / NW, w = x - pp * NW;
            const int64_t node = first + step * (p0 + pp);
            const int w64 = w >> 1;
            const uint64_t word = w64 < W ? src.masks[node * W + w64] : ~0ull;
            const uint32_t half = (w & 1) ? (uint32_t)(word >> 32) : (uint32_t)word;
            const int valid = min(32, max(0, n - 32 * w));
            const uint32_t vmask = valid >= 32 ? 0xFFFFFFFFu : ((1u << valid) - 1u);
            s_u[x] = ~half & vmask;
        }
        for (int x = tid; x < np * M && !compact; x += bd) {
            const int pp = x / M, k = x - pp * M;
            s_R[x] = src.heads[(first + step * (p0 + pp)) * M + k];
        }
        __syncthreads();
        if (compact) {  // heads and unscheduled set folded from the staged prefixes
            for (int pp = tid; pp < np; pp += bd) {
                const uint8_t* pre = s_pre + pp * N;
                int32_t h[M];
                heads_from_prefix<M>(pre, depth, [&](int j, int k) { return __ldg(t.p + j * M + k); }, h);
#pragma unroll
                for (int k = 0; k < M; ++k) s_R[pp * M + k] = h[k];
            }
            for (int x = tid; x < np * NW; x += bd) {
                const int pp = x / NW, w = x - pp * NW;
                const uint8_t* pre = s_pre + pp * N;
                uint32_t sched = 0;
                for (int i = 0; i < depth; ++i) {
                    const int j = pre[i];
                    if ((j >> 5) == w) sched |= 1u << (j & 31);
                }
                const int valid = min(32, max(0, n - 32 * w));
                const uint32_t vmask = valid >= 32 ? 0xFFFFFFFFu : ((1u << valid) - 1u);
                s_u[x] = ~sched & vmask;
            }
            __syncthreads();
        }
        // per parent and job: the slot table and the ascending list of unscheduled jobs
        for (int x = tid; x < np * N; x += bd) {
            const int pp = x / N, j = x - pp * N;
            const uint32_t* u = s_u + pp * NW;
            if (j < n && ((u[j >> 5] >> (j & 31)) & 1u)) {
                int rk = __popc(u[j >> 5] & ((1u << (j & 31)) - 1u));
                for (int w = 0; w < (j >> 5); ++w) rk += __popc(u[w]);
                s_slot16[x] = (uint16_t)(rk * L.rowb / 16);
                s_ujob[pp * N + rk] = (uint8_t)j;
            } else {
                s_slot16[x] = (uint16_t)(0x8000u | ((cmax + pp % G - pp * r) * L.rowb / 16));
            }
        }
        // per (parent, machine): load and the two smallest tails, a warp per item
        for (int x = warp; x < np * M; x += nwarps) {
            const int pp = x / M, k = x - pp * M;
            const uint32_t* u = s_u + pp * NW;
            int32_t load = 0;
            Mins mn{0x7FFF, 0, 0x7FFF};
#pragma unroll
            for (int w = 0; w < NW; ++w) {
                const int j = 32 * w + lane;
                if ((u[w] >> lane) & 1u) {
                    load += __ldg(t.p + j * M + k);
                    const int32_t tv = __ldg(t.tails + j * M + k);
                    mn = mins_merge(mn, Mins{tv, j, 0x7FFF});
                }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                load += __shfl_xor_sync(0xFFFFFFFFu, load, o);
                Mins other{__shfl_xor_sync(0xFFFFFFFFu, mn.m1, o), __shfl_xor_sync(0xFFFFFFFFu, mn.a1, o),
                           __shfl_xor_sync(0xFFFFFFFFu, mn.m2, o)};
                mn = mins_merge(mn, other);
            }
            if (lane == 0) {
                s_load[x] = load;
                s_mins[x] = (uint32_t)mn.m1 | ((uint32_t)mn.m2 << 16);
                s_amin[x] = (uint8_t)mn.a1;
            }
        }
        __syncthreads();
        // ---- Phase A: per (parent, pair) forward / backward max-plus scans into Mq.
        // Per position: the job's slot entry gives the child row (dummy row for a
        // scheduled job) and the membership mask (PRMT sign replication of bit 15);
        // a scheduled job's c drops out of every max (IMAD) and its d becomes 0 (LOP3).
        if (g < G) {
            const uint32_t* rowq = t.rowv3 + q;
            for (int pp = g; pp < np; pp += G) {
                const uint32_t tab_sa = (uint32_t)__cvta_generic_to_shared(s_slot16 + pp * N);
                const uint32_t base_sa =
                    (uint32_t)__cvta_generic_to_shared(s_Mq + (size_t)(pp * r) * L.rowb + 2 * q);
                int32_t D = 0, PM = -32768;  // PM stays within int16 (stored as is)
#pragma unroll kV3Unroll
                for (int i = 0; i < n; ++i) {
                    const uint32_t e = __ldg(rowq + i * P);
                    const uint32_t ent = v3_lds_u16(tab_sa + (e & 0xFFu) * 2u);
                    uint32_t sched, d;
                    asm("prmt.b32 %0, %1, 0, 0x9999;" : "=r"(sched) : "r"(ent));  // bit 15 -> mask
                    asm("prmt.b32 %0, %1, 0, 0x9991;" : "=r"(d) : "r"(e));        // int8 d
                    const uint32_t at = base_sa + (ent & 0x7FFFu) * 16u;
                    const int32_t ce = (int32_t)(e >> 16) + (int32_t)sched * kV3Off;
                    const int32_t dm = (int32_t)(d & ~sched);
                    v3_sts_u16(at, PM);  // exclusive prefix max
                    PM = max(PM, D + ce);
                    D += dm;
                }
                int32_t SM = -32768;
#pragma unroll kV3Unroll
                for (int i = n - 1; i >= 0; --i) {
                    const uint32_t e = __ldg(rowq + i * P);
                    const uint32_t ent = v3_lds_u16(tab_sa + (e & 0xFFu) * 2u);
                    uint32_t sched, d;
                    asm("prmt.b32 %0, %1, 0, 0x9999;" : "=r"(sched) : "r"(ent));
                    asm("prmt.b32 %0, %1, 0, 0x9991;" : "=r"(d) : "r"(e));
                    const uint32_t at = base_sa + (ent & 0x7FFFu) * 16u;
                    const int32_t ce = (int32_t)(e >> 16) + (int32_t)sched * kV3Off;
                    const int32_t dm = (int32_t)(d & ~sched);
                    const int32_t Db = D - dm;  // D before position i
                    v3_sts_u16(at, max(v3_lds_s16(at), SM - dm));
                    SM = max(SM, Db + ce);
                    D = Db;
                }
            }
        }
        __syncthreads();
        // ---- Phase B: per child bound with register-resident heads
        int32_t myR[M];
        int32_t mylb = 0;
        int myx = 0, mypp = 0;
        const bool b_lane = tid < nc;  // cmax <= blockDim
        if (b_lane) {
            const int pp = tid / r, rk = tid - pp * r;
            const int x = s_ujob[pp * N + rk];
            myx = x;
            mypp = pp;
            int32_t Lc[M];
            int32_t prev = 0, lb = 0;
#pragma unroll
            for (int k = 0; k < M; ++k) {
                const int pk = pp * M + k;
                const int32_t px = __ldg(t.p + x * M + k);
                prev = max(prev, s_R[pk]) + px;  // child_heads, instance.hpp:81-89
                myR[k] = prev;
                const uint32_t mins = s_mins[pk];
                const int32_t mt = (x == (int)s_amin[pk]) ? (int32_t)(mins >> 16) : (int32_t)(mins & 0xFFFFu);
                Lc[k] = s_load[pk] - px + mt;
                lb = max(lb, prev + Lc[k]);  // one-machine term (bound.hpp:61-74)
            }
            // Pairs: Lc_l + max(R_l, R_k + M'_kl).  Lc_l + R_l never exceeds the one-machine
            // term already in lb, so per k only max_l (Lc_l + M'_kl) + R_k is needed: one
            // VIADDMNMX per pair (the pairs of one k are consecutive in q order).
            const uint4* mrow = (const uint4*)(s_Mq + (size_t)tid * L.rowb);
#pragma unroll
            for (int k = 0; k < M - 1; ++k) {
                int32_t acc = kNeg3;
#pragma unroll
                for (int l = k + 1; l < M; ++l) {
                    const int qq = k * (2 * M - k - 1) / 2 + (l - k - 1);
                    const uint4 v4 = mrow[qq >> 3];
                    const int wi = (qq >> 1) & 3;
                    const uint32_t w = wi == 0 ? v4.x : wi == 1 ? v4.y : wi == 2 ? v4.z : v4.w;
                    const int32_t mq = (qq & 1) ? ((int32_t)w >> 16) : (int32_t)(int16_t)(w & 0xFFFFu);
                    acc = __viaddmax_s32(Lc[l], mq, acc);
                }
                lb = max(lb, acc + myR[k]);
            }
            mylb = lb;
        }
        // ---- prune + stable compaction into the chunk's staging slot
        const bool keep = b_lane && mylb < ub_eff;
        const unsigned ballot = __ballot_sync(0xFFFFFFFFu, keep);
        if (lane == 0) s_wsum[warp] = __popc(ballot);
        __syncthreads();
        int woff = 0, tot = 0;
        for (int w = 0; w < nwarps; ++w) {
            const int v = s_wsum[w];
            if (w < warp) woff += v;
            tot += v;
        }
        if (tid == 0) {
            out.count[chunk] = tot;
            out.seg[chunk] = s;
        }
        if (keep) {
            const int64_t o = chunk * (int64_t)cmax + woff + __popc(ballot & ((1u << lane) - 1u));
            const NodeStore dst = out.nodes;
            store_heads<M>(dst.heads + o * M, myR);
            const uint32_t* u = s_u + mypp * NW;
            for (int w = 0; w < W; ++w) {
                const uint32_t lo = 2 * w < NW ? u[2 * w] : 0u;
                const uint32_t hi = 2 * w + 1 < NW ? u[2 * w + 1] : 0u;
                const int vlo = min(32, max(0, n - 64 * w));
                const int vhi = min(32, max(0, n - 64 * w - 32));
                const uint32_t mlo = vlo >= 32 ? 0xFFFFFFFFu : ((1u << vlo) - 1u);
                const uint32_t mhi = vhi >= 32 ? 0xFFFFFFFFu : ((1u << vhi) - 1u);
                uint64_t sched = ((uint64_t)(~hi & mhi) << 32) | (uint64_t)(~lo & mlo);
                if ((myx >> 6) == w) sched |= 1ull << (myx & 63);
                dst.masks[o * W + w] = sched;
            }
            store_prefix(dst.prefix + o * n, s_pre + mypp * N, depth, myx, n);
            out.lb[o] = mylb;
        }
    }
    k2_stamp_end(rs);
}

template <int NW, int M>
cudaError_t v3_setup(K2Config& c, int device) {
    int optin = 0, sms = 148, per_sm = 1;
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    cudaError_t e = cudaFuncSetAttribute(k2_v3_kernel<NW, M>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin);
    if (e != cudaSuccess) return e;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k2_v3_kernel<NW, M>, c.threads, c.smem);
    c.blocks = sms * (per_sm < 1 ? 1 : per_sm);
    return cudaSuccess;
}

}  // namespace

bool k2_v3_config(const DevTables& t, int device, K2Config* out) {
    const int m = t.m, n = t.n;
    if (n <= 64 || n > 256 || !(m == 5 || m == 10 || m == 20) || !t.rowv3) return false;
    if (!(t.safe16 & kSafeM16)) return false;  // M' is stored as int16 (DevTables::safe16)
    K2Config c;
    const int NW = n <= 128 ? 4 : 8;
    c.cmax = n;                             // one parent's children always fit a chunk
    c.threads = NW <= 4 ? 192 : 256;        // >= cmax (Phase B: a child per thread), >= P
    if (const char* cm = getenv("FBB_K2_CMAX"))
        c.cmax = std::max(c.cmax, std::min(c.threads, (atoi(cm) / 32) * 32));
    c.ppc_cap = kV3Ppc;
    c.variant = 100000 + NW * 100 + m;
    c.jm_in_smem = false;
    c.smem = v3_layout(m, t.P, c.cmax, c.threads, NW).total;
    cudaError_t e;
    switch (c.variant) {
        case 100405: e = v3_setup<4, 5>(c, device); break;
        case 100410: e = v3_setup<4, 10>(c, device); break;
        case 100420: e = v3_setup<4, 20>(c, device); break;
        case 100805: e = v3_setup<8, 5>(c, device); break;
        case 100810: e = v3_setup<8, 10>(c, device); break;
        case 100820: e = v3_setup<8, 20>(c, device); break;
        default: return false;
    }
    if (e != cudaSuccess) return false;
    *out = c;
    return true;
}

cudaError_t launch_k2_v3(const DevTables& t, const K2Config& cfg, const Pool* d_pool, int first_seg,
                         int blocks, int32_t ub, int frozen, RoundState* rs, ChunkOut out,
                         cudaStream_t stream, bool pdl) {
#define V3_CASE(NW, MM)                                                                      \
    case 100000 + NW * 100 + MM:                                                             \
        return launch_pdl(k2_v3_kernel<NW, MM>, dim3(blocks), dim3(cfg.threads), cfg.smem, stream, pdl, t, \
                          d_pool, first_seg, cfg.cmax, ub, frozen, rs, out);
    switch (cfg.variant) {
        V3_CASE(4, 5)
        V3_CASE(4, 10)
        V3_CASE(4, 20)
        V3_CASE(8, 5)
        V3_CASE(8, 10)
        V3_CASE(8, 20)
        default: return cudaErrorInvalidValue;
    }
#undef V3_CASE
    return cudaGetLastError();
}

}  // namespace fbb
