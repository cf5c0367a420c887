// expand_v2.cu -- K2 specialised for n <= 32 jobs and m in {5, 10, 20}
// (the Taillard 20xm classes: configs 1-2).  Same contract and output as
// k2_internal_kernel (expand_kernel.cu); different mapping:
//
//  * thread (g, q) owns machine pair q for the whole kernel; its Johnson row
//    (n entries: job bit, c, d) lives in REGISTERS, so Phase A issues no table
//    loads.  g = 0..G-1 are parent lanes (G = threads / P).
//  * Phase A is branch-free: per position one LOP3 (job in U?) and predicated
//    max/add; the backward pass emits M'_x to smem Mq[child][q] (int16).
//  * Phase B: thread per child; child heads R' and the per-machine terms Lc'
//    are register arrays (template M), the pair loop is fully unrolled and reads
//    the child's Mq row with 128-bit loads (row stride = odd multiple of 16 B,
//    conflict-free).
#include <climits>
#include <cstdlib>

#include "k2_common.cuh"
#include "loop_plan.cuh"

namespace fbb {

namespace {

constexpr int32_t kNeg2 = -(1 << 20);
// Offset that takes a non-member's c out of every max (not a power of two, so the
// compiler keeps c + sched * kOff as one IMAD).  Values: |D| <= 98 * 64, c < 2^14.
constexpr int32_t kOff = 0x100003;

__host__ __device__ inline size_t b16(size_t x) { return (x + 15) & ~size_t(15); }

// Mq row layout: the slots of one k cover l = lo_k .. hi_k - 1 with lo_k = (k+1) & ~1 and
// hi_k = m rounded up to even, so Phase B reads them as 16x2 words whose halves are
// (l, l+1) with l even.  The pad slots (l = k when k is even, l = m when m is odd) are
// zeroed once per CTA and never written; the terms they produce, Lc_k + R_k and
// -16384 + R_k, never exceed the one-machine term.
__host__ __device__ constexpr int v2_lo(int k) { return (k + 1) & ~1; }
__host__ __device__ constexpr int v2_hi(int m) { return (m + 1) & ~1; }
__host__ __device__ constexpr int v2_group_base(int m, int k) {
    int b = 0;
    for (int kk = 0; kk < k; ++kk) b += v2_hi(m) - v2_lo(kk);
    return b;
}
__host__ __device__ constexpr int v2_slots(int m) { return v2_group_base(m, m - 1); }
// Slot of each pair index q (bound.hpp:97-98 order) in that layout.
template <int M>
struct SlotTab {
    unsigned char s[M * (M - 1) / 2 > 0 ? M * (M - 1) / 2 : 1];
    constexpr SlotTab() : s() {
        int q = 0;
        for (int k = 0; k < M; ++k)
            for (int l = k + 1; l < M; ++l) s[q++] = (unsigned char)(v2_group_base(M, k) + l - v2_lo(k));
    }
};
template <int M>
__constant__ SlotTab<M> kSlotOf = SlotTab<M>();

__host__ __device__ inline int v2_row_bytes(int m) {
    int b = (2 * v2_slots(m) + 15) / 16;  // 16-byte units
    if ((b & 1) == 0) b += 1;             // odd -> 8 consecutive rows hit 8 distinct bank groups
    return b * 16;
}

__host__ __device__ inline int v2_dummy_rows(int P) { return 2 * (192 / P > 0 ? 192 / P : 1); }

struct V2Layout {
    size_t row, um, rank, R, load, mins, amin, Mq, p, tl, pre, wsum, total;
    int ppc_max, rowb;
};

// Per-parent job-indexed arrays (Mq offsets, staged prefixes) hold RW = 32 entries for
// n <= 32 and 64 for the wide variant (32 < n <= 64).
__host__ __device__ inline int v2_rw(int N) { return N <= 32 ? 32 : 64; }
// Parents per chunk: the wide variant caps them at 16 so that its per-parent arrays
// leave room for 2 CTAs per SM (its 64-position rows take 48 KB).
// Measured: 32 at 2 CTAs/SM (smaller per-parent arrays and prefetch registers, +3 % at
// Ta021), none at 3 CTAs/SM (Ta001 -2.3 % with it), 16 for the wide variant.
__host__ __device__ inline int v2_ppc_cap(int N, int occ) { return N <= 32 ? (occ == 2 ? 32 : (1 << 20)) : 16; }

__host__ __device__ inline V2Layout v2_layout(int n, int m, int P, int cmax, int threads, int N, int occ) {
    V2Layout L;
    L.ppc_max = cmax / 3 > 0 ? cmax / 3 : 1;
    if (L.ppc_max > v2_ppc_cap(N, occ)) L.ppc_max = v2_ppc_cap(N, occ);
    L.rowb = v2_row_bytes(m);
    size_t o = 0;
    L.row = o;  o = b16(o + (size_t)N * P * 4);  // rows padded to N positions
    L.um = o;   o = b16(o + (size_t)L.ppc_max * 8);
    L.rank = o; o = b16(o + (size_t)L.ppc_max * v2_rw(N) * 2);  // u16 Mq offsets
    L.R = o;    o = b16(o + (size_t)L.ppc_max * m * 4);
    L.load = o; o = b16(o + (size_t)L.ppc_max * m * 4);
    L.mins = o; o = b16(o + (size_t)L.ppc_max * m * 4);  // min1 | min2 << 16
    L.amin = o; o = b16(o + (size_t)L.ppc_max * m);
    // + dummy rows for non-members: one per parent processed at the same time (two per
    // parent lane, 192 / P lanes), so concurrent garbage stores never share an address
    L.Mq = o;   o = b16(o + (size_t)(cmax + v2_dummy_rows(P)) * L.rowb);
    L.p = o;    o = b16(o + (size_t)n * m * 4);
    L.tl = o;   o = b16(o + (size_t)n * m * 2);  // tails as int16
    L.pre = o;  o = b16(o + (size_t)L.ppc_max * v2_rw(N));
    L.wsum = o; o = b16(o + (size_t)(threads / 32 + 2) * 8 + 16 * 8);  // + direct-placement sums
    L.total = o;
    return L;
}

__device__ inline int v2_find_segment(const Pool* __restrict__ pool, int lo, int64_t chunk) {
    int hi = pool->nseg - 1;
    while (lo < hi) {
        int mid = (lo + hi + 1) >> 1;
        if (pool->seg[mid].chunk_base <= chunk) lo = mid; else hi = mid - 1;
    }
    return lo;
}

// Non-volatile: ptxas may schedule these loads early (the tables are read-only
// after staging).
__device__ __forceinline__ uint32_t lds_u32(uint32_t addr) {
    uint32_t v;
    asm("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ uint32_t lds_u32_v(uint32_t addr) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ uint32_t lds_u16(uint32_t addr) {
    uint32_t v;
    asm("ld.shared.u16 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ uint32_t lds_u8(uint32_t addr) {
    uint32_t v;
    asm("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ void sts_u16(uint32_t addr, int32_t v) {
    asm volatile("st.shared.u16 [%0], %1;" ::"r"(addr), "h"((unsigned short)v));
}

// Is the job of row entry e unscheduled?  Its U bit is moved to the sign bit by a
// wrapped left funnel shift (shift = e & 31 = 31 - (job & 31)); bit 5 of e picks
// the 32-bit word of U (always the low word for n <= 32).
__device__ __forceinline__ bool member(uint32_t e, uint32_t slo, uint32_t shi) {
    return (int32_t)__funnelshift_l(0u, (e & 32u) ? shi : slo, e) >= 0;  // not scheduled
}

// Forward + backward scan of NB consecutive row positions of one pair for one
// parent, entering with D0 and prefix max PM0 (the block's start state) and the
// suffix max SM0 of the positions after the block; emits M' = max(prefix max,
// suffix max - d) of every member to its child's Mq slot and returns the suffix
// max including this block.  Per position the per-parent offset table gives the
// child's Mq row (or the dummy row for a non-member), so the only per-position
// selects are two LOP3 masks (c -> -inf, -d -> 0 for non-members).  The table
// rows hold nd = -d (b - a), which saves the negation.
template <int NB, int P, bool WIDE>
__device__ __forceinline__ int32_t scan_block(uint32_t row_sa, uint32_t slo, uint32_t shi,
                                              uint32_t off_sa, uint32_t base_sa, int32_t D0,
                                              int32_t PM0, int32_t SM0) {
    uint32_t e[NB];
#pragma unroll
    for (int i = 0; i < NB; ++i) e[i] = lds_u32(row_sa + (uint32_t)(i * P * 4));
    uint32_t at[NB];
#pragma unroll
    for (int i = 0; i < NB; ++i) at[i] = base_sa + (lds_u16(off_sa + (e[i] & (WIDE ? 63u : 31u)) * 2u) << 4);
    int32_t D = D0, PM = PM0;
    int32_t pm[NB], ce[NB], ndm[NB];
#pragma unroll
    for (int i = 0; i < NB; ++i) {
        // slo/shi hold the SCHEDULED jobs: the funnel shift moves the job's bit to the
        // sign, and its sign extension (IMAD.HI, FMA pipe) is -1 for a scheduled job
        const uint32_t f = WIDE ? __funnelshift_l(0u, (e[i] & 32u) ? shi : slo, e[i])
                                : __funnelshift_l(0u, slo, e[i]);
        const int32_t sched = __mulhi((int32_t)f, 1);
        const int32_t c = (int32_t)__byte_perm(e[i], 0u, 0x4421);  // bytes 1..2
        const int32_t nd = __mulhi((int32_t)e[i], 256);             // -d (top byte, signed)
        // non-members: c - kOff (IMAD, FMA pipe) can never win a max; -d -> 0 (LOP3, ALU
        // pipe) -- one select per pipe keeps the two pipes balanced
        ce[i] = c + sched * kOff;
        ndm[i] = nd & ~sched;
        pm[i] = PM;
        PM = max(PM, D + ce[i]);
        D -= ndm[i];
    }
    int32_t SM = SM0;
#pragma unroll
    for (int i = NB - 1; i >= 0; --i) {
        const int32_t Db = D + ndm[i];  // D before position i
        sts_u16(at[i], max(pm[i], SM + ndm[i]));
        SM = max(SM, Db + ce[i]);
        D = Db;
    }
    return SM;
}

// Grid-wide barrier of the persistent batch kernel (cooperative launch: every CTA is
// resident).  Thread 0 of each CTA releases the CTA's writes and arrives; the last one
// resets the count and bumps the generation; the others spin on it with acquire loads.
__device__ __forceinline__ void batch_grid_sync(uint32_t* count, uint32_t* gen) {
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t g0, g, old;
        asm volatile("ld.relaxed.gpu.u32 %0, [%1];" : "=r"(g0) : "l"(gen) : "memory");
        // arrive: release the CTA's writes (ordered before by the CTA barrier), and the
        // last arriver acquires everyone's
        asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(count) : "memory");
        if (old == gridDim.x - 1) {
            asm volatile("st.relaxed.gpu.u32 [%0], 0;" ::"l"(count) : "memory");
            asm volatile("st.release.gpu.u32 [%0], %1;" ::"l"(gen), "r"(g0 + 1u) : "memory");
        } else {
            // spin with relaxed loads (an acquire load invalidates the SM's L1, which would
            // keep evicting the planning thread's working set on CTA 0's SM), then one fence
            do {
                asm volatile("ld.relaxed.gpu.u32 %0, [%1];" : "=r"(g) : "l"(gen) : "memory");
            } while (g == g0);
            asm volatile("fence.acq_rel.gpu;" ::: "memory");
        }
    }
    __syncthreads();
}

// Two parents per thread in 16x2 SIMD (n <= 20 at 2 CTAs/SM, where the 168-register
// budget holds six 20-entry arrays): one row entry feeds both parents' max-plus chains,
// each as one VIADDMNMX.S16x2 / VIADD.16x2.  Values fit int16 for n <= 20 (|D| <= 1960,
// c < 2^12); a scheduled job gets c = -16384 and d = 0 in its half.  The backward pass
// uses the suffix form  T = max(d_i + T, c_i),  M'_x = max(prefmax_<x, D_<x + T_x),
// which needs no subtraction (rows hold +d for this path).  Parent 1 may be a copy of
// parent 0 with every job scheduled (odd tail): its half is stored first, so parent
// 0's store to the same slot wins.
template <int NB, int P>
__device__ __forceinline__ void scan_pair16(uint32_t row_sa, uint32_t s0, uint32_t s1, uint32_t off0,
                                            uint32_t off1, uint32_t base0, uint32_t base1) {
    constexpr uint32_t kNeg16x2 = 0xC000C000u;  // (-16384, -16384)
    uint32_t at0[NB], at1[NB], ce2[NB], dm2[NB], pm2[NB], dp2[NB];
    uint32_t D2 = 0u, PM2 = kNeg16x2;
#pragma unroll
    for (int i = 0; i < NB; ++i) {
        const uint32_t e = lds_u32(row_sa + (uint32_t)(i * P * 4));
        const uint32_t code2 = (e & 31u) * 2u;
        at0[i] = base0 + (lds_u16(off0 + code2) << 4);  // tables hold offsets / 16
        at1[i] = base1 + (lds_u16(off1 + code2) << 4);
        const uint32_t f0 = __funnelshift_l(0u, s0, e), f1 = __funnelshift_l(0u, s1, e);
        uint32_t m2, c2, d2;
        asm("prmt.b32 %0, %1, %2, 0xFFBB;" : "=r"(m2) : "r"(f0), "r"(f1));  // 0xFFFF where scheduled
        asm("prmt.b32 %0, %1, 0, 0x2121;" : "=r"(c2) : "r"(e));             // (c, c)
        asm("prmt.b32 %0, %1, 0, 0xB3B3;" : "=r"(d2) : "r"(e));             // (d, d) sign-extended
        ce2[i] = (c2 & ~m2) | (kNeg16x2 & m2);
        dm2[i] = d2 & ~m2;
        pm2[i] = PM2;
        dp2[i] = D2;
        PM2 = __viaddmax_s16x2(D2, ce2[i], PM2);
        D2 = __vadd2(D2, dm2[i]);
    }
    uint32_t T2 = kNeg16x2;
#pragma unroll
    for (int i = NB - 1; i >= 0; --i) {
        const uint32_t r2 = __viaddmax_s16x2(dp2[i], T2, pm2[i]);
        sts_u16(at1[i], (int32_t)(r2 >> 16));
        sts_u16(at0[i], (int32_t)r2);
        T2 = __viaddmax_s16x2(dm2[i], T2, ce2[i]);
    }
}



// OCC = target CTAs per SM: 2 -> up to 168 registers, 3 -> 112 (smaller chunks too)
// DIR: false = staged placement only (the big-pool kernel, untouched by the direct path),
// true = direct placement capable (single-wave pools; Pool::direct decides at run time when
// place_hint < 0)
// BATCH: the persistent form -- one cooperative launch runs a whole device-planned batch:
// per round CTA 0 closes the previous round and plans this one (loop_plan.cuh), a grid
// barrier, [the leaves and the best leaf's schedule], K2 with direct placement, a grid
// barrier.  The row tables stay staged (registers / shared memory) across the rounds and
// no kernel is launched between them.  Every round must fit one wave (the host runs it
// only when the batch's worst-case chunk count does).
template <int N, int M, int OCC, bool DIR, bool BATCH = false>
__global__ void __launch_bounds__(192, OCC) k2_v2_kernel(DevTables t, const Pool* __restrict__ pool_arg,
                                                   int first_seg, int cmax, int place_hint, int frozen,
                                                   RoundState* rs, ChunkOut out, LoopState* ls) {
    constexpr int P = M * (M - 1) / 2;
    // Phase B: the 16x2 grouped form at 2 CTAs/SM (168 registers); at 3 CTAs/SM (96
    // registers) the per-pair form over q-ordered Mq rows, which spills least there
    constexpr bool kGroupedB = OCC == 2;
    constexpr bool kDual16 = OCC == 2 && N == 20;  // Phase A: two parents per thread, 16x2
    extern __shared__ __align__(16) unsigned char smem[];
    // place_hint: 0 staged placement (known to the host), 1 direct, -1 read Pool::direct
    // (device-planned loop).  Staged: place_kernel may be scheduled onto SMs as this
    // grid's CTAs retire (programmatic dependent launch; it waits for the grid's
    // completion before reading anything).  Direct: the dependents may not take SM room
    // before every CTA of this grid is resident (its CTAs wait for each other).
    if (!DIR) asm volatile("griddepcontrol.launch_dependents;");
    const int n = t.n, W = t.W;
    const V2Layout L = v2_layout(n, M, P, cmax, blockDim.x, N, OCC);
    uint64_t* s_um = (uint64_t*)(smem + L.um);  // unscheduled jobs of each parent
    constexpr int RW = N <= 32 ? 32 : 64;
    uint16_t* s_off = (uint16_t*)(smem + L.rank);  // per parent: Mq byte offset of each job code
    int32_t* s_R = (int32_t*)(smem + L.R);
    int32_t* s_load = (int32_t*)(smem + L.load);
    uint32_t* s_mins = (uint32_t*)(smem + L.mins);
    uint8_t* s_amin = (uint8_t*)(smem + L.amin);
    unsigned char* s_Mq = smem + L.Mq;
    int32_t* s_p = (int32_t*)(smem + L.p);
    uint8_t* s_pre = (uint8_t*)(smem + L.pre);
    int64_t* s_slot = (int64_t*)(smem + L.wsum);
    int32_t* s_wsum = (int32_t*)(smem + L.wsum + 16);
    const int tid = threadIdx.x, bd = blockDim.x, lane = tid & 31, warp = tid >> 5;
    const int nwarps = bd >> 5;
    const int G = bd / P;
    const int q = tid % P, g = tid / P;
    const bool a_lane = g < G;

    int16_t* s_tl = (int16_t*)(smem + L.tl);
    for (int x = tid; x < n * M; x += bd) {
        s_p[x] = t.p[x];
        s_tl[x] = (int16_t)t.tails[x];  // < 0x7FFF (checked at configuration)
    }

    // Johnson rows repacked for the scans, one word per (position, pair), [i][q]:
    //   bits 0..4 = 31 - (job & 31) (a left funnel shift by it moves the job's U bit
    //   to the sign bit), bit 5 = job >> 5 (which 32-bit word of U, wide variant),
    //   bits 8..23 c, bits 24..31 -d (int8).  Padding positions i >= n read the top bit
    //   of U (bit 31, or 63 in the wide variant), which is 0 when padding exists.
    uint32_t* s_row = (uint32_t*)(smem + L.row);
    // DevTables::rowk2 holds exactly these words for the configured variant: one TMA bulk
    // copy (cp.async.bulk, completion counted on an mbarrier) stages them while the CTA's
    // threads stage p / tails and clear Mq; the per-thread repacking loop is the fallback
    __shared__ __align__(8) uint64_t s_tma_bar;
    const uint32_t tma_bar = (uint32_t)__cvta_generic_to_shared(&s_tma_bar);
    const bool tma = t.rowk2 != nullptr;
    if (tma && tid == 0) {
        const uint32_t bytes = (uint32_t)(N * P * 4);  // a multiple of 16 (N in {20, 32, 64})
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(tma_bar) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(tma_bar), "r"(bytes) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(s_row)),
                     "l"(t.rowk2), "r"(bytes), "r"(tma_bar)
                     : "memory");
    }
    for (int x = tid; x < N * P && !tma; x += bd) {
        uint32_t v = N <= 32 ? 0u : 32u;
        if (x < n * P) {
            uint32_t e = t.jm[x];
            const uint32_t j = (uint32_t)entry_job(e);
            v = (31u - (j & 31u)) | (j & 32u) | ((uint32_t)entry_c(e) << 8) |
                ((uint32_t)(kDual16 ? entry_d(e) : -entry_d(e)) << 24);
        }
        s_row[x] = v;
    }
    // 32-bit shared addresses: each scan step is one LDS [reg + immediate]
    const uint32_t row_sa = (uint32_t)__cvta_generic_to_shared(s_row + q);
    for (int x = tid; x < (int)((cmax + v2_dummy_rows(P)) * L.rowb / 16); x += bd)  // padding slots stay 0
        ((uint4*)s_Mq)[x] = make_uint4(0u, 0u, 0u, 0u);
    if (tma) {  // the rows are in (the barrier's phase 0 completes with the copy's bytes)
        __syncthreads();  // (the mbarrier's initialisation, for every thread)
        uint32_t done = 0;
        while (!done)
            asm volatile(
                "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\nselp.u32 %0, 1, 0, p;\n}"
                : "=r"(done)
                : "r"(tma_bar)
                : "memory");
        __syncthreads();
    }

    // one round over `pool` (the kernel's argument, or the batch's shared-memory copy)
    auto k2_round = [&](const Pool* __restrict__ pool, RoundState* rs) {
    // the round's bound, semantics and first internal segment come from the pool
    // (written by the host, or by the device-side planner of the batched explorer loop)
    asm volatile("griddepcontrol.wait;" ::: "memory");  // the pool upload kernel (PDL)
    const bool direct = DIR && (place_hint < 0 ? pool->direct != 0 : place_hint == 1);
    if (DIR && !direct) asm volatile("griddepcontrol.launch_dependents;");
    k2_stamp_begin(rs);
    const int32_t ub = pool->ub;
    frozen = pool->frozen;
    first_seg = pool->first_internal;
    if (first_seg >= pool->nseg) return;
    int32_t ub_eff = ub;
    if (!frozen) {
        // (batch: written this kernel by other CTAs -- an L2 read)
        unsigned long long inv = BATCH ? __ldcg(&rs->leaf_inv) : rs->leaf_inv;
        int32_t v = (int32_t)((~inv) >> 32);
        if (inv != 0ull && v < ub_eff) ub_eff = v;
    }

    const int64_t c_begin = pool->seg[first_seg].chunk_base;
    const int64_t c_end = pool->nchunks;
    const int ppc_lim = pool->ppc_lim;
    // Chunk staging.  At 2 CTAs/SM the parents of the NEXT chunk are loaded into
    // registers while this chunk runs Phase A / B (software pipelining: the global --
    // or, host-resident, host-link -- latency of the staging loads hides behind
    // compute), and the next ticket is claimed during setup, so a chunk costs one
    // barrier less.  At 3 CTAs/SM (96 registers) the staging loads stay direct.
    constexpr bool kPipe = OCC == 2 && N != 32;  // (N = 32: the prefetch registers spill)
    constexpr int kPpcCt = N <= 32 ? 32 : 16;                  // >= parents per chunk (v2_ppc_cap)
    constexpr int kPfPre = (kPpcCt * N + 191) / 192;           // prefix bytes per thread
    constexpr int kPfPreW = (kPpcCt * (N / 4) + 191) / 192;    // prefix words per thread
    constexpr int kPfHead = (kPpcCt * M + 191) / 192;          // heads per thread
    // n % 4 == 0 (Ta 20x5 / 20x10 / 20x20): prefix rows are word aligned everywhere (device
    // buckets and host arena blocks are 256-byte aligned), so they are staged as 32-bit
    // words -- a quarter of the loads, which matters most over the host link
    const bool n4 = (n & 3) == 0;
    uint32_t pf_pre[kPipe ? kPfPre : 1];
    int32_t pf_head[kPipe ? kPfHead : 1];
    uint64_t pf_mask = 0;
    auto chunk_geo = [&](int64_t c, int& s_, int& depth_, int& np_, int64_t& p0_) {
        s_ = v2_find_segment(pool, first_seg, c);
        const Segment& g_ = pool->seg[s_];
        depth_ = g_.depth;
        int ppc_ = min(cmax / (n - depth_), v2_ppc_cap(N, OCC));
        if (ppc_lim > 0) ppc_ = min(ppc_, ppc_lim);  // small pools spread over the wave
        p0_ = (c - g_.chunk_base) * ppc_;
        np_ = (int)(g_.count - p0_ < ppc_ ? g_.count - p0_ : ppc_);
    };
    auto prefetch = [&](int64_t c) {  // global loads of chunk c's parents into registers
        if (c >= c_end) return;
        int s_, depth_, np_;
        int64_t p0_;
        chunk_geo(c, s_, depth_, np_, p0_);
        const Segment& g_ = pool->seg[s_];
        const bool cpt_ = g_.src.heads == nullptr;  // compact rows: prefixes only
        if (n4) {
            const int wpr = (depth_ + 3) >> 2;
            const uint32_t* src32 = reinterpret_cast<const uint32_t*>(g_.src.prefix);
#pragma unroll
            for (int u = 0; u < kPfPreW; ++u) {
                const int x = tid + u * 192;
                if (x < np_ * wpr) {
                    const int pp = x / wpr, w = x - pp * wpr;
                    pf_pre[u] = src32[((g_.first + g_.step * (p0_ + pp)) * n >> 2) + w];
                }
            }
        } else {
#pragma unroll
            for (int u = 0; u < kPfPre; ++u) {
                const int x = tid + u * 192;
                if (x < np_ * depth_) {
                    const int pp = x / depth_, i = x - pp * depth_;
                    pf_pre[u] = g_.src.prefix[(g_.first + g_.step * (p0_ + pp)) * n + i];
                }
            }
        }
#pragma unroll
        for (int u = 0; u < kPfHead; ++u) {
            const int x = tid + u * 192;
            if (x < np_ * M && !cpt_) {
                const int pp = x / M, k = x - pp * M;
                pf_head[u] = g_.src.heads[(g_.first + g_.step * (p0_ + pp)) * M + k];
            }
        }
        if (tid < np_ && !cpt_) pf_mask = g_.src.masks[(g_.first + g_.step * (p0_ + tid)) * W];
    };
    // direct placement: CTA i owns chunk c_begin + i (fixed-grid launches may have more
    // CTAs than chunks; those have nothing to do)
    int64_t chunk = (DIR && direct) ? c_begin + blockIdx.x : claim_chunk(rs, c_begin, s_slot);
    if (DIR && direct && chunk >= c_end) return;
    // the prologue's row tables complete before any scan reads them: claim_chunk's barrier
    // does this in the staged form (the row loads are non-volatile asm, which the compiler
    // may hoist up to the nearest barrier -- racecheck caught them above the staging one)
    if (DIR && direct) __syncthreads();
    if constexpr (kPipe) prefetch(chunk);
    while (chunk < c_end) {
        int s, depth, np;
        int64_t p0;
        chunk_geo(chunk, s, depth, np, p0);
        const Segment& sg = pool->seg[s];
        const int r = n - depth;
        const int nc = np * r;
        const uint64_t valid = n >= 64 ? ~0ull : ((1ull << n) - 1ull);
        const bool compact = sg.src.heads == nullptr;  // prefix-only rows (host-resident tree)
        if constexpr (kPipe) {
            if (n4) {
                const int wpr = (depth + 3) >> 2;
#pragma unroll
                for (int u = 0; u < kPfPreW; ++u) {
                    const int x = tid + u * 192;
                    if (x < np * wpr) {
                        const int pp = x / wpr, w = x - pp * wpr;
                        reinterpret_cast<uint32_t*>(s_pre)[pp * (RW / 4) + w] = pf_pre[u];
                    }
                }
            } else {
#pragma unroll
                for (int u = 0; u < kPfPre; ++u) {
                    const int x = tid + u * 192;
                    if (x < np * depth) {
                        const int pp = x / depth, i = x - pp * depth;
                        s_pre[pp * RW + i] = (uint8_t)pf_pre[u];
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < kPfHead; ++u) {
                const int x = tid + u * 192;
                if (x < np * M && !compact) s_R[x] = pf_head[u];
            }
            if (tid < np && !compact) s_um[tid] = ~pf_mask & valid;
        } else {
            const NodeStore src = sg.src;
            const int64_t first = sg.first, step = sg.step;
            if (n4) {
                const int wpr = (depth + 3) >> 2;
                const uint32_t* src32 = reinterpret_cast<const uint32_t*>(src.prefix);
                for (int x = tid; x < np * wpr; x += bd) {
                    const int pp = x / wpr, w = x - pp * wpr;
                    reinterpret_cast<uint32_t*>(s_pre)[pp * (RW / 4) + w] =
                        src32[((first + step * (p0 + pp)) * n >> 2) + w];
                }
            } else {
                for (int x = tid; x < np * depth; x += bd) {
                    int pp = x / depth, i = x - pp * depth;
                    s_pre[pp * RW + i] = src.prefix[(first + step * (p0 + pp)) * n + i];
                }
            }
            for (int pp = tid; pp < np && !compact; pp += bd) {
                int64_t node = first + step * (p0 + pp);
                s_um[pp] = ~src.masks[node * W] & valid;
            }
            for (int x = tid; x < np * M && !compact; x += bd) {
                int pp = x / M, k = x - pp * M;
                s_R[x] = src.heads[(first + step * (p0 + pp)) * M + k];
            }
        }
        __syncthreads();
        if (kPipe && tid == 0)  // next chunk
            *s_slot = (DIR && direct) ? c_end : c_begin + (int64_t)atomicAdd(&rs->ticket, 1u);
        if (compact) {  // heads and scheduled set folded from the staged prefixes
            if (tid < np) {
                const uint8_t* pre = s_pre + tid * RW;
                int32_t h[M];
                heads_from_prefix<M>(pre, depth, [&](int j, int k) { return s_p[j * M + k]; }, h);
#pragma unroll
                for (int k = 0; k < M; ++k) s_R[tid * M + k] = h[k];
                uint64_t sm = 0;
                for (int i = 0; i < depth; ++i) sm |= 1ull << pre[i];
                s_um[tid] = ~sm & valid;
            }
            __syncthreads();
        }
        // per parent and job code: offset (/16) of the job's child row in Mq relative to
        // the parent's first child row (rank of the job among U), or of the dummy row
        // for a scheduled / absent job
        for (int x = tid; x < np * RW; x += bd) {
            const int pp = x / RW, idx = x - pp * RW;
            const int j = (idx & 32) | (31 - (idx & 31));
            const uint64_t um = s_um[pp];
            const bool in = j < n && ((um >> j) & 1ull);
            const int row = in ? __popcll(um & ((1ull << j) - 1ull)) : cmax + pp % v2_dummy_rows(P) - pp * r;
            s_off[x] = (uint16_t)(row * L.rowb / 16);  // rows are 16-byte multiples
        }
        // per (parent, machine): load, two smallest tails (+ argmin, smallest job on ties)
        for (int x = tid; x < np * M; x += bd) {
            int pp = x / M, k = x - pp * M;
            uint64_t um = s_um[pp];
            int32_t load = 0, m1 = 0x7FFF, m2 = 0x7FFF, am = 0;
            if constexpr (N <= 32) {
                // branch-free over all positions: independent (predicated) loads instead of
                // a dependent ffs / load / compare chain per unscheduled job
                const uint32_t u32 = (uint32_t)um;
#pragma unroll
                for (int j = 0; j < N; ++j) {
                    const bool in = (u32 >> j) & 1u;
                    load += in ? s_p[j * M + k] : 0;
                    const int32_t tv = in ? (int32_t)s_tl[j * M + k] : 0x7FFF;
                    const bool lt = tv < m1;
                    m2 = lt ? m1 : min(m2, tv);
                    am = lt ? j : am;
                    m1 = lt ? tv : m1;
                }
            } else {
                while (um) {
                    int j = __ffsll((long long)um) - 1;
                    um &= um - 1;
                    load += s_p[j * M + k];
                    int32_t tv = s_tl[j * M + k];
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
            s_mins[x] = (uint32_t)m1 | ((uint32_t)m2 << 16);
            s_amin[x] = (uint8_t)am;
        }
        __syncthreads();  // rank table and per-machine terms visible to every lane
        int64_t next_chunk = 0;
        if constexpr (kPipe) {
            next_chunk = *s_slot;
            prefetch(next_chunk);
        }
        // ---- Phase A: forward / backward max-plus scans of pair q over parent pp
        if (a_lane && kDual16) {
            const int slot_q = kSlotOf<M>.s[q];
            for (int pp = 2 * g; pp < np; pp += 2 * G) {
                const int pb = pp + 1 < np ? pp + 1 : pp;  // odd tail: a copy with no members
                const uint32_t s0 = ~(uint32_t)s_um[pp];
                const uint32_t s1 = pp + 1 < np ? ~(uint32_t)s_um[pb] : 0xFFFFFFFFu;
                scan_pair16<N, P>(row_sa, s0, s1,
                                  (uint32_t)__cvta_generic_to_shared(s_off + pp * RW),
                                  (uint32_t)__cvta_generic_to_shared(s_off + pb * RW),
                                  (uint32_t)__cvta_generic_to_shared(s_Mq + (size_t)(pp * r) * L.rowb + 2 * slot_q),
                                  (uint32_t)__cvta_generic_to_shared(s_Mq + (size_t)(pb * r) * L.rowb + 2 * slot_q));
            }
        } else if (a_lane) {
            for (int pp = g; pp < np; pp += G) {
                const uint64_t um64 = s_um[pp];
                const uint32_t off_sa = (uint32_t)__cvta_generic_to_shared(s_off + pp * RW);
                // Mq slot of pair q in the grouped row layout, from a __constant__ table (a
                // kernel-long register for it pushed Phase A into spilling at 96 regs)
                const int slot_q = kGroupedB ? (int)kSlotOf<M>.s[q] : q;
                const uint32_t base_sa =
                    (uint32_t)__cvta_generic_to_shared(s_Mq + (size_t)(pp * r) * L.rowb + 2 * slot_q);
                if constexpr (N <= 32) {
                    scan_block<N, P, false>(row_sa, ~(uint32_t)um64, ~0u, off_sa, base_sa, 0, kNeg2, 0);
                } else {
                    // wide: forward pass keeps (D, prefix max) checkpoints every 16
                    // positions; each block is then recomputed and scanned backward
                    const uint32_t lo = ~(uint32_t)um64, hi = ~(uint32_t)(um64 >> 32);  // scheduled
                    int32_t ckD[N / 16], ckP[N / 16];
                    int32_t D = 0, PM = kNeg2;
#pragma unroll
                    for (int b = 0; b < N / 16; ++b) {
                        ckD[b] = D;
                        ckP[b] = PM;
#pragma unroll
                        for (int i = 0; i < 16; ++i) {
                            // volatile: keep the 64 checkpoint-pass loads from being hoisted
                            const uint32_t e = lds_u32_v(row_sa + (uint32_t)((b * 16 + i) * P * 4));
                            const bool in = member(e, lo, hi);
                            const int32_t c = (int32_t)__byte_perm(e, 0u, 0x4421);
                            const int32_t nd = (int32_t)e >> 24;  // -d
                            PM = in ? max(PM, D + c) : PM;
                            D = in ? D - nd : D;
                        }
                    }
                    int32_t SM = kNeg2;
#pragma unroll
                    for (int b = N / 16 - 1; b >= 0; --b)
                        SM = scan_block<16, P, true>(row_sa + (uint32_t)(b * 16 * P * 4), lo, hi,
                                                     off_sa, base_sa, ckD[b], ckP[b], SM);
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
            const uint64_t um = s_um[pp];
            const uint32_t lo = (uint32_t)um;
            const int nlo = __popc(lo);
            const int x = rk < nlo ? (int)__fns(lo, 0, rk + 1)
                                   : 32 + (int)__fns((uint32_t)(um >> 32), 0, rk - nlo + 1);
            myx = x;
            mypp = pp;
            if constexpr (kGroupedB) {
                uint32_t LcE[(M + 1) / 2];  // (Lc_l, Lc_l+1) for even l, int16 halves
                int32_t prev = 0, lb = 0, lc_even = 0;
    #pragma unroll
                for (int k = 0; k < M; ++k) {
                    const int pk = pp * M + k;
                    prev = max(prev, s_R[pk]) + s_p[x * M + k];  // child_heads, instance.hpp:81-89
                    myR[k] = prev;
                    uint32_t mins = s_mins[pk];
                    int32_t mt = (x == (int)s_amin[pk]) ? (int32_t)(mins >> 16) : (int32_t)(mins & 0xFFFFu);
                    const int32_t lc = s_load[pk] - s_p[x * M + k] + mt;
                    lb = max(lb, prev + lc);  // one-machine term (bound.hpp:61-74)
                    if (k & 1) LcE[k >> 1] = ((uint32_t)lc_even & 0xFFFFu) | ((uint32_t)lc << 16);
                    else lc_even = lc;
                }
                if (M & 1) LcE[M >> 1] = ((uint32_t)lc_even & 0xFFFFu) | 0xC0000000u;  // l = M: pad
                // Pairs: Lc_l + max(R_l, R_k + M'_kl).  Lc_l + R_l never exceeds the one-
                // machine term already in lb, so per k only max_l (Lc_l + M'_kl) + R_k is
                // needed: a running max over the k-group's slots, two pairs per 16x2
                // VIADDMNMX (Lc_l + M' < 2^14 for n <= 64).
                const uint4* mrow = (const uint4*)(s_Mq + (size_t)tid * L.rowb);
    #pragma unroll
                for (int k = 0; k < M - 1; ++k) {
                    const int g0 = v2_group_base(M, k) / 2;  // first 32-bit word of the group
                    uint32_t acc = 0xC000C000u;             // (-16384, -16384)
    #pragma unroll
                    for (int w = 0; w < (v2_hi(M) - v2_lo(k)) / 2; ++w) {
                        const int gw = g0 + w;
                        const uint4 v4 = mrow[gw >> 2];
                        const uint32_t word = (gw & 3) == 0 ? v4.x : (gw & 3) == 1 ? v4.y : (gw & 3) == 2 ? v4.z : v4.w;
                        acc = __viaddmax_s16x2(LcE[v2_lo(k) / 2 + w], word, acc);
                    }
                    const int32_t best = max((int32_t)(int16_t)(acc & 0xFFFFu), (int32_t)acc >> 16);
                    lb = max(lb, best + myR[k]);
                }
                mylb = lb;
            } else {
                // 3 CTAs/SM (96 registers): the per-pair form, which keeps fewer values live
                int32_t Lc[M];
                int32_t prev = 0, lb = 0;
#pragma unroll
                for (int k = 0; k < M; ++k) {
                    const int pk = pp * M + k;
                    prev = max(prev, s_R[pk]) + s_p[x * M + k];  // child_heads, instance.hpp:81-89
                    myR[k] = prev;
                    uint32_t mins = s_mins[pk];
                    int32_t mt = (x == (int)s_amin[pk]) ? (int32_t)(mins >> 16) : (int32_t)(mins & 0xFFFFu);
                    Lc[k] = s_load[pk] - s_p[x * M + k] + mt;
                    lb = max(lb, prev + Lc[k]);  // one-machine term (bound.hpp:61-74)
                }
                const uint4* mrow = (const uint4*)(s_Mq + (size_t)tid * L.rowb);
#pragma unroll
                for (int k = 0; k < M - 1; ++k) {
#pragma unroll
                    for (int l = k + 1; l < M; ++l) {
                        const int slot = k * (2 * M - k - 1) / 2 + (l - k - 1);  // q
                        const uint4 v4 = mrow[slot >> 3];
                        const int wi = (slot >> 1) & 3;
                        const uint32_t w = wi == 0 ? v4.x : wi == 1 ? v4.y : wi == 2 ? v4.z : v4.w;
                        const int32_t mq = (slot & 1) ? ((int32_t)w >> 16) : (int32_t)(int16_t)(w & 0xFFFFu);
                        lb = max(lb, Lc[l] + max(myR[l], myR[k] + mq));
                    }
                }
                mylb = lb;
            }
        }
        // ---- prune + stable compaction straight into the destination (one child per thread)
        const bool keep = b_lane && mylb < ub_eff;
        const unsigned ballot = __ballot_sync(0xFFFFFFFFu, keep);
        if (lane == 0) s_wsum[warp] = __popc(ballot);
        __syncthreads();
        int woff = 0, tot = 0;
        for (int w = 0; w < nwarps; ++w) {
            int v = s_wsum[w];
            if (w < warp) woff += v;
            tot += v;
        }
        if (tid == 0) {
            out.count[chunk] = tot;
            out.seg[chunk] = s;
        }
        if (DIR && direct) {
            // every chunk's count in (grid-wide), then this chunk's survivors straight to
            // their bucket rows: segment base + survivors of the segment's earlier chunks
            direct_arrive(rs, s, tot, c_end - c_begin);
            asm volatile("griddepcontrol.launch_dependents;");
            const int64_t before = direct_prefix(out.count, sg.chunk_base, chunk, (int64_t*)(s_wsum + 8));
            if (keep) {
                const int64_t o = sg.dst_base + before + woff + __popc(ballot & ((1u << lane) - 1u));
                const NodeStore dst = sg.dst;
                store_heads<M>(dst.heads + o * M, myR);
                const uint64_t valid = n >= 64 ? ~0ull : ((1ull << n) - 1ull);
                dst.masks[o * W] = (~s_um[mypp] & valid) | (1ull << myx);
                store_prefix(dst.prefix + o * n, s_pre + mypp * RW, depth, myx, n);
            }
            break;  // one chunk per CTA
        }
        if (keep) {
            const int64_t o = chunk * (int64_t)cmax + woff + __popc(ballot & ((1u << lane) - 1u));
            const NodeStore dst = out.nodes;
            store_heads<M>(dst.heads + o * M, myR);
            const uint64_t valid = n >= 64 ? ~0ull : ((1ull << n) - 1ull);
            dst.masks[o * W] = (~s_um[mypp] & valid) | (1ull << myx);
            store_prefix(dst.prefix + o * n, s_pre + mypp * RW, depth, myx, n);
            out.lb[o] = mylb;
        }
        if constexpr (kPipe) {
            __syncthreads();  // this chunk's staging arrays fully consumed
            chunk = next_chunk;
        } else {
            chunk = claim_chunk(rs, c_begin, s_slot);
        }
    }
    k2_stamp_end(rs);
    if (!BATCH && DIR && direct) direct_finish(pool, rs, n, c_end - c_begin);
    };  // k2_round

    if constexpr (!BATCH) {
        k2_round(pool_arg, rs);
    } else {
        // batch state: CTA 0 keeps the bucket sizes in shared memory for the whole batch;
        // every CTA copies each round's plan (written by CTA 0 during this kernel, so read
        // from L2, never through the read-only path) into shared memory
        Pool* gpool = const_cast<Pool*>(pool_arg);
        Pool* s_pool = (Pool*)(smem + L.total);
        int64_t* s_cnt = (int64_t*)(smem + L.total + b16(offsetof(Pool, seg) + (size_t)(n + 1) * sizeof(Segment)));
        int64_t* s_cap = s_cnt + (n + 1);
        NodeStore* s_bucket = (NodeStore*)(s_cap + (n + 1));
        const bool lead = blockIdx.x == 0 && tid == 0;
        if (blockIdx.x == 0) {
            for (int d = tid; d <= n; d += bd) s_cnt[d] = ls->cnt[d];
            stage_buckets(ls, s_bucket, s_cap, n, tid, bd);
            for (int i = tid; i < kLoopMax; i += bd) ls->rec[i].valid = 0;  // see loop_step_kernel
        }
        // Rounds alternate between two (Pool, RoundState) buffers: CTA 0 closes round r and
        // plans round r + 1 right after its own K2 chunk, while the other CTAs still write
        // their survivors (the plan needs only the counts, final at direct_arrive), so a
        // round costs one grid barrier plus K2's arrival count.  Round r + 1's buffers were
        // last used by round r - 1, which every CTA left at round r's barrier.
        const LoopBuckets bk{s_bucket, s_cap};
        auto plan_publish = [&](int round) {  // CTA 0
            if (warp == 0) plan_round(t, ls, s_pool, rs + (round & 1), round, s_cnt, bk, lane);
            if (lead) {
                if (s_pool->nseg > 0 && s_pool->nchunks > 0 && !s_pool->direct) {
                    ls->stop = 6;  // more chunks than one wave: the host runs this round itself
                    s_pool->nseg = 0;
                }
                if (round < kLoopMax) ls->rec[round].tp = loop_ns();
            }
            __syncthreads();
            pool_store(gpool + (round & 1), s_pool, s_pool->nseg, tid, bd);
        };
        __syncthreads();  // CTA 0's staged bucket state
        if (blockIdx.x == 0) plan_publish(0);
        int round = 0;
        for (;; ++round) {
            Pool* gp = gpool + (round & 1);
            RoundState* rsr = rs + (round & 1);
            batch_grid_sync(&ls->bar_count, &ls->bar_gen);  // plan published, last survivors written
            if (lead && round < kLoopMax) ls->rec[round].tb = loop_ns();
            if (blockIdx.x != 0) pool_load(s_pool, gp, __ldcg(&gp->nseg), tid, bd);
            __syncthreads();
            if (s_pool->nseg == 0) break;
            if (s_pool->seg[0].depth >= n - 2) {
                // leaves (search.hpp:48-55), then the best leaf's schedule before K2 recycles
                // the leaf parents' slots
                leaf_children(t, s_pool, rsr, leaf_segments(s_pool, n));
                batch_grid_sync(&ls->bar_count, &ls->bar_gen);
                if (lead) write_leaf_schedule(t, s_pool, rsr);
                batch_grid_sync(&ls->bar_count, &ls->bar_gen);
            }
            k2_round(s_pool, rsr);
            __syncthreads();
            if (blockIdx.x == 0) {
                if (warp == 0) {
                    close_round(t, ls, s_pool, rsr, round, s_cnt, lane);
                    // the previous round's K2 end stamp is final now (before its buffer is reset)
                    if (lane == 0 && round > 0) ls->rec[round - 1].k2_t1 = __ldcg(&rs[(round - 1) & 1].k2_t1);
                    __syncwarp();
                }
                plan_publish(round + 1);
            }
        }
        if (lead && round > 0 && round - 1 < kLoopMax) ls->rec[round - 1].k2_t1 = __ldcg(&rs[(round - 1) & 1].k2_t1);
        if (blockIdx.x == 0)
            for (int d = tid; d <= n; d += bd) ls->cnt[d] = s_cnt[d];
    }
}

template <int N, int M, int OCC, bool DIR>
cudaError_t v2_setup_one(const DevTables& t, K2Config& c, int device) {
    int optin = 0, sms = 148, per_sm = 1;
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    // dynamic + static shared memory must fit the opt-in limit (direct placement keeps a
    // few bytes of static shared memory)
    cudaFuncAttributes fa;
    cudaError_t e = cudaFuncGetAttributes(&fa, k2_v2_kernel<N, M, OCC, DIR>);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(k2_v2_kernel<N, M, OCC, DIR>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             optin - (int)fa.sharedSizeBytes);
    if (e != cudaSuccess) return e;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k2_v2_kernel<N, M, OCC, DIR>, c.threads, c.smem);
    const int blocks = sms * (per_sm < 1 ? 1 : per_sm);
    // the staged kernel's residency sets the grid; the direct one must hold a whole wave
    // of the same size (its CTAs wait for each other)
    if (!DIR) c.blocks = blocks;
    else if (blocks < c.blocks) return cudaErrorInvalidConfiguration;
    return cudaSuccess;
}

// Shared memory of the persistent batch kernel: the round kernel's, + the round's plan
// (Pool head and up to n + 1 segments) + CTA 0's bucket sizes, capacities and storage.
inline size_t v2_batch_smem(size_t smem, int n) {
    return smem + b16(offsetof(Pool, seg) + (size_t)(n + 1) * sizeof(Segment)) +
           (size_t)(n + 1) * (8 + 8 + sizeof(NodeStore));  // + bucket sizes, capacities, storage
}

// The batch kernel is enabled when a whole grid of c.blocks CTAs is resident with its
// larger shared memory (cooperative launch).
template <int N, int M, int OCC>
void v2_setup_batch(const DevTables& t, K2Config& c, int device) {
    auto kern = k2_v2_kernel<N, M, OCC, true, true>;
    int optin = 0, sms = 148, per_sm = 0, coop = 0;
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, device);
    cudaFuncAttributes fa;
    c.batch = false;
    c.batch_smem = v2_batch_smem(c.smem, t.n);
    if (!coop || cudaFuncGetAttributes(&fa, kern) != cudaSuccess) return;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - (int)fa.sharedSizeBytes) !=
        cudaSuccess)
        return;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, c.threads, c.batch_smem) != cudaSuccess) return;
    c.batch = per_sm * sms >= c.blocks;
}

template <int N, int M, int OCC>
cudaError_t v2_setup(const DevTables& t, K2Config& c, int device) {
    cudaError_t e = v2_setup_one<N, M, OCC, false>(t, c, device);
    if (e != cudaSuccess) return e;
    e = v2_setup_one<N, M, OCC, true>(t, c, device);
    if (e != cudaSuccess) return e;
    v2_setup_batch<N, M, OCC>(t, c, device);
    (void)cudaGetLastError();  // a batch kernel that could not be configured leaves no error behind
    return cudaSuccess;
}

}  // namespace

bool k2_v2_config(const DevTables& t, int device, K2Config* out) {
    int m = t.m, n = t.n;
    if (n > 64 || !(m == 5 || m == 10 || m == 20)) return false;
    K2Config c;
    c.threads = 192;
    // measured (profiles/r01_reading.md): m = 20 runs fastest at 2 CTAs/SM with the
    // 16x2 grouped Phase B, m in {5, 10} at 3 CTAs/SM; FBB_K2_OCC=2|3 overrides
    const char* occ_env = getenv("FBB_K2_OCC");
    int occ = occ_env ? (occ_env[0] == '2' ? 2 : 3) : (m == 20 ? 2 : 3);
    int NN = n <= 20 ? 20 : (n <= 32 ? 32 : 64);
    // 16-bit intermediates must be exact for this instance (DevTables::safe16): every M'
    // is stored as int16; the 2-CTA grouped Phase B adds Lc_l + M' in 16x2; the two-parent
    // scan (N = 20 at 2 CTAs/SM) runs D, D + c and its -16384 neutral in 16x2
    if (!(t.safe16 & kSafeM16)) return false;
    if (occ == 2 && !(t.safe16 & kSafeLcM16)) occ = 3;
    if (NN == 20 && occ == 2 && !(t.safe16 & kSafeDual16)) NN = 32;
    // children per chunk, measured (profiles/r01_k2_iterations.md): larger chunks amortise
    // the per-chunk setup and barriers while the CTAs per SM hold -- Ta021 (m = 20, 2
    // CTAs/SM) 128 -> 160: +3.9 %, 192 drops to 1 CTA/SM; Ta001 (m = 5, 3 CTAs/SM)
    // 112 -> 192: +7 %; the wide variant (n > 32) stays at 128 (160: -22 %)
    c.cmax = NN == 64 ? (occ == 3 ? 112 : 128) : (occ == 3 ? 192 : 160);
    if (const char* cm = getenv("FBB_K2_CMAX")) c.cmax = std::max(32, std::min(192, atoi(cm)));
    // the per-parent u16 offset tables address up to (cmax + dummy rows) Mq rows
    while (c.cmax > 32 && (size_t)(c.cmax + v2_dummy_rows(t.P)) * v2_row_bytes(m) / 16 > 65535) c.cmax -= 16;
    c.variant = occ * 10000 + NN * 100 + m;
    c.ppc_cap = v2_ppc_cap(NN, occ) < (1 << 20) ? v2_ppc_cap(NN, occ) : 0;
    c.jm_in_smem = false;
    c.smem = v2_layout(n, m, t.P, c.cmax, c.threads, NN, occ).total;
    cudaError_t e;
    switch (c.variant) {
        case 22005: e = v2_setup<20, 5, 2>(t, c, device); break;
        case 22010: e = v2_setup<20, 10, 2>(t, c, device); break;
        case 22020: e = v2_setup<20, 20, 2>(t, c, device); break;
        case 23205: e = v2_setup<32, 5, 2>(t, c, device); break;
        case 23210: e = v2_setup<32, 10, 2>(t, c, device); break;
        case 23220: e = v2_setup<32, 20, 2>(t, c, device); break;
        case 32005: e = v2_setup<20, 5, 3>(t, c, device); break;
        case 32010: e = v2_setup<20, 10, 3>(t, c, device); break;
        case 32020: e = v2_setup<20, 20, 3>(t, c, device); break;
        case 33205: e = v2_setup<32, 5, 3>(t, c, device); break;
        case 33210: e = v2_setup<32, 10, 3>(t, c, device); break;
        case 33220: e = v2_setup<32, 20, 3>(t, c, device); break;
        case 26405: e = v2_setup<64, 5, 2>(t, c, device); break;
        case 26410: e = v2_setup<64, 10, 2>(t, c, device); break;
        case 26420: e = v2_setup<64, 20, 2>(t, c, device); break;
        case 36405: e = v2_setup<64, 5, 3>(t, c, device); break;
        case 36410: e = v2_setup<64, 10, 3>(t, c, device); break;
        case 36420: e = v2_setup<64, 20, 3>(t, c, device); break;
        default: return false;
    }
    if (e != cudaSuccess) return false;
    *out = c;
    return true;
}

cudaError_t launch_k2_v2_batch(const DevTables& t, const K2Config& cfg, LoopState* ls, Pool* d_pool,
                               RoundState* rs, ChunkOut out, cudaStream_t stream) {
    if (!cfg.batch) return cudaErrorInvalidValue;
#define V2B_CASE(NN, MM, OO)                                                                     \
    case OO * 10000 + NN * 100 + MM:                                                             \
        return launch_coop(k2_v2_kernel<NN, MM, OO, true, true>, dim3(cfg.blocks), dim3(cfg.threads), \
                           cfg.batch_smem, stream, false, t, (const Pool*)d_pool, 0, cfg.cmax, -1, 0, rs, \
                           out, ls);
    switch (cfg.variant) {
        V2B_CASE(20, 5, 2)
        V2B_CASE(20, 10, 2)
        V2B_CASE(20, 20, 2)
        V2B_CASE(32, 5, 2)
        V2B_CASE(32, 10, 2)
        V2B_CASE(32, 20, 2)
        V2B_CASE(20, 5, 3)
        V2B_CASE(20, 10, 3)
        V2B_CASE(20, 20, 3)
        V2B_CASE(32, 5, 3)
        V2B_CASE(32, 10, 3)
        V2B_CASE(32, 20, 3)
        V2B_CASE(64, 5, 2)
        V2B_CASE(64, 10, 2)
        V2B_CASE(64, 20, 2)
        V2B_CASE(64, 5, 3)
        V2B_CASE(64, 10, 3)
        V2B_CASE(64, 20, 3)
        default: return cudaErrorInvalidValue;
    }
#undef V2B_CASE
}

cudaError_t launch_k2_v2(const DevTables& t, const K2Config& cfg, const Pool* d_pool, int first_seg,
                         int blocks, int place_hint, int frozen, RoundState* rs, ChunkOut out,
                         cudaStream_t stream, bool pdl) {
    // direct placement waits for every CTA of the grid: gang-schedule it (cooperative
    // launch, ~2-3 us more per launch) whenever another context of this process may run
    // kernels on the device concurrently; alone on the device, a single-wave grid that fits
    // the occupancy-derived CTA count is resident as a whole anyway
    int dev = 0;
    cudaGetDevice(&dev);
    const bool coop = place_hint != 0 && device_shared(dev);
#define V2_CASE(NN, MM, OO)                                                                   \
    case OO * 10000 + NN * 100 + MM:                                                          \
        return place_hint == 0                                                                \
                   ? launch_pdl(k2_v2_kernel<NN, MM, OO, false>, dim3(blocks), dim3(cfg.threads), cfg.smem, \
                                stream, pdl, t, d_pool, first_seg, cfg.cmax, 0, frozen, rs, out, \
                                (LoopState*)nullptr)                                              \
                   : coop ? launch_coop(k2_v2_kernel<NN, MM, OO, true>, dim3(blocks), dim3(cfg.threads), \
                                        cfg.smem, stream, pdl, t, d_pool, first_seg, cfg.cmax, place_hint, \
                                        frozen, rs, out, (LoopState*)nullptr)                     \
                          : launch_pdl(k2_v2_kernel<NN, MM, OO, true>, dim3(blocks), dim3(cfg.threads), \
                                       cfg.smem, stream, pdl, t, d_pool, first_seg, cfg.cmax, place_hint, \
                                       frozen, rs, out, (LoopState*)nullptr);
    switch (cfg.variant) {
        V2_CASE(20, 5, 2)
        V2_CASE(20, 10, 2)
        V2_CASE(20, 20, 2)
        V2_CASE(32, 5, 2)
        V2_CASE(32, 10, 2)
        V2_CASE(32, 20, 2)
        V2_CASE(20, 5, 3)
        V2_CASE(20, 10, 3)
        V2_CASE(20, 20, 3)
        V2_CASE(32, 5, 3)
        V2_CASE(32, 10, 3)
        V2_CASE(32, 20, 3)
        V2_CASE(64, 5, 2)
        V2_CASE(64, 10, 2)
        V2_CASE(64, 20, 2)
        V2_CASE(64, 5, 3)
        V2_CASE(64, 10, 3)
        V2_CASE(64, 20, 3)
        default: return cudaErrorInvalidValue;
    }
#undef V2_CASE
    return cudaGetLastError();
}

}  // namespace fbb
