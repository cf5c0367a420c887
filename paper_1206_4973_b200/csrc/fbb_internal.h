// fbb_internal.h -- shared definitions of the B200 hot path (device tables,
// node batches, kernel entry points).  Not part of the C-ABI.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <string>
#include <vector>

#include "flowbb_b200.h"

namespace fbb {

constexpr int kMaxJobs = 256;     // uint8 prefixes
constexpr int kMaxMachines = 64;  // per-node machine arrays staged in smem / registers
constexpr int kMaxWords = (kMaxJobs + 63) / 64;

// Packed Johnson-order table entry for (machine pair q, position i):
//   bits  0.. 8  job index j            (n <= 512)
//   bits  9..17  d + 256 = a - b + 256   (|a - b| <= 255)
//   bits 18..31  c = a + lag             (c < 16384)
// with a = p[j][k], b = p[j][l], lag = tail(j,k) - p(j,l) - tail(j,l)
// (bound.hpp:84-86).  Johnson's rule with lags is rewritten as the max-plus
// form   t_B = sum_U b + max(r_l, r_k + max_i (D_<i + c_i)),  D_<i = sum of d
// over the jobs of U before position i, which is the simulation
// t_A += a; t_B = max(t_B, t_A + lag) + b of bound.hpp:37-43 unrolled.
__host__ __device__ inline uint32_t pack_entry(int job, int d, int c) {
    return (uint32_t)job | ((uint32_t)(d + 256) << 9) | ((uint32_t)c << 18);
}
__host__ __device__ inline int entry_job(uint32_t e) { return (int)(e & 0x1FFu); }
__host__ __device__ inline int entry_d(uint32_t e) { return (int)((e >> 9) & 0x1FFu) - 256; }
__host__ __device__ inline int entry_c(uint32_t e) { return (int)(e >> 18); }

// Device-resident instance tables (built once per context, tables.cu).
struct DevTables {
    int n, m, P, W;
    int32_t* p;       // n*m job-major (instance.hpp:65)
    int32_t* tails;   // n*m (instance.hpp:38-45)
    uint32_t* jm;     // n*P, position-major: jm[i*P + q]
    int16_t* pair_k;  // P
    int16_t* pair_l;  // P
    // The same Johnson rows repacked for the register-row kernels (n*P, [i][q]):
    //   bits 0..4  31 - (j & 31)   (a left funnel shift by it moves j's U bit to bit 31)
    //   bits 5..7  j >> 5          (which 32-bit word of U)
    //   bits 8..23 c,  bits 24..31 d as int8
    // so bits 0..7 are also the index of j in the per-parent rank tables.  Null when
    // some |d| > 127 (then only the generic kernel runs).
    uint32_t* rowpk;
    // The rows again for k2_v3 (n*P, [i][q]): bits 0..7 j, bits 8..15 d as int8,
    // bits 16..31 c -- membership and the child slot come from a per-parent table
    // indexed by j, so no code/shift field is needed.  Null when rowpk is.
    uint32_t* rowv3;
    // Unpacked Johnson rows (n*P, [i][q]): {job, d, c, 0} as int32 -- any instance whose
    // total processing time fits int32 arithmetic; read by the kWide kernels.  Null unless
    // some kernel needs it (values outside the packed or the int16 ranges).
    int4* jw;
    // K1 v3 rows (n*P, [i][q]): bits 0..7 j, 8..15 d as int8, 16..31 c + k1_c0, and the
    // two biases of its 16x2 chains (bound_v3.cu): k1_bias lifts the low half of D above
    // zero, k1_c0 lifts every member's candidate above every non-member's.  Null unless
    // kSafeK1x2.
    uint32_t* rowk1;
    // K2 v2's rows exactly as its prologue stages them for the configured variant (N
    // positions, [i][q], the 16x2 two-parent scan's +d or the others' -d), so a CTA stages
    // them with one TMA bulk copy.  Null when K2 v2 is not configured.
    uint32_t* rowk2;
    int32_t k1_bias, k1_c0;
    // Which 16-bit intermediates are exact for this instance (build_host_tables' range
    // analysis): kSafeM16 = every M' fits int16, kSafeLcM16 = every Lc_l + M'_kl fits int16,
    // kSafeDual16 = the 16x2 two-parent scan (D, D + c, the -16384 neutral) fits.
    int32_t safe16;
};
constexpr int32_t kSafeM16 = 1, kSafeLcM16 = 2, kSafeDual16 = 4;
constexpr int32_t kTablesPacked = 8;  // safe16 bit: jm holds the packed rows
constexpr int32_t kSafeK1x2 = 16;     // K1's biased 16x2 chains fit (bound_v3.cu)

// Host copy of the same tables (for tests of the table builder).
struct HostTables {
    int n = 0, m = 0, P = 0, W = 0;
    int64_t max_abs_d = 0;  // max |p[j][k] - p[j][l]| over pairs
    bool packed = true;     // every entry fits pack_entry (|d| <= 255, c < 2^14)
    // Range analysis of the max-plus intermediates (bound.hpp:27-44 in the form of
    // fbb_internal.h's pack_entry comment), over every unscheduled set U:
    //   D_<i in [sum of negative d, sum of positive d] of the pair,  c in [0, max c],
    //   so M' = max(D_<i + c_i) <= m_hi = max_q (sum_j max(d,0) + max_j c) and >= m_lo,
    //   and Lc_l = load_l - p[x][l] + min tail_l <= lc_max = max_l (sum_j p[j][l] + max_j tail).
    int64_t m_hi = 0, m_lo = 0, lc_max = 0;
    int64_t spos_max = 0;   // max_q sum_j max(d, 0)
    int32_t safe16 = 0;     // kSafe* bits derived from the above
    std::vector<int32_t> p, tails;
    std::vector<uint32_t> jm;   // packed rows (zeros when !packed)
    std::vector<int32_t> jw;    // unpacked rows, 4 int32 per entry {job, d, c, 0}
    std::vector<int16_t> pair_k, pair_l;
};

// Builds the Johnson orders: for each pair (k<l), jobs sorted by
// (group, key, job) -- group 0 if a+lag < lag+b, ascending a+lag, else
// group 1 descending lag+b -- which is the order std::stable_sort gives over
// the ascending unscheduled list (bound.hpp:28-36) restricted to any subset.
// Returns FBB_E_RANGE only when the instance exceeds int32 arithmetic (total
// processing time > 2^30) or the device limits (n <= 256, m <= 64); instances whose
// values do not fit the packed / 16-bit forms run the kWide kernels.
int build_host_tables(const int32_t* p, int n, int m, HostTables* out, std::string* why);
int upload_tables(const HostTables& h, DevTables* d, std::string* why);
void free_tables(DevTables* d);

// ---- K1 ----------------------------------------------------------------------------------
struct K1Config {
    bool wide = false;   // k1_bound_kernel over DevTables::jw (unpacked rows)
    int threads = 256;
    int tile = 32;       // nodes per tile
    bool jm_in_smem = true;
    int variant = 0;     // 0: k1_bound_kernel; 1/2/8: k1v2_kernel<NW> (bound_v2.cu);
                         // 100 + NW: k1v3_kernel<NW> (bound_v3.cu)
    int blocks = 0;      // persistent grid
    size_t smem = 0;
};
K1Config k1_config(const DevTables& t, int device);
cudaError_t launch_k1(const DevTables& t, const K1Config& cfg, const uint64_t* masks,
                      const int32_t* heads, const int32_t* depth, int64_t count, int32_t* lb,
                      cudaStream_t stream);

// K1 v2 (bound_v2.cu): packed rows through L1, NPT nodes per row sweep; false when
// the instance does not qualify (|d| > 127, m > 20, n > 256).
bool k1v2_config(const DevTables& t, int device, K1Config* out);
cudaError_t launch_k1v2(const DevTables& t, const K1Config& cfg, const uint64_t* masks,
                        const int32_t* heads, const int32_t* depth, int64_t count, int32_t* lb,
                        cudaStream_t stream);

// K1 v3 (bound_v3.cu): 16x2 SIMD chains, 16 nodes per row sweep; false when the instance
// does not qualify (no rowv3, m > 20, n > 256, or not kSafeK1x2).  variant = 100 + NW.
bool k1v3_config(const DevTables& t, int device, K1Config* out);
cudaError_t launch_k1v3(const DevTables& t, const K1Config& cfg, const uint64_t* masks,
                        const int32_t* heads, const int32_t* depth, int64_t count, int32_t* lb,
                        cudaStream_t stream);

// Synthetic pool (synth.cu): node i = random_node(seed, i) in SoA, device pointers.
cudaError_t launch_synth(const DevTables& t, uint64_t seed, int64_t count, int min_depth, int max_depth,
                         uint64_t* masks, int32_t* heads, int32_t* depth, uint8_t* prefix,
                         cudaStream_t stream);

// ---- K2 ----------------------------------------------------------------------------------
// A pool is a list of parent segments, each a run of parents of one depth read
// from a node store either forward (a host-supplied batch) or backward (the
// top of a pending bucket, LIFO pop order, pending.hpp:30-37).
constexpr int kMaxSegments = kMaxJobs + 1;

struct NodeStore {     // SoA view; node i at masks[i*W], heads[i*m], prefix[i*n]
    uint64_t* masks;
    int32_t* heads;
    uint8_t* prefix;
};

struct Segment {
    NodeStore src;
    int64_t first;       // index of the segment's first parent in src
    int64_t step;        // +1 forward (host batch), -1 backward (bucket top, LIFO)
    int64_t count;       // parents
    int32_t depth;       // parent depth
    int32_t pad;
    int64_t child_base;  // batch position of the segment's first child
    int64_t chunk_base;  // first chunk index of the segment
    NodeStore dst;       // where survivors go (depth+1 bucket, or the output batch)
    int64_t dst_base;    // < 0: one contiguous output for the whole pool
    int32_t* dst_lb;     // optional survivor bounds
};

struct RoundState;

struct Pool {
    int nseg;
    int pad;             // always 0 (an opaque zero for the kernels)
    int64_t nchunks;
    int64_t nchildren;
    int32_t ub;          // pruning bound of the round (the incumbent, or the frozen UB)
    int32_t frozen;      // resolve (1) or solve (0) semantics
    int32_t first_internal;  // first segment with internal children (nseg: none)
    int32_t host_dst;    // survivors go to pinned host buckets (place: contiguous 16-byte stores)
    // direct placement (single-wave pools): K2 CTA i owns chunk first + i, all CTAs are
    // co-resident, and after a grid-wide arrival count each writes its survivors straight
    // to their batch-ordered bucket rows -- no staging, no place kernel
    int32_t direct;
    int32_t ppc_lim;     // > 0: at most this many parents per chunk this round (spread_ppc)
    RoundState* summary; // direct: the mapped host RoundState K2's CTA 0 publishes into (or null)
    Segment seg[kMaxSegments];
};

struct K2Config {
    bool wide = false;   // generic kernel with int32 Mq over DevTables::jw
    int threads = 128;
    int cmax = 128;      // children per chunk (>= n)
    bool jm_in_smem = true;
    int variant = 0;     // 0: generic kernel; OCC*10000+N*100+M: k2_v2_kernel (expand_v2.cu);
                         // 100000+NW*100+M: k2_v3_kernel (expand_v3.cu)
    int ppc_cap = 0;     // > 0: at most this many parents per chunk
    int blocks = 0;
    size_t smem = 0;
    // persistent batch kernel (k2_v2_kernel<..., BATCH>): a whole device-planned batch of
    // single-wave rounds in one cooperative launch of `blocks` CTAs
    bool batch = false;
    size_t batch_smem = 0;
};
K2Config k2_config(const DevTables& t, int device);

// Per-chunk staging of survivors (compacted, batch order inside the chunk), moved
// to their final place by place_kernel.
struct ChunkOut {
    NodeStore nodes;  // capacity nchunks * cmax, chunk c at [c * cmax, c * cmax + count[c])
    int32_t* lb;      // survivor bounds (same indexing)
    int32_t* count;   // survivors per chunk
    int32_t* seg;     // segment of each chunk
};

// Per-round device state; the head (everything before `schedule`) is zeroed by
// one memset before the round.
struct RoundState {
    unsigned long long leaf_inv;  // ~((best leaf value << 32) | batch position); 0 = no leaf
    int32_t found;                // leaf schedule written (value < ub)
    uint32_t ticket;              // next chunk to claim
    int64_t total;                // survivors of the pool
    uint32_t place_done;          // place CTAs past their counting (the last one publishes)
    uint32_t arrived;             // direct placement: K2 CTAs past their counts (grid barrier)
    unsigned long long k2_t0_inv; // ~(first K2 CTA start), %globaltimer ns (0 = none)
    unsigned long long k2_t1;     // last K2 CTA end, %globaltimer ns
    int64_t seg_surv[kMaxSegments];
    int32_t schedule[kMaxJobs];
};
constexpr size_t kRoundStateHead = offsetof(RoundState, schedule);

// n <= 32, m in {5,10,20}: the register/shared-row kernel; false when not applicable.
bool k2_v2_config(const DevTables& t, int device, K2Config* out);
// place_hint: 0 staged placement, 1 direct (Pool::direct, known to the host), -1 read it
// from the pool (device-planned loop)
// The persistent batch kernel: plans, runs (leaves, K2 with direct placement) and closes
// rounds until the loop state stops it; every round must fit one wave (direct placement).
struct LoopState;
cudaError_t launch_k2_v2_batch(const DevTables& t, const K2Config& cfg, LoopState* ls, Pool* d_pool,
                               RoundState* rs, ChunkOut out, cudaStream_t stream);
cudaError_t launch_k2_v2(const DevTables& t, const K2Config& cfg, const Pool* d_pool, int first_seg,
                         int blocks, int place_hint, int frozen, RoundState* rs, ChunkOut out,
                         cudaStream_t stream, bool pdl = false);

// 64 < n <= 256, m in {5,10,20}: rows through L1, RMW scans; false when not applicable.
bool k2_v3_config(const DevTables& t, int device, K2Config* out);
cudaError_t launch_k2_v3(const DevTables& t, const K2Config& cfg, const Pool* d_pool, int first_seg,
                         int blocks, int32_t ub, int frozen, RoundState* rs, ChunkOut out,
                         cudaStream_t stream, bool pdl = false);

// Leaves (parents at depth >= n-2): batch minimum (value, first position).
cudaError_t launch_k2_leaves(const DevTables& t, const Pool* d_pool, const Pool& h_pool,
                             int seg_index, RoundState* rs, cudaStream_t stream, bool pdl = false);
// Internal children: bound, prune against min(ub, leaf minimum) (frozen: ub),
// survivors compacted per chunk into `out`.
cudaError_t launch_k2_internal(const DevTables& t, const K2Config& cfg, const Pool* d_pool,
                               const Pool& h_pool, int first_seg, int32_t ub, int frozen,
                               RoundState* rs, ChunkOut out, cudaStream_t stream, bool pdl = false);
// Uploads `words` 8-byte words from pinned host memory (UVA) to the device with one CTA:
// the round's zeroed state + pool, as a kernel so that K2 can be its programmatic dependent.
cudaError_t launch_pool_upload(const void* h_src, void* d_dst, int words, cudaStream_t stream);
// Every chunk's survivors moved, in batch order, to its segment's dst; per-segment
// and pool survivor totals added to `rs` (zeroed before the round).
cudaError_t launch_place(const DevTables& t, const K2Config& cfg, const Pool* d_pool,
                         const Pool& h_pool, RoundState* rs, ChunkOut out, cudaStream_t stream,
                         RoundState* summary = nullptr);
// Schedule of the best leaf when it beats ub (before the parents are recycled).


// ---- batched explorer loop (explorer_loop.cu): rounds planned and closed on the device --
constexpr int kLoopMax = 64;  // rounds per batch

struct LoopRecord {  // one round's counters (search.hpp:21-26, 75-79)
    int64_t target, branched, bounded, inserted, pruned, leaves, pending;
    int32_t incumbent, valid;
    // device clock (%globaltimer, ns): plan start, close end, first K2 CTA start, last K2
    // CTA end -- the per-round timing of a batch that has no events inside it
    unsigned long long t0, t1, k2_t0, k2_t1;
    unsigned long long tp, tb;  // persistent batch kernel: plan end, CTA 0 past the plan's grid barrier
};

// Device-resident explorer state for a batch of rounds.  The host writes the head
// (everything before `rec`; the batch's first step kernel clears the records) before a
// batch and reads the whole struct back after it.
struct LoopState {
    int64_t cnt[kMaxJobs + 1];        // pending bucket sizes
    int64_t cap[kMaxJobs + 1];        // their capacities (rows)
    NodeStore bucket[kMaxJobs + 1];   // their storage (HBM, or device-mapped host memory)
    int64_t targets[kLoopMax];        // pool target of each round of the batch
    int64_t tot_bounded, budget;      // cumulative bounded count; stop when >= budget (> 0)
    int32_t incumbent, best, found, frozen;
    int32_t stop;                     // 0 running, 1 pending empty, 2 budget, 3 bucket too small,
                                      // 4 corrupt node, 5 staging too small (never, by sizing),
                                      // 6 persistent kernel: the next round is not single-wave
    int32_t need_depth;               // stop == 3: the bucket that must grow ...
    int64_t need_rows;                // ... to at least this many rows
    int32_t cmax, ppc_cap, nrounds, chunk_cap;  // chunk_cap: staging chunks available
    int32_t direct_cap;               // > 0: pools of at most this many chunks use direct placement
    int32_t cur_round;                // conditional-graph batches: the round the next step closes / plans
    int32_t host_dst;                 // the buckets are pinned host memory (Pool::host_dst)
    int32_t spread_blocks;            // > 0: small pools spread over this many K2 CTAs (spread_ppc)
    uint32_t bar_count, bar_gen;      // grid barrier of the persistent batch kernel (zeroed by the host)
    int32_t schedule[kMaxJobs];       // incumbent schedule (solve mode)
    LoopRecord rec[kLoopMax];
};

// pdl: each kernel of the batch is a programmatic dependent of the one before (every one
// of them waits -- griddepcontrol.wait -- before it reads its predecessor's output)
// the step of a batch driven by a conditional WHILE graph node (round index in the loop
// state; sets the node's condition to "another round planned")
cudaError_t launch_loop_step_dyn(const DevTables& t, LoopState* ls, Pool* pool, RoundState* rs,
                                 cudaGraphConditionalHandle loop_cond, cudaGraphConditionalHandle leaf_cond,
                                 cudaStream_t stream, bool pdl);
// close of round - 1 (round > 0) + plan of round (!last), one single-warp kernel
cudaError_t launch_loop_step(const DevTables& t, LoopState* ls, Pool* pool, RoundState* rs, int round,
                             bool last, cudaStream_t stream, bool pdl);
// place_chunks: the staging's chunk capacity (the place grid covers it); 0: every pool of the
// batch is small enough for direct placement (K2 writes the survivors itself), so the place
// kernel is left out
cudaError_t launch_round_device(const DevTables& t, const K2Config& cfg, const Pool* d_pool,
                                RoundState* rs, ChunkOut out, cudaStream_t stream, bool pdl, int64_t place_chunks);
// Load the explorer's kernels at context creation (CUDA loads kernels lazily, at first use)
void preload_round_kernels();
void preload_loop_kernels();
// its two halves, for graphs that put the leaf kernels under a conditional node
cudaError_t launch_round_leaves(const DevTables& t, const Pool* d_pool, RoundState* rs, cudaStream_t stream,
                                bool pdl_first, bool pdl);
cudaError_t launch_round_k2_place(const DevTables& t, const K2Config& cfg, const Pool* d_pool, RoundState* rs,
                                  ChunkOut out, cudaStream_t stream, bool pdl_k2, bool pdl, int64_t place_chunks);

// Launches kern<<<grid, block, smem, st>>>(args...), as a programmatic dependent of the
// previous kernel in the stream when pdl (the kernel must griddepcontrol.wait before it
// reads that kernel's output).
template <class... KArgs, class... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              bool pdl, Args... args) {
    cudaLaunchConfig_t lc = {};
    lc.gridDim = grid;
    lc.blockDim = block;
    lc.dynamicSmemBytes = smem;
    lc.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    lc.attrs = at;
    lc.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&lc, kern, static_cast<KArgs>(args)...);
}

// More than one live context of this process on `device` (capi.cu): kernels of several
// contexts may then run on it concurrently.
bool device_shared(int device);

// Same, as a cooperative launch: the grid is gang-scheduled (all CTAs resident at once),
// which the direct-placement K2 needs for its grid-wide count -- without it, two such grids
// running concurrently (two contexts on one device) could each hold SMs while waiting for
// CTAs of their own that cannot be scheduled.
template <class... KArgs, class... Args>
inline cudaError_t launch_coop(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                               bool pdl, Args... args) {
    cudaLaunchConfig_t lc = {};
    lc.gridDim = grid;
    lc.blockDim = block;
    lc.dynamicSmemBytes = smem;
    lc.stream = st;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    lc.attrs = at;
    lc.numAttrs = pdl ? 2 : 1;
    return cudaLaunchKernelEx(&lc, kern, static_cast<KArgs>(args)...);
}

// Chunk geometry of a segment: parents per chunk.
__host__ __device__ inline int parents_per_chunk(int n, int depth, int cmax, int ppc_cap) {
    int r = n - depth;
    int ppc = r > 0 ? cmax / r : 1;
    return ppc_cap > 0 && ppc > ppc_cap ? ppc_cap : ppc;
}
// The tighter of the kernel's parents-per-chunk cap and a round's Pool::ppc_lim.
__host__ __device__ inline int round_ppc_cap(int ppc_cap, int ppc_lim) {
    return ppc_lim > 0 && (ppc_cap <= 0 || ppc_lim < ppc_cap) ? ppc_lim : ppc_cap;
}
// Small pools: when the internal parents of a round fill fewer chunks than the K2 grid has
// resident CTAs (`blocks`), the chunks get fewer parents each, so that they spread over
// the whole wave instead of leaving most SMs idle -- a single-wave round's time is one
// chunk's serial chain (staging, tables, scans, bounds, compaction), so it shrinks with
// the chunk.  Returns the smallest Pool::ppc_lim that keeps the round within `blocks`
// chunks (0: none -- the pool already fills the wave).
// ceil(a / b) for a >= 0, b > 0 -- in 32 bits when a fits: the device planner runs on one
// thread, where a 64-bit division is a long dependent subroutine
__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) {
    if (((uint64_t)a >> 31) == 0 && ((uint64_t)b >> 31) == 0)
        return (int64_t)(((uint32_t)a + (uint32_t)b - 1u) / (uint32_t)b);
    return (a + b - 1) / b;
}
__host__ __device__ inline int64_t spread_chunks(const Segment* seg, int nseg, int n, int cmax, int cap) {
    int64_t chunks = 0;
    for (int s = 0; s < nseg; ++s) {
        if (seg[s].depth >= n - 2) continue;  // leaves: no chunks
        const int ppc = parents_per_chunk(n, seg[s].depth, cmax, cap);
        chunks += ceil_div(seg[s].count, ppc);
    }
    return chunks;
}
__host__ __device__ inline int spread_ppc(const Segment* seg, int nseg, int n, int cmax, int ppc_cap,
                                          int blocks) {
    if (blocks <= 0) return 0;
    int64_t parents = 0;
    int nint = 0, ppc_max = 0;
    for (int s = 0; s < nseg; ++s) {
        if (seg[s].depth >= n - 2) continue;
        const int ppc = parents_per_chunk(n, seg[s].depth, cmax, ppc_cap);
        parents += seg[s].count;
        ppc_max = ppc > ppc_max ? ppc : ppc_max;
        ++nint;
    }
    if (nint == 0 || spread_chunks(seg, nseg, n, cmax, ppc_cap) >= blocks || blocks <= nint) return 0;
    // the smallest cap whose chunk count fits (the count falls as the cap grows): binary
    // search between a lower bound (every segment at the cap) and ppc_max (fits)
    int64_t lo = ceil_div(parents, blocks - nint), hi = ppc_max;
    if (lo < 1) lo = 1;
    if (lo < hi && spread_chunks(seg, nseg, n, cmax, (int)lo) <= blocks) hi = lo;  // usual case
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (spread_chunks(seg, nseg, n, cmax, (int)mid) > blocks) lo = mid + 1;
        else hi = mid;
    }
    return lo < ppc_max ? (int)lo : 0;
}

}  // namespace fbb
