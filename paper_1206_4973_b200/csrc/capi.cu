// capi.cu -- the C-ABI (include/flowbb_b200.h): contexts, K1/K2 host-buffer
// entry points and the device-resident explorer.
//
// The explorer keeps the reference's PendingTree (pending.hpp:13-56) in HBM:
// one stack per depth (SoA: masks, heads, prefixes).  A round is
//   selection  fill_buffer (search.hpp:64-73): pop the deepest bucket top,
//              LIFO, until the children count reaches the target -- computed
//              on the host from the bucket sizes alone (O(n)), no node moves;
//   K2         expand + bound + prune straight from the bucket tops;
//   push       survivors appended, in batch order, to bucket depth+1
//              (integrate, search.hpp:84-107 / bench.hpp:96-106).
// Only the per-segment survivor counts and the leaf minimum come back.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "fbb_internal.h"

using namespace fbb;

namespace {

// Device buffers come from the device's stream-ordered memory pool (release
// threshold raised at context creation), so growing a pending bucket between
// rounds is an async alloc + D2D copy + async free on the context stream, with
// no host synchronisation and no cudaMalloc latency.
// Pinned, device-mapped host memory for the host-resident pending tree.  Page
// locking is slow (milliseconds per tens of MB), so buckets are carved out of a
// few large pinned blocks by a first-fit free list instead of being allocated
// one by one; a bucket's growth is then an arena allocation + a copy.  Every
// user of the arena is ordered on the context stream, so a freed range can be
// reused at once.
class PinnedArena {
   public:
    ~PinnedArena() {
        for (Block& b : blocks_) cudaFreeHost(b.base);
    }
    cudaError_t alloc(size_t bytes, void** out) {
        bytes = (bytes + 255) & ~size_t(255);
        for (Block& b : blocks_)
            for (auto it = b.free.begin(); it != b.free.end(); ++it)
                if (it->second >= bytes) {
                    const size_t off = it->first, len = it->second;
                    b.free.erase(it);
                    if (len > bytes) b.free[off + bytes] = len - bytes;
                    *out = b.base + off;
                    return cudaSuccess;
                }
        size_t sz = std::max<size_t>(bytes, blocks_.empty() ? (size_t)256 << 20 : 2 * blocks_.back().size);
        Block nb;
        const char* wc = getenv("FBB_PINNED_WC");  // write-combined: no CPU caching / snooping
        const unsigned flags = cudaHostAllocMapped | cudaHostAllocPortable |
                               (wc && wc[0] == '1' ? cudaHostAllocWriteCombined : 0u);
        cudaError_t e = cudaHostAlloc((void**)&nb.base, sz, flags);
        if (e != cudaSuccess) return e;
        nb.size = sz;
        if (getenv("FBB_VERBOSE")) std::fprintf(stderr, "[fbb] pinned arena +%zu MiB\n", sz >> 20);
        if (sz > bytes) nb.free[bytes] = sz - bytes;
        blocks_.push_back(std::move(nb));
        *out = blocks_.back().base;
        return cudaSuccess;
    }
    void release(void* p, size_t bytes) {
        bytes = (bytes + 255) & ~size_t(255);
        for (Block& b : blocks_) {
            if ((char*)p < b.base || (char*)p >= b.base + b.size) continue;
            size_t off = (size_t)((char*)p - b.base);
            auto nx = b.free.lower_bound(off);
            if (nx != b.free.end() && off + bytes == nx->first) {  // merge with the next range
                bytes += nx->second;
                nx = b.free.erase(nx);
            }
            if (nx != b.free.begin()) {
                auto pv = std::prev(nx);
                if (pv->first + pv->second == off) {  // and with the previous one
                    pv->second += bytes;
                    return;
                }
            }
            b.free[off] = bytes;
            return;
        }
    }

   private:
    struct Block {
        char* base = nullptr;
        size_t size = 0;
        std::map<size_t, size_t> free;  // offset -> length
    };
    std::vector<Block> blocks_;
};

struct DBuf {
    void* p = nullptr;
    size_t bytes = 0;
    cudaStream_t st = nullptr;
    PinnedArena* arena = nullptr;  // set: pinned host memory (host-resident pending tree)
    cudaError_t ensure(size_t want) {
        if (want <= bytes) return cudaSuccess;
        size_t nb = std::max(want, bytes * 2);
        void* q = nullptr;
        cudaError_t e = arena ? arena->alloc(nb, &q) : cudaMallocAsync(&q, nb, st);
        if (e != cudaSuccess) return e;
        release();
        p = q;
        bytes = nb;
        return cudaSuccess;
    }
    void release() {
        if (p) {
            if (arena) arena->release(p, bytes);
            else cudaFreeAsync(p, st);
        }
        p = nullptr;
        bytes = 0;
    }
    template <class T>
    T* as() const { return static_cast<T*>(p); }
};

struct HBuf {  // pinned host
    void* p = nullptr;
    size_t bytes = 0;
    cudaError_t ensure(size_t want) {
        if (want <= bytes) return cudaSuccess;
        size_t nb = std::max(want, bytes * 2);
        void* q = nullptr;
        cudaError_t e = cudaMallocHost(&q, nb);
        if (e != cudaSuccess) return e;
        cudaFreeHost(p);
        p = q;
        bytes = nb;
        return cudaSuccess;
    }
    void release() {
        cudaFreeHost(p);
        p = nullptr;
        bytes = 0;
    }
    template <class T>
    T* as() const { return static_cast<T*>(p); }
};

// A growable node store (one pending bucket, or a scratch batch).  Compact stores
// (the host-resident pending tree) keep the prefixes only: heads and masks are folded
// from the prefix by the K2 kernels when they stage a parent, which cuts the bytes
// that cross the host link per pending node from W*8 + 4m + n to n (108 -> 20 at 20x20).
struct Store {
    DBuf masks, heads, prefix;
    int64_t cap = 0;
    bool compact = false;
    void set(cudaStream_t st, PinnedArena* arena) {
        for (DBuf* b : {&masks, &heads, &prefix}) {
            b->st = st;
            b->arena = arena;
        }
    }
    NodeStore view() const {
        return compact ? NodeStore{nullptr, nullptr, prefix.as<uint8_t>()}
                       : NodeStore{masks.as<uint64_t>(), heads.as<int32_t>(), prefix.as<uint8_t>()};
    }
};

}  // namespace

static std::mutex g_err_mu;
// live contexts per device (this process): K2's direct placement is gang-scheduled (a
// cooperative launch) only when another context may run kernels on the same device
static std::atomic<int> g_ctx_on_device[64];
static std::string g_create_err = "";
static int g_create_status = FBB_OK;

// What a captured batch graph bakes in: its length and the buffers its kernels and copies
// address (bucket storage travels in the uploaded LoopState, so bucket growth needs no
// recapture).
struct LoopGraphKey {
    int rounds = 0;
    const void* p[8] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
    LoopGraphKey() = default;
    LoopGraphKey(int r, const void* a, const void* b, const void* c, const void* d, const void* e,
                 const void* f, const void* g, const void* h)
        : rounds(r), p{a, b, c, d, e, f, g, h} {}
    bool operator==(const LoopGraphKey& o) const {
        if (rounds != o.rounds) return false;
        for (int i = 0; i < 8; ++i)
            if (p[i] != o.p[i]) return false;
        return true;
    }
};

struct fbb_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    HostTables ht;
    DevTables dt{};
    K1Config k1;
    K2Config k2;
    int status = FBB_OK;
    std::string msg;

    // scratch for the host-buffer entry points
    DBuf k1_masks, k1_heads, k1_depth, k1_lb;
    Store batch_in, batch_out;
    DBuf out_lb;
    // shared per-round device state
    Store staging;          // per-chunk compacted survivors (chunk c at c * cmax)
    Store parents;          // host-resident explorer: this round's parents, uploaded
    DBuf st_lb, st_count, st_seg;
    DBuf d_pool, d_round;   // Pool, RoundState (device-planned loop)
    HBuf h_pool, h_round;
    DBuf d_rp;              // host-planned rounds: [RoundState | Pool], uploaded by one copy
    HBuf h_rp;              // its pinned source; the RoundState part stays zero
    cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
    // batched device-planned explorer loop (explorer_loop.cu)
    DBuf d_loop;
    HBuf h_loop;
    // captured batches (explorer_run_batched), one per (length, buffers); lengths are
    // powers of two, so a context captures at most a handful
    std::vector<std::pair<LoopGraphKey, cudaGraphExec_t>> loop_graphs;
    cudaStream_t capture_stream = nullptr;   // captures the conditional loop body ...
    cudaStream_t capture_stream2 = nullptr;  // ... and the leaf branch inside it
    // batched device-planned rounds (explorer_loop.cu): -1 (default) for calls of two rounds
    // or more, FBB_DEVICE_LOOP=1 always, FBB_DEVICE_LOOP=0 never
    int device_loop = -1;
    float last_k2_ms = 0.f, last_round_ms = 0.f, last_sync_ms = 0.f, last_place_ms = 0.f;
    int last_launches = 0;

    // explorer
    std::vector<Store> bucket;
    std::vector<int64_t> cnt;
    int32_t incumbent = 0;  // pruning bound (frozen: the snapshot UB)
    int32_t best = 0;       // best leaf value found (== incumbent when not frozen)
    int frozen = 1;
    int found = 0;
    std::vector<int32_t> schedule;
    int64_t tot_branched = 0, tot_bounded = 0, tot_pruned = 0, tot_leaves = 0;
    bool explorer_ready = false;
    bool host_pending = false;  // pending tree in pinned host memory (fbb_explorer_set_residency)
    PinnedArena arena;          // its storage
    bool mapped_in = true;      // K2 reads the parents in place from the mapped host buckets
                                // over the host link; FBB_HOST_IN=copy: upload them first
    bool compact_rows = true;   // host-resident tree as prefixes only (FBB_HOST_ROWS=compact|full)
    bool mapped_out = true;     // place_kernel writes survivors straight into the (device-
                                // mapped) host buckets; FBB_HOST_OUT=staged: device output + D2H
    int64_t last_h2d = 0, last_d2h = 0;
    bool summary_by_place = true;  // FBB_SUMMARY=copy: download the round summary instead
    bool direct_place = true;      // FBB_DIRECT=0: always stage survivors + place_kernel
    bool check = false;  // FBB_CHECK=1: validate the pending tree after every round

    int fail(int code, const std::string& m) {
        status = code;
        msg = m;
        return code;
    }
    int cuda_fail(cudaError_t e, const char* where) {
        return fail(FBB_E_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
    }
};

#define CK(expr, where)                                 \
    do {                                                \
        cudaError_t e_ = (expr);                        \
        if (e_ != cudaSuccess) return ctx->cuda_fail(e_, where); \
    } while (0)

namespace {

size_t node_bytes(const fbb_ctx* ctx) {
    return (size_t)ctx->dt.W * 8 + (size_t)ctx->dt.m * 4 + (size_t)ctx->dt.n;
}
size_t row_bytes(const fbb_ctx* ctx, bool compact) { return compact ? (size_t)ctx->dt.n : node_bytes(ctx); }

cudaError_t store_ensure(fbb_ctx* ctx, Store& s, int64_t want, int64_t keep) {
    if (want <= s.cap) return cudaSuccess;
    // pinned host growth is slow (page locking): start host stores at ~4 MB
    const int64_t floor_rows =
        s.prefix.arena ? std::max<int64_t>(1024, (1 << 20) / (int64_t)row_bytes(ctx, s.compact)) : 1024;
    int64_t nc = std::max<int64_t>(want, std::max<int64_t>(s.cap * 2, floor_rows));
    const int n = ctx->dt.n, m = ctx->dt.m, W = ctx->dt.W;
    PinnedArena* host = s.prefix.arena;
    Store t;
    t.compact = s.compact;
    t.set(ctx->stream, host);
    s.set(ctx->stream, host);
    cudaError_t e;
    if (!t.compact) {
        if ((e = t.masks.ensure((size_t)nc * W * 8)) != cudaSuccess) return e;
        if ((e = t.heads.ensure((size_t)nc * m * 4)) != cudaSuccess) return e;
    }
    if ((e = t.prefix.ensure((size_t)nc * n)) != cudaSuccess) return e;
    if (keep > 0) {  // stream-ordered: the copy precedes the old buffers' release
        if (!t.compact) {
            cudaMemcpyAsync(t.masks.p, s.masks.p, (size_t)keep * W * 8, cudaMemcpyDefault, ctx->stream);
            cudaMemcpyAsync(t.heads.p, s.heads.p, (size_t)keep * m * 4, cudaMemcpyDefault, ctx->stream);
        }
        cudaMemcpyAsync(t.prefix.p, s.prefix.p, (size_t)keep * n, cudaMemcpyDefault, ctx->stream);
    }
    s.masks.release();
    s.heads.release();
    s.prefix.release();
    s = t;
    s.cap = nc;
    t.masks.p = t.heads.p = t.prefix.p = nullptr;  // ownership moved
    return cudaSuccess;
}

// Builds a pool over `segs` (depth-descending runs) and lays out chunks.
// Returns the index of the first internal segment.
int layout_pool(const fbb_ctx* ctx, Pool& pool) {
    const int n = ctx->dt.n, cmax = ctx->k2.cmax;
    pool.pad = 0;  // read by the kernels as an opaque zero
    int64_t child = 0, chunk = 0;
    int first_internal = pool.nseg;
    // small pools of the register-row kernel spread over the whole K2 wave
    const bool v2 = ctx->k2.variant != 0 && ctx->k2.variant < 100000;
    pool.ppc_lim = v2 ? spread_ppc(pool.seg, pool.nseg, n, cmax, ctx->k2.ppc_cap, ctx->k2.blocks) : 0;
    const int cap = round_ppc_cap(ctx->k2.ppc_cap, pool.ppc_lim);
    for (int s = 0; s < pool.nseg; ++s) {
        Segment& sg = pool.seg[s];
        int r = n - sg.depth;
        sg.child_base = child;
        child += sg.count * r;
        sg.chunk_base = chunk;
        if (sg.depth >= n - 2) continue;  // leaves: no chunks
        if (first_internal == pool.nseg) first_internal = s;
        int ppc = parents_per_chunk(n, sg.depth, cmax, cap);
        chunk += (sg.count + ppc - 1) / ppc;
    }
    pool.nchunks = chunk;
    pool.nchildren = child;
    return first_internal;
}

// Launches one pool: [leaves], internal K2 (bound + prune + ordered writes),
// [leaf schedule]; then downloads the RoundState.  Synchronises; the result is
// in ctx->h_round.
int run_pool(fbb_ctx* ctx, Pool& pool, int first_internal, int32_t ub, int frozen) {
    const int n = ctx->dt.n;
    cudaStream_t st = ctx->stream;
    const int64_t slots = std::max<int64_t>(pool.nchunks * ctx->k2.cmax, 1);
    CK(store_ensure(ctx, ctx->staging, slots, 0), "staging");
    CK(ctx->st_lb.ensure((size_t)slots * 4), "staging");
    CK(ctx->st_count.ensure((size_t)std::max<int64_t>(pool.nchunks, 1) * 4), "staging");
    CK(ctx->st_seg.ensure((size_t)std::max<int64_t>(pool.nchunks, 1) * 4), "staging");
    constexpr size_t kPoolOff = (sizeof(RoundState) + 255) & ~size_t(255);
    if (ctx->h_rp.bytes < kPoolOff + sizeof(Pool)) {
        CK(ctx->h_rp.ensure(kPoolOff + sizeof(Pool)), "pool");
        std::memset(ctx->h_rp.p, 0, kPoolOff);
    }
    CK(ctx->d_rp.ensure(kPoolOff + sizeof(Pool)), "pool");
    CK(ctx->h_round.ensure(sizeof(RoundState)), "round state");

    pool.ub = ub;  // the round's bound, semantics and first internal segment travel with the pool
    pool.frozen = frozen;
    pool.first_internal = first_internal;
    // direct placement (K2 writes the survivors to their bucket rows itself, no place
    // kernel): single-wave pools of the v2 kernel into device buckets
    pool.direct = 0;
    pool.summary = nullptr;
    if (ctx->direct_place && ctx->k2.variant != 0 && ctx->k2.variant < 100000 && !pool.host_dst &&
        first_internal < pool.nseg && pool.nchunks > 0 && pool.nchunks <= ctx->k2.blocks) {
        bool ok = true;
        for (int s = first_internal; s < pool.nseg; ++s)
            ok = ok && pool.seg[s].dst_base >= 0 && pool.seg[s].dst_lb == nullptr && pool.seg[s].dst.heads;
        pool.direct = ok ? 1 : 0;
    }
    if (pool.direct && ctx->summary_by_place) pool.summary = ctx->h_round.as<RoundState>();
    size_t pool_bytes = offsetof(Pool, seg) + (size_t)pool.nseg * sizeof(Segment);
    std::memcpy((char*)ctx->h_rp.p + kPoolOff, &pool, pool_bytes);
    int launches = 0;
    static const bool pdl = [] { const char* e = getenv("FBB_PDL"); return !(e && e[0] == '0'); }();
    bool has_leaf = pool.nseg > 0 && pool.seg[0].depth >= n - 2;
    // the upload is a one-CTA kernel and the round's kernels form a programmatic-
    // dependent-launch chain (upload -> [leaves -> leaf schedule] -> K2 -> place): each
    // one's prologue overlaps its predecessor; FBB_PDL=0: DMA copy and plain stream order
    const bool kernel_upload = pdl;
    CK(cudaEventRecord(ctx->ev[0], st), "event");
    // one upload carries the pool and zeroes the round state (counters, ticket, leaf key)
    if (kernel_upload)
        CK(launch_pool_upload(ctx->h_rp.p, ctx->d_rp.p, (int)((kPoolOff + pool_bytes + 7) / 8), st), "pool upload");
    else
        CK(cudaMemcpyAsync(ctx->d_rp.p, ctx->h_rp.p, kPoolOff + pool_bytes, cudaMemcpyHostToDevice, st), "pool H2D");
    const Pool* dp = (const Pool*)((char*)ctx->d_rp.p + kPoolOff);
    RoundState* rs = ctx->d_rp.as<RoundState>();
    if (has_leaf) {
        // leaves, then the best leaf's schedule -- before K2 recycles the leaf
        // parents' slots (bucket n-2 receives the next segment's survivors)
        CK(launch_k2_leaves(ctx->dt, dp, pool, 0, rs, st, kernel_upload), "K2 leaves");
        launches += 2;  // leaves + the best leaf's schedule
    }
    if (!pdl) CK(cudaEventRecord(ctx->ev[1], st), "event");
    bool has_internal = first_internal < pool.nseg && pool.nchunks > 0;
    ChunkOut out{ctx->staging.view(), ctx->st_lb.as<int32_t>(), ctx->st_count.as<int32_t>(),
                 ctx->st_seg.as<int32_t>()};
    CK(launch_k2_internal(ctx->dt, ctx->k2, dp, pool, first_internal, ub, frozen, rs, out, st, kernel_upload),
       "K2 internal");
    // place_kernel is a programmatic dependent of K2 (scheduled onto SMs as K2's CTAs
    // retire; FBB_PDL=0: plain stream order); no event may sit between the two, so K2's
    // time then comes from the device clock stamps K2 leaves in the round state
    if (!pdl) CK(cudaEventRecord(ctx->ev[2], st), "event");
    // with internal chunks, place_kernel's last CTA writes the round summary straight into
    // the pinned (UVA-mapped) h_round; otherwise one download of the counters (and, after
    // a leaf round, the schedule behind them)
    const bool publish = has_internal && ctx->summary_by_place;
    if (!pool.direct)
        CK(launch_place(ctx->dt, ctx->k2, dp, pool, rs, out, st, publish ? ctx->h_round.as<RoundState>() : nullptr),
           "place");
    launches += has_internal ? (pool.direct ? 1 : 2) : 0;  // K2 [+ place]
    if (!publish) {
        const size_t head = has_leaf ? offsetof(RoundState, schedule) + (size_t)n * 4
                                     : offsetof(RoundState, seg_surv) + (size_t)pool.nseg * 8;
        CK(cudaMemcpyAsync(ctx->h_round.p, rs, head, cudaMemcpyDeviceToHost, st), "round D2H");
    }
    CK(cudaEventRecord(ctx->ev[3], st), "event");
    const auto t_sync = std::chrono::steady_clock::now();
    CK(cudaStreamSynchronize(st), "round");
    ctx->last_sync_ms = std::chrono::duration<float, std::milli>(std::chrono::steady_clock::now() - t_sync).count();
    if (ctx->h_round.as<RoundState>()->found < 0)
        return ctx->fail(FBB_E_STATE, "corrupt pending node (unscheduled-job count mismatch)");
    if (pdl) {
        const RoundState* hr = ctx->h_round.as<RoundState>();
        ctx->last_k2_ms = hr->k2_t1 && hr->k2_t0_inv ? (float)((double)(hr->k2_t1 - ~hr->k2_t0_inv) * 1e-6) : 0.f;
    } else {
        cudaEventElapsedTime(&ctx->last_k2_ms, ctx->ev[1], ctx->ev[2]);
    }
    cudaEventElapsedTime(&ctx->last_round_ms, ctx->ev[0], ctx->ev[3]);
    if (pdl) ctx->last_place_ms = -1.f;
    else cudaEventElapsedTime(&ctx->last_place_ms, ctx->ev[2], ctx->ev[3]);  // place + summary download
    ctx->last_launches = launches;
    return FBB_OK;
}

// Best leaf of the round (value, position), when any.
bool round_leaf(const RoundState* r, int32_t* value, int64_t* pos) {
    if (r->leaf_inv == 0ull) return false;
    unsigned long long key = ~r->leaf_inv;
    *value = (int32_t)(key >> 32);
    *pos = (int64_t)(key & 0xFFFFFFFFull);
    return true;
}

void node_from_prefix(const HostTables& h, const uint8_t* prefix, int depth, uint64_t* mask,
                      int32_t* heads) {
    for (int w = 0; w < h.W; ++w) mask[w] = 0;
    for (int k = 0; k < h.m; ++k) heads[k] = 0;
    for (int i = 0; i < depth; ++i) {
        int j = prefix[i];
        mask[j >> 6] |= 1ull << (j & 63);
        int32_t prev = 0;
        for (int k = 0; k < h.m; ++k) {  // instance.hpp:81-89
            prev = std::max(prev, heads[k]) + h.p[(size_t)j * h.m + k];
            heads[k] = prev;
        }
    }
}

int64_t pending_total(const fbb_ctx* ctx) {
    int64_t s = 0;
    for (int64_t c : ctx->cnt) s += c;
    return s;
}

// Pushes host nodes (in order) onto the device buckets.
int push_host_nodes(fbb_ctx* ctx, const uint8_t* prefix, const int32_t* depth, int64_t count) {
    const int n = ctx->dt.n, m = ctx->dt.m, W = ctx->dt.W;
    // group by depth preserving order
    std::vector<std::vector<int64_t>> by(n + 1);
    for (int64_t i = 0; i < count; ++i) {
        if (depth[i] < 0 || depth[i] > n) return ctx->fail(FBB_E_ARG, "node depth out of range");
        if (depth[i] == n) return ctx->fail(FBB_E_ARG, "complete nodes cannot be pending");
        by[depth[i]].push_back(i);
    }
    std::vector<uint64_t> hm;
    std::vector<int32_t> hh;
    std::vector<uint8_t> hp;
    for (int d = 0; d <= n; ++d) {
        if (by[d].empty()) continue;
        int64_t k = (int64_t)by[d].size();
        hm.assign((size_t)k * W, 0);
        hh.assign((size_t)k * m, 0);
        hp.assign((size_t)k * n, 0);
        for (int64_t t = 0; t < k; ++t) {
            const uint8_t* pr = prefix + by[d][t] * n;
            std::vector<uint8_t> seen(n, 0);
            for (int i = 0; i < d; ++i) {
                if (pr[i] >= n || seen[pr[i]]) return ctx->fail(FBB_E_ARG, "invalid prefix");
                seen[pr[i]] = 1;
            }
            node_from_prefix(ctx->ht, pr, d, &hm[t * W], &hh[t * m]);
            std::memcpy(&hp[t * n], pr, (size_t)d);
        }
        int64_t c0 = ctx->cnt[d];
        CK(store_ensure(ctx, ctx->bucket[d], c0 + k, c0), "bucket grow");
        Store& b = ctx->bucket[d];
        cudaStream_t st = ctx->stream;
        if (!b.compact) {
            CK(cudaMemcpyAsync(b.masks.as<uint64_t>() + c0 * W, hm.data(), hm.size() * 8, cudaMemcpyDefault, st), "push");
            CK(cudaMemcpyAsync(b.heads.as<int32_t>() + c0 * m, hh.data(), hh.size() * 4, cudaMemcpyDefault, st), "push");
        }
        CK(cudaMemcpyAsync(b.prefix.as<uint8_t>() + c0 * n, hp.data(), hp.size(), cudaMemcpyDefault, st), "push");
        CK(cudaStreamSynchronize(st), "push");  // host vectors are reused
        ctx->cnt[d] = c0 + k;
    }
    return FBB_OK;
}

// FBB_CHECK=1: after every round, every pending node must have popcount(mask)
// == depth == the number of prefix entries, and heads must fold from the prefix.
int check_pending(fbb_ctx* ctx) {
    const int n = ctx->dt.n, m = ctx->dt.m, W = ctx->dt.W;
    for (int d = 0; d <= n; ++d) {
        int64_t k = ctx->cnt[d];
        if (k == 0) continue;
        if (k > ctx->bucket[d].cap) return ctx->fail(FBB_E_STATE, "check: count exceeds capacity");
        std::vector<uint64_t> mk((size_t)k * W);
        std::vector<int32_t> hd((size_t)k * m);
        std::vector<uint8_t> pr((size_t)k * n);
        cudaStream_t st = ctx->stream;
        const bool compact = ctx->bucket[d].compact;
        if (!compact) {
            CK(cudaMemcpyAsync(mk.data(), ctx->bucket[d].masks.p, mk.size() * 8, cudaMemcpyDefault, st), "check");
            CK(cudaMemcpyAsync(hd.data(), ctx->bucket[d].heads.p, hd.size() * 4, cudaMemcpyDefault, st), "check");
        }
        CK(cudaMemcpyAsync(pr.data(), ctx->bucket[d].prefix.p, pr.size(), cudaMemcpyDefault, st), "check");
        CK(cudaStreamSynchronize(st), "check");
        std::vector<uint64_t> m2(W);
        std::vector<int32_t> h2(m);
        for (int64_t i = 0; i < k; ++i) {
            node_from_prefix(ctx->ht, &pr[i * n], d, m2.data(), h2.data());
            int jobs = 0;  // compact rows: the prefix must name d distinct jobs
            for (int w = 0; w < W; ++w) jobs += __builtin_popcountll(m2[w]);
            bool ok = compact ? jobs == d
                              : std::memcmp(m2.data(), &mk[i * W], W * 8) == 0 &&
                                    std::memcmp(h2.data(), &hd[i * m], m * 4) == 0;
            if (!ok) {
                char buf[160];
                std::snprintf(buf, sizeof buf, "check: bad pending node depth %d index %lld of %lld",
                              d, (long long)i, (long long)k);
                return ctx->fail(FBB_E_STATE, buf);
            }
        }
    }
    return FBB_OK;
}

void explorer_clear(fbb_ctx* ctx) {
    const int n = ctx->dt.n;
    if ((int)ctx->bucket.size() != n + 1) ctx->bucket.resize(n + 1);
    PinnedArena* want = ctx->host_pending ? &ctx->arena : nullptr;
    const bool compact = ctx->host_pending && ctx->compact_rows;
    for (Store& b : ctx->bucket) {
        if (b.prefix.arena != want || b.compact != compact) {  // residency changed: drop the old storage
            cudaStreamSynchronize(ctx->stream);
            b.masks.release();
            b.heads.release();
            b.prefix.release();
            b.cap = 0;
        }
        b.compact = compact;
        b.set(ctx->stream, want);
    }
    if (ctx->parents.compact != compact) {  // the upload scratch follows the tree's row format
        cudaStreamSynchronize(ctx->stream);
        ctx->parents.masks.release();
        ctx->parents.heads.release();
        ctx->parents.prefix.release();
        ctx->parents.cap = 0;
        ctx->parents.compact = compact;
    }
    ctx->cnt.assign(n + 1, 0);
    ctx->schedule.assign(n, 0);
    ctx->found = 0;
    ctx->tot_branched = ctx->tot_bounded = ctx->tot_pruned = ctx->tot_leaves = 0;
    ctx->explorer_ready = true;
}

// One explorer round with pool target `target` (> 0).
int explorer_round(fbb_ctx* ctx, int64_t target, fbb_round_t* rec) {
    const auto t0 = std::chrono::steady_clock::now();
    const int n = ctx->dt.n;
    std::memset(rec, 0, sizeof(*rec));
    rec->target = target;
    static thread_local Pool local;
    local.nseg = 0;
    std::vector<int64_t> after = ctx->cnt;
    int64_t have = 0;
    for (int d = n; d >= 0 && have < target; --d) {  // fill_buffer, search.hpp:69-72
        if (after[d] == 0) continue;
        int r = n - d;
        int64_t need = (target - have + r - 1) / r;
        int64_t k = std::min<int64_t>(after[d], need);
        Segment& sg = local.seg[local.nseg++];
        std::memset(&sg, 0, sizeof(sg));
        sg.src = ctx->bucket[d].view();
        sg.first = after[d] - 1;
        sg.step = -1;
        sg.count = k;
        sg.depth = d;
        after[d] -= k;
        have += k * r;
    }
    if (local.nseg == 0) return FBB_OK;
    int first_internal = layout_pool(ctx, local);
    local.host_dst = ctx->host_pending && ctx->mapped_out;  // survivors written over the host link
    // destinations (bucket depth+1) sized for the worst case before launching
    // device buckets: sized for the worst case (all children survive) before K2 writes
    // into them; host buckets grow after the round, to the actual survivor count
    const bool staged_out = ctx->host_pending && !ctx->mapped_out;  // device output, then D2H
    for (int s = first_internal; s < local.nseg && !staged_out; ++s) {
        Segment& sg = local.seg[s];
        int d1 = sg.depth + 1;
        int64_t worst = after[d1] + sg.count * (n - sg.depth);
        // keep the full old content: this round's parents may sit in bucket d1's popped region
        CK(store_ensure(ctx, ctx->bucket[d1], worst, ctx->cnt[d1]), "bucket grow");
    }
    int64_t h2d = 0, npar = 0;
    const bool upload = ctx->host_pending && !ctx->mapped_in;
    if (ctx->host_pending && ctx->mapped_in) {  // parents read in place over the host link
        for (int s = 0; s < local.nseg; ++s) npar += local.seg[s].count;
        h2d = npar * (int64_t)row_bytes(ctx, ctx->compact_rows);
    }
    if (upload) {
        // host-resident pending tree: this round's parents (the top rows of each
        // selected bucket, contiguous) go host -> device; survivors are written by
        // place_kernel straight into the (device-mapped, pinned) host buckets
        for (int s = 0; s < local.nseg; ++s) npar += local.seg[s].count;
        CK(store_ensure(ctx, ctx->parents, npar, 0), "parents");
        const int m = ctx->dt.m, W = ctx->dt.W;
        const NodeStore pv = ctx->parents.view();
        int64_t o = 0;
        for (int s = 0; s < local.nseg; ++s) {
            Segment& sg = local.seg[s];
            const NodeStore b = ctx->bucket[sg.depth].view();
            const int64_t lo = after[sg.depth], k = sg.count;
            if (b.heads) {
                CK(cudaMemcpyAsync(pv.masks + o * W, b.masks + lo * W, (size_t)k * W * 8, cudaMemcpyDefault, ctx->stream), "parents H2D");
                CK(cudaMemcpyAsync(pv.heads + o * m, b.heads + lo * m, (size_t)k * m * 4, cudaMemcpyDefault, ctx->stream), "parents H2D");
            }
            CK(cudaMemcpyAsync(pv.prefix + o * n, b.prefix + lo * n, (size_t)k * n, cudaMemcpyDefault, ctx->stream), "parents H2D");
            sg.first = o + k - 1;  // LIFO: the bucket top is popped first
            o += k;
        }
        h2d = npar * (int64_t)row_bytes(ctx, ctx->compact_rows);
    }
    if (staged_out) CK(store_ensure(ctx, ctx->batch_out, std::max<int64_t>(local.nchildren, 1), 0), "alloc");
    for (int s = 0; s < local.nseg; ++s) {  // views may have moved after growth
        Segment& sg = local.seg[s];
        sg.src = upload ? ctx->parents.view() : ctx->bucket[sg.depth].view();
        if (sg.depth < n - 2 && staged_out) {  // contiguous device output, then D2H
            sg.dst = ctx->batch_out.view();
            sg.dst_base = -1;
        } else if (sg.depth < n - 2) {
            sg.dst = ctx->bucket[sg.depth + 1].view();
            sg.dst_base = after[sg.depth + 1];
        } else {
            sg.dst = NodeStore{nullptr, nullptr, nullptr};
            sg.dst_base = 0;
        }
        sg.dst_lb = nullptr;
    }
    int rc = run_pool(ctx, local, first_internal, ctx->incumbent, ctx->frozen);
    if (rc != FBB_OK) return rc;
    const RoundState* sm = ctx->h_round.as<RoundState>();
    int64_t internal = 0, leaves = 0, out_row = 0;
    for (int s = 0; s < local.nseg; ++s) {
        const Segment& sg = local.seg[s];
        int64_t kids = sg.count * (n - sg.depth);
        rec->branched += sg.count;
        if (sg.depth >= n - 2) {
            leaves += kids;
        } else {
            internal += kids;
            const int64_t k = sm->seg_surv[s];
            if (staged_out && k > 0) {  // survivors -> the host bucket, in batch order
                const int m = ctx->dt.m, W = ctx->dt.W;
                const int64_t at = after[sg.depth + 1];
                CK(store_ensure(ctx, ctx->bucket[sg.depth + 1], at + k, at), "bucket grow");
                const NodeStore b = ctx->bucket[sg.depth + 1].view(), o = ctx->batch_out.view();
                if (b.heads) {
                    CK(cudaMemcpyAsync(b.masks + at * W, o.masks + out_row * W, (size_t)k * W * 8, cudaMemcpyDefault, ctx->stream), "survivors D2H");
                    CK(cudaMemcpyAsync(b.heads + at * m, o.heads + out_row * m, (size_t)k * m * 4, cudaMemcpyDefault, ctx->stream), "survivors D2H");
                }
                CK(cudaMemcpyAsync(b.prefix + at * n, o.prefix + out_row * n, (size_t)k * n, cudaMemcpyDefault, ctx->stream), "survivors D2H");
            }
            out_row += k;
            after[sg.depth + 1] += k;
        }
    }
    if (staged_out && out_row > 0) CK(cudaStreamSynchronize(ctx->stream), "survivors D2H");
    ctx->cnt = after;
    rec->bounded = internal + leaves;
    rec->leaves = leaves;
    rec->inserted = sm->total;
    rec->pruned = internal - sm->total;
    int32_t v;
    int64_t vpos;
    if (leaves > 0 && round_leaf(sm, &v, &vpos)) {
        if (ctx->frozen) {
            // frozen incumbent: track the best leaf strictly under UB (bench.hpp:99-102)
            if (v < ctx->incumbent && (!ctx->found || v < ctx->best)) {
                ctx->best = v;
                ctx->found = 1;
            }
        } else if (v < ctx->incumbent) {
            // integrate: strict improvement, first leaf attaining the minimum (search.hpp:93-99)
            ctx->incumbent = v;
            ctx->best = v;
            ctx->found = 1;
            if (sm->found) std::memcpy(ctx->schedule.data(), sm->schedule, (size_t)n * 4);
        }
    }
    rec->incumbent = ctx->frozen ? (ctx->found ? ctx->best : ctx->incumbent) : ctx->incumbent;
    rec->k2_ms = ctx->last_k2_ms;
    rec->round_ms = ctx->last_round_ms;
    rec->place_ms = ctx->last_place_ms;
    rec->launches = ctx->last_launches;
    if (ctx->check) {
        int rc2 = check_pending(ctx);
        if (rc2 != FBB_OK) return rc2;
    }
    ctx->tot_branched += rec->branched;
    ctx->tot_bounded += rec->bounded;
    ctx->tot_pruned += rec->pruned;
    ctx->tot_leaves += rec->leaves;
    rec->pending = pending_total(ctx);
    rec->sync_ms = ctx->last_sync_ms;
    rec->h2d_bytes = h2d;
    rec->d2h_bytes = ctx->host_pending ? rec->inserted * (int64_t)row_bytes(ctx, ctx->compact_rows) : 0;
    rec->host_ms = std::chrono::duration<float, std::milli>(std::chrono::steady_clock::now() - t0).count();
    return FBB_OK;
}

// Rounds planned and closed on the device (explorer_loop.cu), up to kLoopMax per batch
// with no host synchronisation inside a batch; same semantics and per-round records as
// explorer_round.  Used when the parents can be read in place (HBM buckets, or host
// buckets read and written through the mapping).
bool device_loop_ok(const fbb_ctx* ctx, int64_t max_rounds) {
    // auto: multi-round calls, on an HBM tree or a host tree of prefix-only rows.  (A host
    // tree was host-planned until the loop kernels were preloaded at context creation:
    // lazy loading put a graph capture into the first timed batch, and e2e swung 0.5-1.6
    // G/s; with it, Ta021 262 K e2e runs 1.68 G/s batched vs 1.58 G/s host-planned -- no
    // host round trip per round.  Full-row host trees (n > 32) stay host-planned: their
    // many deep buckets grow often, each growth ends a batch, and Ta101 e2e measured 0.84
    // G/s batched vs 0.92 host-planned.)
    const bool want = ctx->device_loop == 1 ||
                      (ctx->device_loop == -1 && max_rounds >= 2 && (!ctx->host_pending || ctx->compact_rows));
    return want && (!ctx->host_pending || (ctx->mapped_in && ctx->mapped_out));
}

int explorer_run_batched(fbb_ctx* ctx, const int64_t* targets, int ntargets, int64_t max_rounds,
                         int64_t budget, fbb_round_t* rounds, int64_t* done) {
    const int n = ctx->dt.n;
    cudaStream_t st = ctx->stream;
    int64_t r = 0;
    if (done) *done = 0;
    CK(ctx->d_loop.ensure(sizeof(LoopState)), "loop state");
    CK(ctx->h_loop.ensure(sizeof(LoopState)), "loop state");
    // (two of each: the persistent kernel alternates between them)
    CK(ctx->d_pool.ensure(2 * sizeof(Pool)), "pool");
    CK(ctx->d_round.ensure(2 * sizeof(RoundState)), "round state");
    LoopState* hl = ctx->h_loop.as<LoopState>();
    static const bool dbg = [] { const char* e = getenv("FBB_LOOP_DEBUG"); return e && e[0] == '1'; }();
    while (r < max_rounds) {
        const auto b0 = std::chrono::steady_clock::now();
        if (pending_total(ctx) == 0) break;
        if (budget > 0 && ctx->tot_bounded >= budget) break;
        const int R = (int)std::min<int64_t>(kLoopMax, max_rounds - r);
        int64_t tmax = 1;
        for (int i = 0; i < R; ++i) {
            const int64_t ri = r + i;
            tmax = std::max<int64_t>(tmax, targets[ri < ntargets ? ri : ntargets - 1]);
        }
        // staging for the largest pool of the batch, worst case: every internal segment
        // (r >= 3) at its fewest children per chunk, min(cmax / r, ppc_cap) * r, plus one
        // partial chunk per segment; fill_buffer overshoots the target by < n children
        const int cmax = ctx->k2.cmax;
        int64_t cpc_min = cmax;
        for (int r = 3; r <= n; ++r) {
            const int ppc = parents_per_chunk(n, n - r, cmax, ctx->k2.ppc_cap);
            cpc_min = std::min<int64_t>(cpc_min, (int64_t)std::max(ppc, 1) * r);
        }
        int64_t chunks = (tmax + n + cpc_min - 1) / std::max<int64_t>(cpc_min, 1) + n + 2;
        // small pools may be spread over up to k2.blocks chunks (spread_ppc)
        if (ctx->k2.variant != 0 && ctx->k2.variant < 100000) chunks = std::max<int64_t>(chunks, ctx->k2.blocks);
        CK(store_ensure(ctx, ctx->staging, chunks * cmax, 0), "staging");
        CK(ctx->st_lb.ensure((size_t)chunks * cmax * 4), "staging");
        CK(ctx->st_count.ensure((size_t)chunks * 4), "staging");
        CK(ctx->st_seg.ensure((size_t)chunks * 4), "staging");
        std::memset(hl, 0, offsetof(LoopState, rec));  // (the first step clears the records)
        for (int d = 0; d <= n; ++d) {
            hl->cnt[d] = ctx->cnt[d];
            hl->cap[d] = ctx->bucket[d].cap;
            hl->bucket[d] = ctx->bucket[d].view();
        }
        for (int i = 0; i < R; ++i) {
            const int64_t ri = r + i;
            hl->targets[i] = targets[ri < ntargets ? ri : ntargets - 1];
        }
        hl->tot_bounded = ctx->tot_bounded;
        hl->budget = budget;
        hl->incumbent = ctx->incumbent;
        hl->best = ctx->best;
        hl->found = ctx->found;
        hl->frozen = ctx->frozen;
        hl->cmax = cmax;
        hl->ppc_cap = ctx->k2.ppc_cap;
        hl->nrounds = R;
        hl->chunk_cap = (int32_t)std::min<int64_t>(chunks, INT32_MAX);
        hl->direct_cap = (ctx->direct_place && ctx->k2.variant != 0 && ctx->k2.variant < 100000 &&
                          !ctx->host_pending) ? ctx->k2.blocks : 0;
        hl->host_dst = ctx->host_pending ? 1 : 0;  // survivors written over the host link
        hl->spread_blocks = (ctx->k2.variant != 0 && ctx->k2.variant < 100000) ? ctx->k2.blocks : 0;
        // every pool of the batch fits one wave (worst-case chunk count): K2 places them all
        const bool all_direct = hl->direct_cap > 0 && chunks <= hl->direct_cap;
        // the place grid covers the staging's whole chunk capacity: tied to the staging
        // buffers, which are part of a cached graph's key (a batch of smaller pools reusing
        // a graph captured for larger ones launches CTAs that exit at once)
        const int64_t place_chunks = ctx->staging.cap / cmax;
        for (int i = 0; i < n; ++i) hl->schedule[i] = ctx->schedule[i];
        LoopState* dl = ctx->d_loop.as<LoopState>();
        Pool* dp = ctx->d_pool.as<Pool>();
        RoundState* rs = ctx->d_round.as<RoundState>();
        ChunkOut out{ctx->staging.view(), ctx->st_lb.as<int32_t>(), ctx->st_count.as<int32_t>(),
                     ctx->st_seg.as<int32_t>()};
        const auto w0 = std::chrono::steady_clock::now();
        // the batch: state upload, R x (step, leaves, leaf schedule, K2, place), step, state
        // download -- every kernel a programmatic dependent of the one before, the whole
        // sequence one CUDA graph (captured once per batch length and staging buffers, then
        // replayed: one host call per batch)
        auto enqueue = [&](bool pdl, int rounds) -> cudaError_t {
            cudaError_t e = cudaMemcpyAsync(dl, hl, offsetof(LoopState, rec), cudaMemcpyHostToDevice, st);
            for (int i = 0; i < rounds && e == cudaSuccess; ++i) {
                if ((e = launch_loop_step(ctx->dt, dl, dp, rs, i, false, st, pdl && i > 0)) != cudaSuccess) break;
                e = launch_round_device(ctx->dt, ctx->k2, dp, rs, out, st, pdl, all_direct ? 0 : place_chunks);
            }
            if (e == cudaSuccess) e = launch_loop_step(ctx->dt, dl, dp, rs, rounds, true, st, pdl);
            if (e == cudaSuccess) e = cudaMemcpyAsync(hl, dl, sizeof(LoopState), cudaMemcpyDeviceToHost, st);
            return e;
        };
        static const bool use_graph = [] { const char* e = getenv("FBB_LOOP_GRAPH"); return !(e && e[0] == '0'); }();
        static const bool loop_pdl = [] { const char* e = getenv("FBB_PDL"); return !(e && e[0] == '0'); }();
        static const bool persist = [] { const char* e = getenv("FBB_PERSIST"); return !(e && e[0] == '0'); }();
        // the persistent kernel when the batch's pools are mostly single-wave (a round that
        // is not comes back as stop 6 and runs host-planned)
        const bool pbk = persist && ctx->k2.batch && hl->direct_cap > 0 &&
                         (tmax + n) * 4 <= (int64_t)hl->direct_cap * cmax * 3;
        if (pbk) {
            // every round of the batch fits one wave: ONE cooperative launch of the
            // persistent K2 plans, runs and closes them all (expand_v2.cu, BATCH)
            CK(cudaMemcpyAsync(dl, hl, offsetof(LoopState, rec), cudaMemcpyHostToDevice, st), "loop state");
            CK(launch_k2_v2_batch(ctx->dt, ctx->k2, dl, dp, rs, out, st), "persistent batch");
            CK(cudaMemcpyAsync(hl, dl, sizeof(LoopState), cudaMemcpyDeviceToHost, st), "loop state");
        } else if (use_graph) {
            // one graph for every batch length: state upload, a step planning round 0, then a
            // conditional WHILE node whose body -- leaves, leaf schedule, K2, [place], step --
            // repeats while the step planned another round (the round index lives in the loop
            // state), then the state download
            const LoopGraphKey key{(all_direct ? 2 : 0) + (device_shared(ctx->device) ? 1 : 0),
                                   out.nodes.masks, out.nodes.heads,
                                   out.nodes.prefix, out.lb, out.count, out.seg, dl, hl};
            cudaGraphExec_t exec = nullptr;
            for (auto& kv : ctx->loop_graphs)
                if (kv.first == key) exec = kv.second;
            if (!exec) {
                if (ctx->loop_graphs.size() >= 16) {  // buffers moved many times: start over
                    for (auto& kv : ctx->loop_graphs) cudaGraphExecDestroy(kv.second);
                    ctx->loop_graphs.clear();
                }
                for (cudaStream_t* cs_ : {&ctx->capture_stream, &ctx->capture_stream2})
                    if (!*cs_) CK(cudaStreamCreateWithFlags(cs_, cudaStreamNonBlocking), "stream");
                // outer graph: state upload -> WHILE(loop_cond, starts at 1 every launch) ->
                // state download.  Loop body: step (close the last round, plan the next, set
                // both conditions) -> IF(leaf_cond) {leaf kernel -> leaf schedule} -> K2 ->
                // [place].  Inside a body graph the kernels keep their programmatic edges
                // except across the IF node (K2 waits for it in full).
                cudaGraph_t g = nullptr;
                cudaGraphConditionalHandle loop_cond, leaf_cond;
                cudaStreamCaptureStatus cs;
                const cudaGraphNode_t* deps = nullptr;
                size_t ndeps = 0;
                cudaGraphNode_t wnode, inode;
                cudaGraphNodeParams wp = {}, ip = {};
                CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal), "loop capture");
                cudaError_t ce = cudaMemcpyAsync(dl, hl, offsetof(LoopState, rec), cudaMemcpyHostToDevice, st);
                if (ce == cudaSuccess) ce = cudaStreamGetCaptureInfo(st, &cs, nullptr, &g, &deps, &ndeps);
                if (ce == cudaSuccess) ce = cudaGraphConditionalHandleCreate(&loop_cond, g, 1, cudaGraphCondAssignDefault);
                wp.type = cudaGraphNodeTypeConditional;
                wp.conditional.handle = loop_cond;
                wp.conditional.type = cudaGraphCondTypeWhile;
                wp.conditional.size = 1;
                if (ce == cudaSuccess) ce = cudaGraphAddNode(&wnode, g, deps, ndeps, &wp);
                if (ce == cudaSuccess) {
                    cudaGraph_t body = wp.conditional.phGraph_out[0];
                    cudaStream_t bs = ctx->capture_stream, ls2 = ctx->capture_stream2;
                    ce = cudaGraphConditionalHandleCreate(&leaf_cond, body, 0, 0);
                    if (ce == cudaSuccess)
                        ce = cudaStreamBeginCaptureToGraph(bs, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed);
                    if (ce == cudaSuccess)
                        ce = launch_loop_step_dyn(ctx->dt, dl, dp, rs, loop_cond, leaf_cond, bs, false);
                    cudaGraph_t bg = nullptr;
                    if (ce == cudaSuccess) ce = cudaStreamGetCaptureInfo(bs, &cs, nullptr, &bg, &deps, &ndeps);
                    ip.type = cudaGraphNodeTypeConditional;
                    ip.conditional.handle = leaf_cond;
                    ip.conditional.type = cudaGraphCondTypeIf;
                    ip.conditional.size = 1;
                    if (ce == cudaSuccess) ce = cudaGraphAddNode(&inode, bg, deps, ndeps, &ip);
                    if (ce == cudaSuccess) {
                        ce = cudaStreamBeginCaptureToGraph(ls2, ip.conditional.phGraph_out[0], nullptr, nullptr, 0,
                                                           cudaStreamCaptureModeRelaxed);
                        if (ce == cudaSuccess) ce = launch_round_leaves(ctx->dt, dp, rs, ls2, false, loop_pdl);
                        cudaError_t le = cudaStreamEndCapture(ls2, nullptr);
                        if (ce == cudaSuccess) ce = le;
                    }
                    if (ce == cudaSuccess) ce = cudaStreamUpdateCaptureDependencies(bs, &inode, 1, cudaStreamSetCaptureDependencies);
                    if (ce == cudaSuccess)
                        ce = launch_round_k2_place(ctx->dt, ctx->k2, dp, rs, out, bs, false, loop_pdl,
                                                   all_direct ? 0 : place_chunks);
                    cudaError_t be = cudaStreamEndCapture(bs, nullptr);
                    if (ce == cudaSuccess) ce = be;
                }
                if (ce == cudaSuccess) ce = cudaStreamUpdateCaptureDependencies(st, &wnode, 1, cudaStreamSetCaptureDependencies);
                if (ce == cudaSuccess) ce = cudaMemcpyAsync(hl, dl, sizeof(LoopState), cudaMemcpyDeviceToHost, st);
                cudaGraph_t gg = nullptr;
                cudaError_t ee = cudaStreamEndCapture(st, &gg);
                CK(ce, "loop capture");
                CK(ee, "loop capture");
                ce = cudaGraphInstantiate(&exec, gg, 0);
                cudaGraphDestroy(gg);
                CK(ce, "loop graph instantiate");
                ctx->loop_graphs.emplace_back(key, exec);
            }
            CK(cudaGraphLaunch(exec, st), "loop graph");
        } else {
            CK(enqueue(loop_pdl, R), "loop batch");
        }
        const auto t_sync = std::chrono::steady_clock::now();
        CK(cudaStreamSynchronize(st), "batch");
        const auto w1 = std::chrono::steady_clock::now();
        const float sync_ms = std::chrono::duration<float, std::milli>(w1 - t_sync).count();
        const float wall_ms = std::chrono::duration<float, std::milli>(w1 - w0).count();
        if (hl->stop == 4) return ctx->fail(FBB_E_STATE, "corrupt pending node (unscheduled-job count mismatch)");
        if (hl->stop == 5) return ctx->fail(FBB_E_STATE, "device loop: staging smaller than a planned pool");
        int valid = 0;
        while (valid < R && hl->rec[valid].valid) ++valid;
        const int64_t nb = (int64_t)row_bytes(ctx, ctx->host_pending && ctx->compact_rows);
        for (int i = 0; i < valid; ++i) {
            const LoopRecord& lr = hl->rec[i];
            fbb_round_t rec;
            std::memset(&rec, 0, sizeof(rec));
            rec.target = lr.target;
            rec.branched = lr.branched;
            rec.bounded = lr.bounded;
            rec.inserted = lr.inserted;
            rec.pruned = lr.pruned;
            rec.leaves = lr.leaves;
            rec.incumbent = lr.incumbent;
            rec.pending = lr.pending;
            // device clock: a round runs from its plan's start to the next round's plan
            // start (the last one: to its close's end), so the rounds tile the batch
            const unsigned long long t_next = i + 1 < valid ? hl->rec[i + 1].t0 : lr.t1;
            rec.round_ms = (float)((double)(t_next - lr.t0) * 1e-6);
            rec.k2_ms = lr.k2_t0 && lr.k2_t1 > lr.k2_t0 ? (float)((double)(lr.k2_t1 - lr.k2_t0) * 1e-6) : 0.f;
            // device-planned rounds: the lead-in, plan start .. first K2 CTA start (plan,
            // the launch or barrier after it, the leaves)
            rec.place_ms = lr.k2_t0 > lr.t0 ? (float)((double)(lr.k2_t0 - lr.t0) * 1e-6) : -1.f;
            rec.launches = pbk ? (i == 0 ? 1 : 0) : 5;  // the persistent kernel: one per batch
            rec.host_ms = wall_ms / valid;
            rec.sync_ms = sync_ms / valid;
            rec.h2d_bytes = ctx->host_pending ? lr.branched * nb : 0;  // rows of the host tree
            rec.d2h_bytes = ctx->host_pending ? lr.inserted * nb : 0;
            ctx->tot_branched += lr.branched;
            ctx->tot_bounded += lr.bounded;
            ctx->tot_pruned += lr.pruned;
            ctx->tot_leaves += lr.leaves;
            if (rounds) rounds[r] = rec;
            ++r;
        }
        if (done) *done = r;
        for (int d = 0; d <= n; ++d) ctx->cnt[d] = hl->cnt[d];
        ctx->incumbent = hl->incumbent;
        ctx->best = hl->best;
        ctx->found = hl->found;
        if (!ctx->frozen && hl->found)
            for (int i = 0; i < n; ++i) ctx->schedule[i] = hl->schedule[i];
        if (ctx->check) {
            int rc2 = check_pending(ctx);
            if (rc2 != FBB_OK) return rc2;
        }
        if (dbg && pbk && valid > 1) {  // where a persistent round's time goes (device clock)
            double a = 0, b = 0, k = 0, s = 0, e = 0;
            for (int i = 0; i + 1 < valid; ++i) {
                const LoopRecord& q = hl->rec[i];
                a += (double)(q.tp - q.t0);
                b += (double)(q.tb - q.tp);
                k += q.k2_t0 > q.tb ? (double)(q.k2_t0 - q.tb) : 0.0;
                s += (double)(q.k2_t1 - q.k2_t0);
                e += (double)(hl->rec[i + 1].t0 - q.k2_t1);
            }
            const double d = 1e3 * (valid - 1);
            fprintf(stderr, "[loop] per round us: plan %.2f barrier %.2f to-K2 %.2f K2 %.2f K2-end..next plan %.2f\n",
                    a / d, b / d, k / d, s / d, e / d);
        }
        if (dbg)
            fprintf(stderr, "[loop] batch R=%d valid=%d stop=%d persistent=%d setup_us=%.1f wall_us=%.1f\n", R, valid,
                    hl->stop, pbk ? 1 : 0,
                    std::chrono::duration<float, std::micro>(w0 - b0).count(), wall_ms * 1e3f);
        if (hl->stop == 3) {  // a destination bucket must grow before the next round
            const int d = hl->need_depth;
            const auto g0 = std::chrono::steady_clock::now();
            CK(store_ensure(ctx, ctx->bucket[d], hl->need_rows, ctx->cnt[d]), "bucket grow");
            if (dbg)
                fprintf(stderr, "[loop] grow bucket %d to %lld rows (cap %lld) in %.1f us\n", d,
                        (long long)hl->need_rows, (long long)ctx->bucket[d].cap,
                        std::chrono::duration<float, std::micro>(std::chrono::steady_clock::now() - g0).count());
            continue;
        }
        if (hl->stop == 6 && r < max_rounds) {  // a round larger than one wave: host-planned
            int64_t target = targets[r < ntargets ? r : ntargets - 1];
            fbb_round_t rec;
            const int rc = explorer_round(ctx, target < 1 ? 1 : target, &rec);
            if (rc != FBB_OK) return rc;
            if (rounds) rounds[r] = rec;
            ++r;
            if (done) *done = r;
            continue;
        }
        if (hl->stop == 1 || hl->stop == 2) break;
    }
    return FBB_OK;
}

}  // namespace

namespace fbb {
bool device_shared(int device) {
    // FBB_COOP=1: always (e.g. several processes sharing a GPU through MPS)
    static const bool force = [] { const char* e = getenv("FBB_COOP"); return e && e[0] == '1'; }();
    return force || device < 0 || device >= 64 || g_ctx_on_device[device].load() > 1;
}
}  // namespace fbb

// =========================================================================================
extern "C" {

const char* fbb_version(void) { return "flowbb-b200 0.2 (sm_100a)"; }

int fbb_kernels(fbb_ctx* ctx, char* buf, size_t cap) {
    if (!ctx || !buf || cap == 0) return FBB_E_ARG;
    char k1[64], k2[64];
    const K1Config& a = ctx->k1;
    if (a.variant == 0)
        std::snprintf(k1, sizeof k1, "k1_bound_kernel<%d,%d,%d>", ctx->dt.n <= 32 && !a.wide, a.jm_in_smem, a.wide);
    else if (a.variant >= 100) std::snprintf(k1, sizeof k1, "k1v3_kernel<%d>", a.variant - 100);
    else std::snprintf(k1, sizeof k1, "k1v2_kernel<%d,4>", a.variant);
    const K2Config& b = ctx->k2;
    if (b.variant >= 100000)
        std::snprintf(k2, sizeof k2, "k2_v3_kernel<%d,%d>", (b.variant / 100) % 100, b.variant % 100);
    else if (b.variant != 0)
        std::snprintf(k2, sizeof k2, "k2_v2_kernel<%d,%d,%d>", (b.variant / 100) % 100, b.variant % 100,
                      b.variant / 10000);
    else
        std::snprintf(k2, sizeof k2, "k2_internal_kernel<%d,%d>", b.jm_in_smem, b.wide);
    std::snprintf(buf, cap, "K1=%s K2=%s cmax=%d ppc_cap=%d blocks=%d batch=%d", k1, k2, b.cmax, b.ppc_cap, b.blocks,
                  b.batch ? 1 : 0);
    return FBB_OK;
}

fbb_ctx* fbb_create(int device, const int32_t* p, int n, int m) {
    auto fail = [&](int code, const std::string& m_) -> fbb_ctx* {
        std::lock_guard<std::mutex> g(g_err_mu);
        g_create_status = code;
        g_create_err = m_;
        return nullptr;
    };
    if (!p) return fail(FBB_E_ARG, "null processing-time matrix");
    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess || ndev == 0)
        return fail(FBB_E_CUDA, std::string("no CUDA device: ") + cudaGetErrorString(e));
    if (device < 0 || device >= ndev) return fail(FBB_E_ARG, "device index out of range");
    cudaDeviceProp prop;
    cudaGetDeviceProperties(&prop, device);
    if (prop.major != 10)
        return fail(FBB_E_CUDA, "this build targets sm_100a (B200); device is sm_" +
                                    std::to_string(prop.major * 10 + prop.minor));
    fbb_ctx* ctx = new fbb_ctx();
    ctx->device = device;
    if (device >= 0 && device < 64) g_ctx_on_device[device].fetch_add(1);
    std::string why;
    int rc = build_host_tables(p, n, m, &ctx->ht, &why);
    if (rc != FBB_OK) {
        g_ctx_on_device[device].fetch_sub(1);
        delete ctx;
        return fail(rc, why);
    }
    cudaSetDevice(device);
    if ((e = cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking)) != cudaSuccess) {
        g_ctx_on_device[device].fetch_sub(1);
        delete ctx;
        return fail(FBB_E_CUDA, std::string("stream: ") + cudaGetErrorString(e));
    }
    for (cudaEvent_t& ev : ctx->ev) cudaEventCreate(&ev);
    {
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
            uint64_t keep_all = UINT64_MAX;  // retain freed blocks for reuse
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep_all);
            // once per process and device: map a working set up front so that
            // pending-tree growth during a run is a pool hit, not a new mapping
            static std::mutex reserve_mu;
            static bool reserved[64] = {false};
            std::lock_guard<std::mutex> g(reserve_mu);
            if (device < 64 && !reserved[device]) {
                reserved[device] = true;
                size_t free_b = 0, total_b = 0;
                cudaMemGetInfo(&free_b, &total_b);
                // deep trees at large n keep one worst-case bucket per depth (200x20:
                // ~80 MB each), so map a generous working set: min(24 GiB, free / 4)
                size_t want = std::min<size_t>((size_t)24 << 30, free_b / 4);
                void* tmp = nullptr;
                if (cudaMallocAsync(&tmp, want, ctx->stream) == cudaSuccess) {
                    cudaFreeAsync(tmp, ctx->stream);
                    cudaStreamSynchronize(ctx->stream);
                }
            }
        }
        for (DBuf* b : {&ctx->k1_masks, &ctx->k1_heads, &ctx->k1_depth, &ctx->k1_lb, &ctx->out_lb,
                        &ctx->st_lb, &ctx->st_count, &ctx->st_seg, &ctx->d_pool, &ctx->d_round, &ctx->d_loop,
                        &ctx->d_rp})
            b->st = ctx->stream;
        for (Store* st : {&ctx->batch_in, &ctx->batch_out, &ctx->staging, &ctx->parents})
            st->set(ctx->stream, nullptr);
    }
    rc = upload_tables(ctx->ht, &ctx->dt, &why);
    if (rc != FBB_OK) {
        fbb_destroy(ctx);
        return fail(rc, why);
    }
    ctx->k1 = k1_config(ctx->dt, device);
    ctx->k2 = k2_config(ctx->dt, device);
    {
        // register-row K2 for n <= 32, m in {5,10,20}; tails packed as 16-bit there
        int32_t max_tail = 0;
        for (int32_t v : ctx->ht.tails) max_tail = std::max(max_tail, v);
        // FBB_K2=generic forces the generic kernel (A/B comparisons)
        K2Config kc;
        const char* sel = getenv("FBB_K2");
        bool generic = sel && std::string(sel) == "generic";
        // (both register-row kernels pack d as int8 and tails as 16 bits)
        if (max_tail < 0x7FFF && ctx->ht.max_abs_d <= 127 && !generic) {
            if (k2_v2_config(ctx->dt, device, &kc)) {
                ctx->k2 = kc;
                // the variant's staged rows (expand_v2.cu prologue), for its TMA bulk copy
                const int N = (kc.variant / 100) % 100, occ = kc.variant / 10000, n = ctx->dt.n, P = ctx->dt.P;
                const bool dual = occ == 2 && N == 20;
                std::vector<uint32_t> rows((size_t)N * P, N <= 32 ? 0u : 32u);
                for (int x = 0; x < n * P; ++x) {
                    const uint32_t e = ctx->ht.jm[x];
                    const uint32_t j = (uint32_t)entry_job(e);
                    rows[x] = (31u - (j & 31u)) | (j & 32u) | ((uint32_t)entry_c(e) << 8) |
                              ((uint32_t)(dual ? entry_d(e) : -entry_d(e)) << 24);
                }
                if (const char* tm = getenv("FBB_TMA"); !(tm && tm[0] == '0')) {
                    if (cudaMalloc(&ctx->dt.rowk2, rows.size() * 4) == cudaSuccess)
                        cudaMemcpy(ctx->dt.rowk2, rows.data(), rows.size() * 4, cudaMemcpyHostToDevice);
                    else
                        ctx->dt.rowk2 = nullptr;
                }
            }
            else if (k2_v3_config(ctx->dt, device, &kc)) ctx->k2 = kc;
        }
        // a variant that could not be configured must not leave its error behind for the
        // next launch check (cudaGetLastError)
        (void)cudaGetLastError();
    }
    int max_smem = 0;
    cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
    if (ctx->k1.smem > (size_t)max_smem || ctx->k2.smem > (size_t)max_smem) {
        fbb_destroy(ctx);
        return fail(FBB_E_RANGE, "instance tables exceed shared memory (n*P too large)");
    }
    explorer_clear(ctx);
    ctx->incumbent = INT_MAX;
    // Measured (r02): a single round is cheapest host-planned (fewer, exactly sized
    // launches: Ta021 262 K 121 vs 138 us of device time); a call of several rounds on an
    // HBM tree runs them as one conditional-graph batch with no host round trip (the Ta021
    // exhaustion: 19.5 vs 22.4 s)
    const char* dlp = getenv("FBB_DEVICE_LOOP");
    ctx->device_loop = !dlp ? -1 : (dlp[0] == '1' ? 1 : (dlp[0] == '0' ? 0 : -1));
    const char* sm = getenv("FBB_SUMMARY");
    ctx->summary_by_place = !(sm && std::string(sm) == "copy");
    const char* dir = getenv("FBB_DIRECT");
    ctx->direct_place = !(dir && dir[0] == '0');
    const char* chk = getenv("FBB_CHECK");
    ctx->check = chk && chk[0] == '1';
    preload_round_kernels();  // kernels load lazily: not inside the first round or graph capture
    preload_loop_kernels();
    return ctx;
}

void fbb_destroy(fbb_ctx* ctx) {
    if (!ctx) return;
    if (ctx->device >= 0 && ctx->device < 64) g_ctx_on_device[ctx->device].fetch_sub(1);
    cudaSetDevice(ctx->device);
    free_tables(&ctx->dt);
    for (DBuf* b : {&ctx->k1_masks, &ctx->k1_heads, &ctx->k1_depth, &ctx->k1_lb, &ctx->out_lb,
                    &ctx->st_lb, &ctx->st_count, &ctx->st_seg, &ctx->d_pool, &ctx->d_round, &ctx->d_rp})
        b->release();
    for (Store* s : {&ctx->batch_in, &ctx->batch_out, &ctx->staging, &ctx->parents}) {
        s->masks.release();
        s->heads.release();
        s->prefix.release();
    }
    for (Store& s : ctx->bucket) {
        s.masks.release();
        s.heads.release();
        s.prefix.release();
    }
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    ctx->h_pool.release();
    ctx->h_round.release();
    ctx->h_rp.release();
    ctx->h_loop.release();
    ctx->d_loop.release();
    for (auto& kv : ctx->loop_graphs) cudaGraphExecDestroy(kv.second);
    if (ctx->capture_stream) cudaStreamDestroy(ctx->capture_stream);
    if (ctx->capture_stream2) cudaStreamDestroy(ctx->capture_stream2);
    for (cudaEvent_t ev : ctx->ev)
        if (ev) cudaEventDestroy(ev);
    if (ctx->stream) cudaStreamDestroy(ctx->stream);
    delete ctx;
}

int fbb_last_error(const fbb_ctx* ctx, int* device, char* msg, size_t cap) {
    int status;
    std::string m;
    int dev = -1;
    if (ctx) {
        status = ctx->status;
        m = ctx->msg;
        dev = ctx->device;
    } else {
        std::lock_guard<std::mutex> g(g_err_mu);
        status = g_create_status;
        m = g_create_err;
    }
    if (device) *device = dev;
    if (msg && cap > 0) {
        size_t k = std::min(cap - 1, m.size());
        std::memcpy(msg, m.data(), k);
        msg[k] = 0;
    }
    return status;
}

int fbb_descriptor(fbb_ctx* ctx, fbb_descriptor_t* out) {
    if (!ctx || !out) return FBB_E_ARG;
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device);
    out->grain = ctx->k2.cmax;                                   // children per K2 tile
    out->base_units = std::max(1, ctx->k2.blocks);               // resident tiles (SMs x occupancy)
    size_t free_b = 0, total_b = 0;
    cudaSetDevice(ctx->device);
    cudaMemGetInfo(&free_b, &total_b);
    // children per round bounded by what the staging + buckets can hold in a quarter of HBM
    int64_t per_child = (int64_t)node_bytes(ctx) * 3 + 16;
    int64_t cap = (int64_t)(total_b / 4) / per_child;
    // and by 128 waves of resident tiles: past a few million children per round the
    // per-round fixed costs are amortised and bigger pools only grow the pending tree
    cap = std::min<int64_t>(cap, (int64_t)out->grain * out->base_units * 128);
    out->max_batch = std::max<int64_t>(cap - cap % out->grain, (int64_t)out->grain * out->base_units);
    (void)sms;
    return FBB_OK;
}

int fbb_bound_device(fbb_ctx* ctx, const uint64_t* d_masks, const int32_t* d_heads,
                     const int32_t* d_depth, int64_t count, int32_t* d_lb_out, void* stream) {
    if (!ctx) return FBB_E_ARG;
    if (count < 0) return ctx->fail(FBB_E_ARG, "negative count");
    if (count == 0) return FBB_OK;
    cudaSetDevice(ctx->device);
    cudaStream_t st = stream ? (cudaStream_t)stream : ctx->stream;
    // HBM-filling pools (billions of nodes): launches of at most 2^26 nodes, so every
    // in-kernel node x row index stays within 32 bits
    constexpr int64_t kSlice = int64_t(1) << 26;
    const int W = ctx->dt.W, m = ctx->dt.m;
    for (int64_t off = 0; off < count; off += kSlice) {
        const int64_t k = std::min(kSlice, count - off);
        CK(launch_k1(ctx->dt, ctx->k1, d_masks + off * W, d_heads + off * m, d_depth + off, k, d_lb_out + off, st),
           "K1 launch");
    }
    return FBB_OK;
}

int fbb_synth_pool(fbb_ctx* ctx, uint64_t seed, int64_t count, int32_t min_depth, int32_t max_depth,
                   uint64_t* d_masks, int32_t* d_heads, int32_t* d_depth, uint8_t* d_prefix, void* stream) {
    if (!ctx) return FBB_E_ARG;
    const int n = ctx->dt.n;
    if (count < 0 || min_depth < 0 || max_depth < min_depth || max_depth > n ||
        (count > 0 && (!d_masks || !d_heads || !d_depth)))
        return ctx->fail(FBB_E_ARG, "invalid synthetic pool request");
    cudaSetDevice(ctx->device);
    cudaStream_t st = stream ? (cudaStream_t)stream : ctx->stream;
    CK(launch_synth(ctx->dt, seed, count, min_depth, max_depth, d_masks, d_heads, d_depth, d_prefix, st),
       "synth launch");
    return FBB_OK;
}

int fbb_bound(fbb_ctx* ctx, const uint64_t* masks, const int32_t* heads, const int32_t* depth,
              int64_t count, int32_t* lb_out) {
    if (!ctx) return FBB_E_ARG;
    if (count < 0 || (count > 0 && (!masks || !heads || !depth || !lb_out)))
        return ctx->fail(FBB_E_ARG, "invalid node batch");
    if (count == 0) return FBB_OK;
    cudaSetDevice(ctx->device);
    const int m = ctx->dt.m, W = ctx->dt.W, n = ctx->dt.n;
    for (int64_t i = 0; i < count; ++i)
        if (depth[i] < 0 || depth[i] > n) return ctx->fail(FBB_E_ARG, "node depth out of range");
    CK(ctx->k1_masks.ensure((size_t)count * W * 8), "alloc");
    CK(ctx->k1_heads.ensure((size_t)count * m * 4), "alloc");
    CK(ctx->k1_depth.ensure((size_t)count * 4), "alloc");
    CK(ctx->k1_lb.ensure((size_t)count * 4), "alloc");
    cudaStream_t st = ctx->stream;
    CK(cudaMemcpyAsync(ctx->k1_masks.p, masks, (size_t)count * W * 8, cudaMemcpyHostToDevice, st), "H2D");
    CK(cudaMemcpyAsync(ctx->k1_heads.p, heads, (size_t)count * m * 4, cudaMemcpyHostToDevice, st), "H2D");
    CK(cudaMemcpyAsync(ctx->k1_depth.p, depth, (size_t)count * 4, cudaMemcpyHostToDevice, st), "H2D");
    CK(launch_k1(ctx->dt, ctx->k1, ctx->k1_masks.as<uint64_t>(), ctx->k1_heads.as<int32_t>(),
                 ctx->k1_depth.as<int32_t>(), count, ctx->k1_lb.as<int32_t>(), st),
       "K1 launch");
    CK(cudaMemcpyAsync(lb_out, ctx->k1_lb.p, (size_t)count * 4, cudaMemcpyDeviceToHost, st), "D2H");
    CK(cudaStreamSynchronize(st), "K1");
    return FBB_OK;
}

int fbb_expand_bound_prune(fbb_ctx* ctx, const uint64_t* masks, const int32_t* heads,
                           const int32_t* depth, const uint8_t* prefix, int64_t nparents,
                           int32_t ub, int frozen, uint64_t* out_masks, int32_t* out_heads,
                           int32_t* out_depth, uint8_t* out_prefix, int32_t* out_lb,
                           int64_t* out_count, int32_t* leaf_best, int64_t* leaf_pos,
                           int32_t* leaf_schedule, fbb_round_t* counts) {
    if (!ctx) return FBB_E_ARG;
    const int n = ctx->dt.n, m = ctx->dt.m, W = ctx->dt.W;
    if (nparents < 0 || (nparents > 0 && (!masks || !heads || !depth || !prefix)) || !out_count)
        return ctx->fail(FBB_E_ARG, "invalid parent batch");
    cudaSetDevice(ctx->device);
    // runs of equal depth, non-increasing (fill_buffer's pop order)
    Pool pool;
    pool.nseg = 0;
    for (int64_t i = 0; i < nparents; ++i) {
        int d = depth[i];
        if (d < 0 || d >= n) return ctx->fail(FBB_E_ARG, "parent depth must be in [0, n)");
        if (pool.nseg > 0 && pool.seg[pool.nseg - 1].depth == d) {
            pool.seg[pool.nseg - 1].count++;
            continue;
        }
        if (pool.nseg > 0 && d > pool.seg[pool.nseg - 1].depth)
            return ctx->fail(FBB_E_ARG, "parents must be in non-increasing depth order (pop order)");
        Segment& sg = pool.seg[pool.nseg++];
        std::memset(&sg, 0, sizeof(sg));
        sg.first = i;
        sg.step = 1;
        sg.count = 1;
        sg.depth = d;
    }
    fbb_round_t rec;
    std::memset(&rec, 0, sizeof(rec));
    rec.incumbent = ub;
    *out_count = 0;
    if (leaf_best) *leaf_best = INT32_MAX;
    if (leaf_pos) *leaf_pos = -1;
    if (nparents == 0) {
        if (counts) *counts = rec;
        return FBB_OK;
    }
    CK(store_ensure(ctx, ctx->batch_in, nparents, 0), "alloc");
    cudaStream_t st = ctx->stream;
    Store& in = ctx->batch_in;
    CK(cudaMemcpyAsync(in.masks.p, masks, (size_t)nparents * W * 8, cudaMemcpyHostToDevice, st), "H2D");
    CK(cudaMemcpyAsync(in.heads.p, heads, (size_t)nparents * m * 4, cudaMemcpyHostToDevice, st), "H2D");
    CK(cudaMemcpyAsync(in.prefix.p, prefix, (size_t)nparents * n, cudaMemcpyHostToDevice, st), "H2D");
    int first_internal = layout_pool(ctx, pool);
    pool.host_dst = 0;  // survivors go to the device output batch
    CK(store_ensure(ctx, ctx->batch_out, std::max<int64_t>(pool.nchildren, 1), 0), "alloc");
    CK(ctx->out_lb.ensure((size_t)std::max<int64_t>(pool.nchildren, 1) * 4), "alloc");
    for (int s = 0; s < pool.nseg; ++s) {
        pool.seg[s].src = in.view();
        pool.seg[s].dst = ctx->batch_out.view();
        pool.seg[s].dst_base = -1;
        pool.seg[s].dst_lb = ctx->out_lb.as<int32_t>();
    }
    int rc = run_pool(ctx, pool, first_internal, ub, frozen);
    if (rc != FBB_OK) return rc;
    const RoundState* sm = ctx->h_round.as<RoundState>();
    int64_t total = sm->total;
    *out_count = total;
    if (total > 0) {
        if (out_masks)
            CK(cudaMemcpyAsync(out_masks, ctx->batch_out.masks.p, (size_t)total * W * 8, cudaMemcpyDeviceToHost, st), "D2H");
        if (out_heads)
            CK(cudaMemcpyAsync(out_heads, ctx->batch_out.heads.p, (size_t)total * m * 4, cudaMemcpyDeviceToHost, st), "D2H");
        if (out_prefix)
            CK(cudaMemcpyAsync(out_prefix, ctx->batch_out.prefix.p, (size_t)total * n, cudaMemcpyDeviceToHost, st), "D2H");
        if (out_lb)
            CK(cudaMemcpyAsync(out_lb, ctx->out_lb.p, (size_t)total * 4, cudaMemcpyDeviceToHost, st), "D2H");
        CK(cudaStreamSynchronize(st), "D2H");
    }
    int64_t internal = 0, leaves = 0, o = 0;
    for (int s = 0; s < pool.nseg; ++s) {
        const Segment& sg = pool.seg[s];
        int64_t kids = sg.count * (n - sg.depth);
        rec.branched += sg.count;
        if (sg.depth >= n - 2) {
            leaves += kids;
        } else {
            internal += kids;
            if (out_depth)
                for (int64_t i = 0; i < sm->seg_surv[s]; ++i) out_depth[o + i] = sg.depth + 1;
            o += sm->seg_surv[s];
        }
    }
    rec.bounded = internal + leaves;
    rec.leaves = leaves;
    rec.inserted = total;
    rec.pruned = internal - total;
    rec.k2_ms = ctx->last_k2_ms;
    rec.round_ms = ctx->last_round_ms;
    rec.launches = ctx->last_launches;
    int32_t v;
    int64_t vpos;
    if (leaves > 0 && round_leaf(sm, &v, &vpos)) {
        if (v < ub) {
            if (leaf_best) *leaf_best = v;
            if (leaf_pos) *leaf_pos = vpos;
            if (leaf_schedule && sm->found) std::memcpy(leaf_schedule, sm->schedule, (size_t)n * 4);
            if (!frozen) rec.incumbent = v;
        }
    }
    if (counts) *counts = rec;
    return FBB_OK;
}

int fbb_explorer_set_residency(fbb_ctx* ctx, int pending_on_host) {
    if (!ctx) return FBB_E_ARG;
    cudaSetDevice(ctx->device);
    ctx->host_pending = pending_on_host != 0;
    if (ctx->host_pending) {
        // reserve the pinned arena now (page locking costs ~0.25 s per GB), not mid-run:
        // 1 GiB, or twice what the HBM-resident tree of this context has grown to
        size_t dev_bytes = 0;
        for (const Store& b : ctx->bucket)
            if (!b.prefix.arena) dev_bytes += (size_t)b.cap * node_bytes(ctx);
        const char* mb = getenv("FBB_PINNED_MB");
        size_t want = mb ? (size_t)std::max(64L, atol(mb)) << 20
                         : std::max<size_t>((size_t)1 << 30, 2 * dev_bytes);
        void* p = nullptr;
        if (ctx->arena.alloc(want, &p) == cudaSuccess) ctx->arena.release(p, want);
        // compact (prefix-only) rows when the staging fold is short: it costs depth * m
        // dependent max-plus steps per parent, free at n <= 32 (Ta021: K2 unchanged) but
        // +20 % of K2 at 100x20, where deep parents fold up to ~100 jobs
        const char* rows = getenv("FBB_HOST_ROWS");
        ctx->compact_rows = rows ? std::string(rows) != "full" : ctx->dt.n <= 32;
        const char* o = getenv("FBB_HOST_OUT");
        ctx->mapped_out = !(o && std::string(o) == "staged");
        const char* i = getenv("FBB_HOST_IN");
        // in-place reads need occupancy to hide the host-link latency: only the
        // register-row K2 (3 CTAs/SM) reads mapped parents by default
        ctx->mapped_in = i ? std::string(i) != "copy" : ctx->k2.variant != 0;
    }
    explorer_clear(ctx);
    return FBB_OK;
}

int fbb_explorer_reset(fbb_ctx* ctx, const uint8_t* prefix, const int32_t* depth, int64_t count,
                       int32_t ub, int frozen) {
    if (!ctx) return FBB_E_ARG;
    if (count < 0 || (count > 0 && (!prefix || !depth))) return ctx->fail(FBB_E_ARG, "invalid nodes");
    cudaSetDevice(ctx->device);
    explorer_clear(ctx);
    ctx->incumbent = ub;
    ctx->frozen = frozen ? 1 : 0;
    ctx->found = 0;
    return push_host_nodes(ctx, prefix, depth, count);
}

int fbb_explorer_start_solve(fbb_ctx* ctx, int32_t ub, fbb_round_t* round0) {
    if (!ctx) return FBB_E_ARG;
    cudaSetDevice(ctx->device);
    explorer_clear(ctx);
    const int n = ctx->dt.n, m = ctx->dt.m, W = ctx->dt.W;
    ctx->frozen = 0;
    if (ub >= 0) {
        ctx->incumbent = ub;
        ctx->found = 0;
    } else {  // identity permutation, search.hpp:131-137
        std::vector<int32_t> h(m, 0);
        for (int j = 0; j < n; ++j) {
            int32_t prev = 0;
            for (int k = 0; k < m; ++k) {
                prev = std::max(prev, h[k]) + ctx->ht.p[(size_t)j * m + k];
                h[k] = prev;
            }
            ctx->schedule[j] = j;
        }
        ctx->incumbent = h[m - 1];
        ctx->best = ctx->incumbent;
        ctx->found = 1;
    }
    // round 0: bound the root (search.hpp:150-153), integrate it
    std::vector<uint64_t> mk(W, 0);
    std::vector<int32_t> hd(m, 0);
    int32_t dep = 0, lb = 0;
    int rc = fbb_bound(ctx, mk.data(), hd.data(), &dep, 1, &lb);
    if (rc != FBB_OK) return rc;
    fbb_round_t rec;
    std::memset(&rec, 0, sizeof(rec));
    rec.bounded = 1;
    if (lb < ctx->incumbent) {  // the root is internal for every n >= 1
        rec.inserted = 1;
        uint8_t pr = 0;
        rc = push_host_nodes(ctx, &pr, &dep, 1);
        if (rc != FBB_OK) return rc;
    } else {
        rec.pruned = 1;
    }
    ctx->tot_bounded = 1;
    ctx->tot_pruned = rec.pruned;
    rec.incumbent = ctx->incumbent;
    rec.pending = pending_total(ctx);
    if (round0) *round0 = rec;
    return FBB_OK;
}

int fbb_explorer_run(fbb_ctx* ctx, const int64_t* targets, int ntargets, int64_t max_rounds,
                     int64_t budget, fbb_round_t* rounds, int64_t* done) {
    if (!ctx) return FBB_E_ARG;
    if (!targets || ntargets < 1) return ctx->fail(FBB_E_ARG, "need at least one target");
    cudaSetDevice(ctx->device);
    if (device_loop_ok(ctx, max_rounds))
        return explorer_run_batched(ctx, targets, ntargets, max_rounds, budget, rounds, done);
    int64_t r = 0;
    if (done) *done = 0;
    while (r < max_rounds) {
        if (pending_total(ctx) == 0) break;
        if (budget > 0 && ctx->tot_bounded >= budget) break;
        int64_t target = targets[r < ntargets ? r : ntargets - 1];
        if (target < 1) target = 1;
        fbb_round_t rec;
        int rc = explorer_round(ctx, target, &rec);
        if (rc != FBB_OK) return rc;
        if (rounds) rounds[r] = rec;
        ++r;
        if (done) *done = r;
    }
    return FBB_OK;
}

int fbb_explorer_state(fbb_ctx* ctx, int32_t* incumbent, int32_t* found, int32_t* schedule,
                       int64_t* pending, int64_t* totals4) {
    if (!ctx) return FBB_E_ARG;
    if (incumbent) *incumbent = ctx->frozen ? (ctx->found ? ctx->best : ctx->incumbent) : ctx->incumbent;
    if (found) *found = ctx->found;
    if (schedule && ctx->found) std::memcpy(schedule, ctx->schedule.data(), ctx->schedule.size() * 4);
    if (pending) *pending = pending_total(ctx);
    if (totals4) {
        totals4[0] = ctx->tot_branched;
        totals4[1] = ctx->tot_bounded;
        totals4[2] = ctx->tot_pruned;
        totals4[3] = ctx->tot_leaves;
    }
    return FBB_OK;
}

int fbb_explorer_set_incumbent(fbb_ctx* ctx, int32_t ub) {
    if (!ctx) return FBB_E_ARG;
    if (ctx->frozen) return ctx->fail(FBB_E_STATE, "the incumbent of a frozen exploration is fixed");
    if (ub < ctx->incumbent) ctx->incumbent = ub;  // a better incumbent found elsewhere
    return FBB_OK;
}

int fbb_explorer_best(fbb_ctx* ctx, int32_t* value, int32_t* schedule) {
    if (!ctx) return FBB_E_ARG;
    if (!ctx->found) {
        if (value) *value = INT32_MAX;
        return 0;
    }
    if (value) *value = ctx->best;
    if (schedule && !ctx->frozen) std::memcpy(schedule, ctx->schedule.data(), ctx->schedule.size() * 4);
    return 1;
}

int fbb_explorer_take(fbb_ctx* ctx, int64_t k, uint8_t* prefix, int32_t* depth, int64_t* taken) {
    if (!ctx || !taken || k < 0 || (k > 0 && (!prefix || !depth))) return FBB_E_ARG;
    cudaSetDevice(ctx->device);
    const int n = ctx->dt.n;
    int64_t t = 0;
    for (int d = 0; d <= n && t < k; ++d) {
        const int64_t j = std::min<int64_t>(ctx->cnt[d], k - t);
        if (j == 0) continue;
        const int64_t lo = ctx->cnt[d] - j;  // the bucket's top rows
        CK(cudaMemcpyAsync(prefix + t * n, ctx->bucket[d].prefix.as<uint8_t>() + lo * n, (size_t)j * n,
                           cudaMemcpyDefault, ctx->stream),
           "take D2H");
        for (int64_t i = 0; i < j; ++i) depth[t + i] = d;
        ctx->cnt[d] = lo;
        t += j;
    }
    CK(cudaStreamSynchronize(ctx->stream), "take");
    *taken = t;
    return FBB_OK;
}

int fbb_explorer_push(fbb_ctx* ctx, const uint8_t* prefix, const int32_t* depth, int64_t count) {
    if (!ctx) return FBB_E_ARG;
    if (count < 0 || (count > 0 && (!prefix || !depth))) return ctx->fail(FBB_E_ARG, "invalid nodes");
    if (!ctx->explorer_ready) return ctx->fail(FBB_E_STATE, "explorer not reset");
    cudaSetDevice(ctx->device);
    return push_host_nodes(ctx, prefix, depth, count);
}

int fbb_explorer_pending(fbb_ctx* ctx, uint8_t* prefix, int32_t* depth, int64_t cap, int64_t* count) {
    if (!ctx || !count) return FBB_E_ARG;
    cudaSetDevice(ctx->device);
    const int n = ctx->dt.n;
    int64_t total = pending_total(ctx);
    *count = total;
    if (cap < total) return ctx->fail(FBB_E_ARG, "buffer too small for the pending tree");
    int64_t o = 0;
    for (int d = 0; d <= n; ++d) {
        int64_t k = ctx->cnt[d];
        if (k == 0) continue;
        if (prefix) {
            CK(cudaMemcpyAsync(prefix + o * n, ctx->bucket[d].prefix.p, (size_t)k * n,
                               cudaMemcpyDefault, ctx->stream),
               "pending D2H");
            CK(cudaStreamSynchronize(ctx->stream), "pending D2H");
        }
        if (depth)
            for (int64_t i = 0; i < k; ++i) depth[o + i] = d;
        o += k;
    }
    return FBB_OK;
}

}  // extern "C"
