// gpu_backend.hpp -- header-only C++ drop-in for the reference flowbb API.
//
// Include AFTER the reference headers are on the include path (-I proj/include)
// and link libflowbb_b200.so.  Provides:
//
//   flowbb_b200::GpuBackend      models the reference's duck-typed Backend concept
//                                (descriptor() + evaluate(inst, span<const Node>),
//                                backend.hpp:50-69, used by evaluate_multi<Backend>,
//                                backend.hpp:105-138) over fbb_bound (K1);
//   flowbb_b200::GpuBackendSet   BackendSet (backend.hpp:140-158) over GPUs;
//   flowbb_b200::gpu_round       the fused replacement of one reference round
//                                fill_buffer -> evaluate -> integrate / frozen
//                                prune (search.hpp:64-107, bench.hpp:88-106)
//                                over fbb_expand_bound_prune (K2), operating on
//                                the reference's own PendingTree and Incumbent.
//
// Errors surface as flowbb::BackendError(device, message), like a failing
// CpuBackend slice (backend.hpp:124-136).
#ifndef FLOWBB_B200_GPU_BACKEND_HPP
#define FLOWBB_B200_GPU_BACKEND_HPP

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <functional>
#include <memory>
#include <mutex>
#include <optional>
#include <span>
#include <string>
#include <vector>

#include "flowbb/autotune.hpp"
#include "flowbb/backend.hpp"
#include "flowbb/bench.hpp"
#include "flowbb/pending.hpp"
#include "flowbb/search.hpp"
#include "flowbb/workload.hpp"
#include "flowbb_b200.h"

namespace flowbb_b200 {

namespace detail {

inline std::string last_error(const fbb_ctx* ctx, int* device) {
    char buf[512];
    fbb_last_error(ctx, device, buf, sizeof(buf));
    return buf;
}

// One device context per (device, instance); created on first use.
class ContextCache {
public:
    explicit ContextCache(int device) : device_(device) {}
    ~ContextCache() {
        if (ctx_) fbb_destroy(ctx_);
    }
    fbb_ctx* get(const flowbb::Instance& inst) {
        std::lock_guard<std::mutex> g(mu_);
        std::vector<int32_t> p(static_cast<std::size_t>(inst.jobs()) * inst.machines());
        for (int j = 0; j < inst.jobs(); ++j)
            for (int k = 0; k < inst.machines(); ++k) p[j * inst.machines() + k] = inst.p(j, k);
        if (ctx_ && p == p_) return ctx_;
        if (ctx_) fbb_destroy(ctx_);
        ctx_ = fbb_create(device_, p.data(), inst.jobs(), inst.machines());
        if (!ctx_) {
            int dev = device_;
            throw flowbb::BackendError(device_, last_error(nullptr, &dev));
        }
        p_ = std::move(p);
        return ctx_;
    }
    std::mutex& call_mutex() { return call_mu_; }

private:
    int device_;
    std::mutex mu_, call_mu_;
    fbb_ctx* ctx_ = nullptr;
    std::vector<int32_t> p_;
};

// Node (node.hpp:28-53) -> SoA row
inline void pack(const flowbb::Instance& inst, const flowbb::Node& node, uint64_t* mask,
                 int32_t* heads, uint8_t* prefix) {
    const int n = inst.jobs(), W = (n + 63) / 64;
    for (int w = 0; w < W; ++w) mask[w] = 0;
    for (int j = 0; j < n; ++j)
        if (node.scheduled.test(j)) mask[j >> 6] |= uint64_t{1} << (j & 63);
    for (int k = 0; k < inst.machines(); ++k) heads[k] = node.heads[k];
    if (prefix)
        for (int i = 0; i < node.depth(); ++i) prefix[i] = static_cast<uint8_t>(node.prefix[i]);
}

}  // namespace detail

class GpuBackend {
public:
    explicit GpuBackend(int device = 0,
                        flowbb::BackendDescriptor descriptor = flowbb::BackendDescriptor{256, 148, 1 << 24})
        : device_(device), descriptor_(descriptor),
          cache_(std::make_shared<detail::ContextCache>(device)) {}

    const flowbb::BackendDescriptor& descriptor() const { return descriptor_; }
    int device() const { return device_; }

    // CpuBackend::evaluate (backend.hpp:63-65): position-aligned lower_bound of every node.
    std::vector<int> evaluate(const flowbb::Instance& inst, std::span<const flowbb::Node> nodes) const {
        std::vector<int> out(nodes.size());
        if (nodes.empty()) return out;
        fbb_ctx* ctx = cache_->get(inst);
        const int n = inst.jobs(), m = inst.machines(), W = (n + 63) / 64;
        thread_local std::vector<uint64_t> masks;  // reused across calls (no re-initialisation)
        thread_local std::vector<int32_t> heads, depth;
        // each buffer sized on its own: W and m change with the instance
        if (masks.size() < nodes.size() * W) masks.resize(nodes.size() * W);
        if (heads.size() < nodes.size() * m) heads.resize(nodes.size() * m);
        if (depth.size() < nodes.size()) depth.resize(nodes.size());
        for (std::size_t i = 0; i < nodes.size(); ++i) {
            detail::pack(inst, nodes[i], &masks[i * W], &heads[i * m], nullptr);
            depth[i] = nodes[i].depth();
        }
        std::lock_guard<std::mutex> g(cache_->call_mutex());
        int rc = fbb_bound(ctx, masks.data(), heads.data(), depth.data(),
                           static_cast<int64_t>(nodes.size()), out.data());
        if (rc != FBB_OK) {
            int dev = device_;
            throw flowbb::BackendError(device_, detail::last_error(ctx, &dev));
        }
        return out;
    }

    fbb_ctx* context(const flowbb::Instance& inst) const { return cache_->get(inst); }
    std::mutex& call_mutex() const { return cache_->call_mutex(); }

private:
    int device_;
    flowbb::BackendDescriptor descriptor_;
    std::shared_ptr<detail::ContextCache> cache_;
};

// BackendSet (backend.hpp:140-158) with backend i on device devices[i % size].
class GpuBackendSet {
public:
    GpuBackendSet(int count, std::vector<int> devices = {0},
                  flowbb::BackendDescriptor descriptor = flowbb::BackendDescriptor{256, 148, 1 << 24}) {
        if (count < 1) throw std::invalid_argument("backend count must be positive");
        for (int i = 0; i < count; ++i)
            backends_.emplace_back(devices[static_cast<std::size_t>(i) % devices.size()], descriptor);
    }
    int size() const { return static_cast<int>(backends_.size()); }
    const flowbb::BackendDescriptor& descriptor() const { return backends_.front().descriptor(); }
    std::vector<int> evaluate(const flowbb::Instance& inst, std::span<const flowbb::Node> batch) const {
        return flowbb::evaluate_multi<GpuBackend>(backends_, inst, batch);
    }
    const GpuBackend& front() const { return backends_.front(); }

private:
    std::vector<GpuBackend> backends_;
};

struct RoundCounts {
    std::int64_t branched = 0, bounded = 0, inserted = 0, pruned = 0, leaves = 0;
};

// One fused round on the reference's own PendingTree: pops exactly the parents
// fill_buffer would (search.hpp:64-73), expands/bounds/prunes their children on
// the GPU (K2), pushes the survivors in batch order.  frozen == false follows
// integrate (search.hpp:84-107: strict improvement, mid-batch incumbent);
// frozen == true the resolve loop (bench.hpp:96-106; `best` tracks the leaf
// minimum under the frozen incumbent).
inline RoundCounts gpu_round(const GpuBackend& backend, const flowbb::Instance& inst,
                             flowbb::PendingTree& pending, flowbb::Incumbent& incumbent,
                             std::size_t target, bool frozen, std::optional<int>* best = nullptr) {
    RoundCounts rc;
    const int n = inst.jobs(), m = inst.machines(), W = (n + 63) / 64;
    // per-thread buffers reused across rounds (a 262 K-child round's output arrays are
    // ~30 MB: value-initialising them every round cost more than the GPU round itself)
    thread_local std::vector<uint64_t> masks, omask;
    thread_local std::vector<int32_t> heads, depth, oheads, odepth, olb;
    thread_local std::vector<uint8_t> prefix, oprefix;
    depth.clear();
    std::size_t children = 0;
    while (children < target && !pending.empty()) {
        flowbb::Node node = pending.pop();
        ++rc.branched;
        std::size_t i = depth.size();
        // each buffer sized on its own (n, m, W change with the instance)
        if (masks.size() < (i + 1) * W) masks.resize(2 * (i + 1) * W);
        if (heads.size() < (i + 1) * m) heads.resize(2 * (i + 1) * m);
        if (prefix.size() < (i + 1) * n) prefix.resize(2 * (i + 1) * n);
        detail::pack(inst, node, &masks[i * W], &heads[i * m], &prefix[i * n]);
        depth.push_back(node.depth());
        children += static_cast<std::size_t>(n - node.depth());
    }
    if (depth.empty()) return rc;
    if (omask.size() < children * W) omask.resize(children * W);
    if (oheads.size() < children * m) oheads.resize(children * m);
    if (odepth.size() < children) odepth.resize(children);
    if (olb.size() < children) olb.resize(children);
    if (oprefix.size() < children * n) oprefix.resize(children * n);
    std::vector<int32_t> sched(n);
    int64_t count = 0, pos = 0;
    int32_t leaf_best = 0;
    fbb_round_t rec;
    fbb_ctx* ctx = backend.context(inst);
    {
        std::lock_guard<std::mutex> g(backend.call_mutex());
        int st = fbb_expand_bound_prune(ctx, masks.data(), heads.data(), depth.data(), prefix.data(),
                                        static_cast<int64_t>(depth.size()), incumbent.value,
                                        frozen ? 1 : 0, omask.data(), oheads.data(), odepth.data(),
                                        oprefix.data(), olb.data(), &count, &leaf_best, &pos,
                                        sched.data(), &rec);
        if (st != FBB_OK) {
            int dev = backend.device();
            throw flowbb::BackendError(backend.device(), detail::last_error(ctx, &dev));
        }
    }
    for (int64_t i = 0; i < count; ++i) {
        flowbb::Node node = flowbb::Node::root(inst);
        node.prefix.reserve(static_cast<std::size_t>(odepth[i]));
        for (int d = 0; d < odepth[i]; ++d) {
            int j = oprefix[i * n + d];
            node.prefix.push_back(j);
            node.scheduled.set(j);
        }
        for (int k = 0; k < m; ++k) node.heads[k] = oheads[i * m + k];
        node.lb = olb[i];
        pending.push(std::move(node));
    }
    if (leaf_best != INT32_MAX) {
        if (frozen) {
            if (best && leaf_best < incumbent.value && (!*best || leaf_best < **best)) *best = leaf_best;
        } else if (leaf_best < incumbent.value) {
            incumbent.value = leaf_best;
            incumbent.schedule = flowbb::Permutation(sched.begin(), sched.end());
        }
    }
    rc.bounded = rec.bounded;
    rc.inserted = rec.inserted;
    rc.pruned = rec.pruned;
    rc.leaves = rec.leaves;
    return rc;
}

// ---- workload snapshots and the speedup protocol ----------------------------

// generate_workload (workload.hpp:62-98) with the children's bounds from the GPU: the
// same frozen-UB sequential capture, the same mt19937 deterministic shuffle of each
// expansion's children, the same pushes -- so save_workload of the result is
// byte-identical to the reference's.
inline flowbb::WorkloadSnapshot generate_workload(const GpuBackend& gpu, const flowbb::Instance& inst,
                                                  int initial_ub, flowbb::CaptureCutoff cutoff,
                                                  std::uint32_t seed,
                                                  std::function<double()> clock = {}) {
    using flowbb::CaptureCutoff;
    if (cutoff.kind == CaptureCutoff::Kind::wall_time && !clock) {
        auto start = std::chrono::steady_clock::now();
        clock = [start] {
            return std::chrono::duration<double>(std::chrono::steady_clock::now() - start).count();
        };
    }
    std::mt19937 rng(seed);
    flowbb::PendingTree pending(inst.jobs());
    auto expand = [&](const flowbb::Node& node) {
        std::vector<flowbb::Node> children = flowbb::branch(inst, node);
        flowbb::detail::deterministic_shuffle(children, rng);
        std::vector<int> lbs = gpu.evaluate(inst, children);  // K1, one call per expansion
        for (std::size_t i = 0; i < children.size(); ++i) {
            flowbb::Node& child = children[i];
            if (child.depth() == inst.jobs()) continue;  // incumbent frozen, leaves dropped
            child.lb = lbs[i];
            if (child.lb < initial_ub) pending.push(std::move(child));
        }
    };
    expand(flowbb::Node::root(inst));
    std::int64_t branched = 0;
    while (!pending.empty()) {
        if (cutoff.kind == CaptureCutoff::Kind::node_count) {
            if (branched >= cutoff.nodes) break;
        } else if (clock() >= cutoff.seconds) {
            break;
        }
        expand(pending.pop());
        ++branched;
    }
    return flowbb::WorkloadSnapshot{inst, pending.drain(), initial_ub, seed, cutoff};
}

// resolve_workload (bench.hpp:63-114) on the GPU: fused rounds (gpu_round, frozen) over
// the reference's own PendingTree; batch from config.batch, or the adaptive tuner
// observing each round's time (config.autotune).  Same best and nodes_bounded as the
// reference for every batch (frozen-UB exploration is partition-invariant).
inline flowbb::ResolutionResult resolve_workload(const GpuBackend& gpu,
                                                 const flowbb::WorkloadSnapshot& snapshot,
                                                 const flowbb::BenchConfig& config) {
    using clock = std::chrono::steady_clock;
    const flowbb::Instance& inst = snapshot.instance;
    std::optional<flowbb::Tuner> tuner;
    if (config.autotune) tuner.emplace(config.descriptor, config.window, config.probes);
    const std::size_t fixed = config.batch ? static_cast<std::size_t>(*config.batch)
                                           : static_cast<std::size_t>(config.descriptor.grain) *
                                                 config.descriptor.base_units;
    auto t0 = clock::now();
    flowbb::PendingTree pending(inst.jobs());
    for (const flowbb::Node& node : snapshot.nodes) pending.push(node);
    flowbb::Incumbent inc{snapshot.incumbent_value, std::nullopt};
    flowbb::ResolutionResult result;
    std::size_t last = fixed;
    while (!pending.empty()) {
        const std::size_t target = tuner ? static_cast<std::size_t>(tuner->target()) : fixed;
        last = target;
        auto e0 = clock::now();
        RoundCounts rc = gpu_round(gpu, inst, pending, inc, target, true, &result.best);
        result.nodes_bounded += rc.bounded;
        if (tuner)
            tuner->observe(rc.bounded, std::max(std::chrono::duration<double>(clock::now() - e0).count(), 1e-9));
    }
    result.elapsed_seconds = std::chrono::duration<double>(clock::now() - t0).count();
    result.batch_used = tuner ? tuner->best_batch() : static_cast<int>(last);
    if (tuner && result.batch_used == 0) result.batch_used = tuner->target();
    return result;
}

// run_experiment (bench.hpp:119-145) with the parallel side on the GPU: the reference's
// strictly sequential CPU resolution (one backend, batch 1 -- the paper's Tcpu) against
// each GPU configuration; any disagreement in the best leaf or the bounded-node count
// throws flowbb::ResolutionMismatch.
inline flowbb::Report run_experiment(const GpuBackend& gpu, const flowbb::WorkloadSnapshot& snapshot,
                                     const std::vector<flowbb::BenchConfig>& configs) {
    flowbb::BenchConfig sequential;
    sequential.backends = 1;
    sequential.batch = 1;
    flowbb::ResolutionResult seq = flowbb::resolve_workload(snapshot, sequential);
    flowbb::Report report;
    for (const flowbb::BenchConfig& config : configs) {
        flowbb::ResolutionResult par = resolve_workload(gpu, snapshot, config);
        if (par.best != seq.best)
            throw flowbb::ResolutionMismatch("optimum mismatch between sequential and GPU resolution");
        if (par.nodes_bounded != seq.nodes_bounded)
            throw flowbb::ResolutionMismatch("bounded-node count mismatch between resolutions");
        flowbb::ReportRow row;
        row.jobs = snapshot.instance.jobs();
        row.machines = snapshot.instance.machines();
        row.batch = par.batch_used;
        row.backends = 1;
        row.t_seq = seq.elapsed_seconds;
        row.t_par = par.elapsed_seconds;
        row.speedup = seq.elapsed_seconds / std::max(par.elapsed_seconds, 1e-12);
        row.nodes_bounded = par.nodes_bounded;
        report.rows.push_back(row);
    }
    return report;
}

// The multi-GPU explorer of one process over fbb_group_* (include/flowbb_b200.h): the
// reference's solve / resolve_workload (search.hpp:124-174, bench.hpp:63-114) with each
// GPU exploring its own share of the pending tree, the incumbent min-exchanged between
// steps and starving GPUs fed subtrees.  Frozen exploration gives the
// reference's node counts for any GPU count (bench.hpp:60-62).
class GpuGroupExplorer {
public:
    GpuGroupExplorer(const flowbb::Instance& inst, const std::vector<int>& devices) : n_(inst.jobs()) {
        std::vector<int32_t> p((std::size_t)inst.jobs() * inst.machines());
        for (int j = 0; j < inst.jobs(); ++j)
            for (int k = 0; k < inst.machines(); ++k) p[(std::size_t)j * inst.machines() + k] = inst.p(j, k);
        g_ = fbb_group_create(devices.data(), (int)devices.size(), p.data(), inst.jobs(), inst.machines());
        if (!g_) {
            int dev = -1;
            std::string m = detail::last_error(nullptr, &dev);
            throw flowbb::BackendError{dev < 0 ? 0 : dev, m};
        }
    }
    ~GpuGroupExplorer() { fbb_group_destroy(g_); }
    GpuGroupExplorer(const GpuGroupExplorer&) = delete;
    GpuGroupExplorer& operator=(const GpuGroupExplorer&) = delete;

    // resolve_workload's start (bench.hpp:80-85): the snapshot nodes, frozen incumbent
    void reset(const std::vector<flowbb::Node>& nodes, int ub, bool frozen = true) {
        std::vector<uint8_t> pre(std::max<std::size_t>(nodes.size(), 1) * n_);
        std::vector<int32_t> dep(std::max<std::size_t>(nodes.size(), 1));
        for (std::size_t i = 0; i < nodes.size(); ++i) {
            dep[i] = nodes[i].depth();
            for (int d = 0; d < nodes[i].depth(); ++d) pre[i * n_ + d] = static_cast<uint8_t>(nodes[i].prefix[d]);
        }
        check(fbb_group_reset(g_, pre.data(), dep.data(), (int64_t)nodes.size(), ub, frozen ? 1 : 0));
    }
    // solve's start (search.hpp:131-153); ub < 0: the identity makespan
    void start_solve(int ub = -1) { check(fbb_group_start_solve(g_, ub)); }
    fbb_group_stats_t run(std::int64_t target, std::int64_t max_steps = INT64_MAX, int rounds_per_step = 4,
                          int balance_every = 1, std::int64_t budget = 0) {
        fbb_group_stats_t st;
        check(fbb_group_run(g_, target, max_steps, rounds_per_step, balance_every, budget, &st));
        return st;
    }
    // the group's best leaf (value, schedule when solving), if any
    std::optional<std::pair<int, flowbb::Permutation>> best() {
        int32_t v = 0;
        std::vector<int32_t> s(n_, -1);
        int f = fbb_group_best(g_, &v, s.data());
        if (f < 0) check(f);
        if (!f) return std::nullopt;
        return std::make_pair((int)v, flowbb::Permutation(s.begin(), s.end()));
    }
    int size() const { return fbb_group_size(g_); }

private:
    void check(int rc) {
        if (rc == FBB_OK) return;
        int member = -1;
        char buf[512] = {0};
        fbb_group_last_error(g_, &member, buf, sizeof buf);
        throw flowbb::BackendError{member < 0 ? 0 : member, buf};
    }
    fbb_group* g_ = nullptr;
    int n_;
};

}  // namespace flowbb_b200


#endif  // FLOWBB_B200_GPU_BACKEND_HPP
