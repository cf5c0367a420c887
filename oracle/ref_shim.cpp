// ref_shim.cpp -- C entry points over the UNMODIFIED reference flowbb headers.
//
// TEST INFRASTRUCTURE ONLY.  Compiled in place against
// /root/reference/proj/include (and proj/tests for helpers.hpp) by
// oracle/Makefile into oracle/_ref/libflowbb_ref.so.  No reference source is
// copied into this repository: this file only calls the reference's public
// API (Instance, Node, lower_bound, BackendSet, fill_buffer, integrate, solve,
// brute_force, testutil::random_*).  Used for
//   - generating the golden fixtures under tests/golden/ (make_golden.py),
//   - validating the C restatement in oracle/flowbb_oracle.c,
//   - bench.py --impl reference and the cpu_baseline leg (the reference CPU
//     explorer timed on the host cores).
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <optional>
#include <random>
#include <span>
#include <vector>

#include "flowbb/flowbb.hpp"
#include "helpers.hpp"
#include "flowbb_oracle.h"  // orc_round / orc_result record layouts only

using namespace flowbb;

namespace {

Instance make_instance(int n, int m, const int32_t* p) {
    return Instance(n, m, std::vector<int>(p, p + static_cast<std::size_t>(n) * m));
}

Node node_from_prefix(const Instance& inst, const int32_t* prefix, int depth) {
    Node node = Node::root(inst);
    for (int i = 0; i < depth; ++i) node = node.child(inst, prefix[i]);
    return node;
}

std::size_t target_at(const int64_t* targets, int ntargets, int64_t r) {
    if (ntargets <= 0) return 1;
    return static_cast<std::size_t>(targets[r < ntargets ? r : ntargets - 1]);
}

BackendDescriptor wide_descriptor() { return BackendDescriptor{1, 1, 1 << 30}; }

}  // namespace

extern "C" {

int ref_generate_instance(int n, int m, int32_t seed, int32_t* p_out) {
    try {
        Instance inst = generate_instance(n, m, seed);
        for (int j = 0; j < n; ++j)
            for (int k = 0; k < m; ++k) p_out[j * m + k] = inst.p(j, k);
        return 0;
    } catch (const std::exception&) {
        return -1;
    }
}

// tests/helpers.hpp:22-28 with std::mt19937(seed)
void ref_random_instance(uint32_t seed, int n, int m, int low, int high, int32_t* p_out) {
    std::mt19937 rng(seed);
    Instance inst = testutil::random_instance(rng, n, m, low, high);
    for (int j = 0; j < n; ++j)
        for (int k = 0; k < m; ++k) p_out[j * m + k] = inst.p(j, k);
}

// tests/helpers.hpp:47-55 repeated `count` times on one std::mt19937(seed)
void ref_random_nodes(int n, int m, const int32_t* p, uint32_t seed, int64_t count,
                      int32_t* prefix_out, int32_t* depth_out) {
    Instance inst = make_instance(n, m, p);
    std::mt19937 rng(seed);
    for (int64_t i = 0; i < count; ++i) {
        Node node = testutil::random_node(inst, rng);
        depth_out[i] = node.depth();
        for (int j = 0; j < n; ++j)
            prefix_out[i * n + j] = j < node.depth() ? node.prefix[j] : -1;
    }
}

// Node::child fold + BackendSet(k).evaluate (backend.hpp:142-158, bound.hpp:104-109)
int ref_evaluate(int n, int m, const int32_t* p, int64_t count, const int32_t* prefix,
                 const int32_t* depth, int backends, int32_t* lb_out, int32_t* heads_out) {
    try {
        Instance inst = make_instance(n, m, p);
        std::vector<Node> nodes;
        nodes.reserve(static_cast<std::size_t>(count));
        for (int64_t i = 0; i < count; ++i)
            nodes.push_back(node_from_prefix(inst, prefix + i * n, depth[i]));
        BackendSet set(backends, wide_descriptor());
        std::vector<int> lbs = set.evaluate(inst, nodes);
        for (int64_t i = 0; i < count; ++i) {
            lb_out[i] = lbs[static_cast<std::size_t>(i)];
            if (heads_out)
                for (int k = 0; k < m; ++k) heads_out[i * m + k] = nodes[i].heads[k];
        }
        return 0;
    } catch (const std::exception&) {
        return -1;
    }
}

// bound.hpp:61-90 components, for finer-grained fixtures
int32_t ref_lb_one_machine(int n, int m, const int32_t* p, const int32_t* prefix, int depth) {
    Instance inst = make_instance(n, m, p);
    return lb_one_machine(inst, node_from_prefix(inst, prefix, depth));
}
int32_t ref_lb_machine_pair(int n, int m, const int32_t* p, const int32_t* prefix, int depth,
                            int k, int l) {
    Instance inst = make_instance(n, m, p);
    return lb_machine_pair(inst, node_from_prefix(inst, prefix, depth), k, l);
}
int32_t ref_johnson(const int32_t* a, const int32_t* lag, const int32_t* b, int count,
                    int32_t ra, int32_t rb) {
    std::vector<LagJob> jobs;
    for (int i = 0; i < count; ++i) jobs.push_back({a[i], lag[i], b[i]});
    return johnson_two_machine(jobs, ra, rb);
}

// search.hpp:40-59
int ref_branch(int n, int m, const int32_t* p, const int32_t* prefix, int depth,
               int32_t* child_prefix, int32_t* child_depth, int32_t* child_heads) {
    try {
        Instance inst = make_instance(n, m, p);
        std::vector<Node> kids = branch(inst, node_from_prefix(inst, prefix, depth));
        for (std::size_t c = 0; c < kids.size(); ++c) {
            child_depth[c] = kids[c].depth();
            for (int j = 0; j < n; ++j)
                child_prefix[c * n + j] = j < kids[c].depth() ? kids[c].prefix[j] : -1;
            for (int k = 0; k < m; ++k) child_heads[c * m + k] = kids[c].heads[k];
        }
        return static_cast<int>(kids.size());
    } catch (const std::exception&) {
        return -1;
    }
}

// bench.hpp:63-114 resolve_workload's loop, call for call (fill_buffer,
// BackendSet::evaluate, the frozen prune), with a per-round target schedule
// and a bounded-node budget checked after each round.
// With drain_cap >= 0, the pending tree left by a budget stop is drained
// (PendingTree::drain, pending.hpp:41-50: shallowest bucket first, insertion order)
// into drain_prefix (n int32 per node) / drain_depth; *drain_count = its size.
static int resolve_impl(int n, int m, const int32_t* p, int32_t ub, int64_t nroots,
                        const int32_t* roots_prefix, const int32_t* roots_depth,
                        const int64_t* targets, int ntargets, int64_t budget, int backends,
                        orc_result* res, orc_round* trace, int64_t max_trace, double* seconds,
                        int64_t drain_cap, int32_t* drain_prefix, int32_t* drain_depth,
                        int64_t* drain_count) {
    try {
        Instance inst = make_instance(n, m, p);
        BackendSet set(backends, wide_descriptor());
        std::memset(res, 0, sizeof(*res));
        res->optimum = -1;
        PendingTree pending(inst.jobs());
        for (int64_t i = 0; i < nroots; ++i)
            pending.push(node_from_prefix(inst, roots_prefix + i * n, roots_depth[i]));
        std::optional<int> best;
        auto t0 = std::chrono::steady_clock::now();
        int64_t r = 0;
        while (!pending.empty()) {
            orc_round rec{};
            std::size_t target = target_at(targets, ntargets, r);
            rec.target = static_cast<int64_t>(target);
            std::int64_t branched = 0;
            std::vector<Node> batch = fill_buffer(inst, pending, target, &branched);
            std::vector<int> bounds = set.evaluate(inst, batch);
            rec.branched = branched;
            rec.bounded = static_cast<int64_t>(batch.size());
            for (std::size_t i = 0; i < batch.size(); ++i) {
                Node& node = batch[i];
                node.lb = bounds[i];
                if (node.depth() == inst.jobs()) {
                    ++rec.leaves;
                    if (node.lb < ub && (!best || node.lb < *best)) best = node.lb;
                } else if (node.lb < ub) {
                    ++rec.inserted;
                    pending.push(std::move(node));
                } else {
                    ++rec.pruned;
                }
            }
            res->branched += rec.branched;
            res->bounded += rec.bounded;
            res->pruned += rec.pruned;
            res->leaves += rec.leaves;
            rec.incumbent = best ? *best : ub;
            rec.pending = static_cast<int64_t>(pending.size());
            if (trace && r < max_trace) trace[r] = rec;
            ++r;
            if (budget > 0 && res->bounded >= budget) break;
        }
        if (seconds)
            *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        res->rounds = r;
        res->found = best.has_value();
        res->optimum = best ? *best : -1;
        res->pending = static_cast<int64_t>(pending.size());
        if (drain_cap >= 0) {
            std::vector<Node> left = pending.drain();
            *drain_count = static_cast<int64_t>(left.size());
            if (static_cast<int64_t>(left.size()) > drain_cap) return -2;
            for (std::size_t i = 0; i < left.size(); ++i) {
                drain_depth[i] = left[i].depth();
                for (int d = 0; d < left[i].depth(); ++d) drain_prefix[i * n + d] = left[i].prefix[d];
            }
        }
        return 0;
    } catch (const std::exception&) {
        return -1;
    }
}

int ref_resolve(int n, int m, const int32_t* p, int32_t ub, int64_t nroots,
                const int32_t* roots_prefix, const int32_t* roots_depth, const int64_t* targets,
                int ntargets, int64_t budget, int backends, orc_result* res, orc_round* trace,
                int64_t max_trace, double* seconds) {
    return resolve_impl(n, m, p, ub, nroots, roots_prefix, roots_depth, targets, ntargets, budget,
                        backends, res, trace, max_trace, seconds, -1, nullptr, nullptr, nullptr);
}

int ref_resolve_drain(int n, int m, const int32_t* p, int32_t ub, int64_t nroots,
                      const int32_t* roots_prefix, const int32_t* roots_depth,
                      const int64_t* targets, int ntargets, int64_t budget, int backends,
                      orc_result* res, int64_t drain_cap, int32_t* drain_prefix,
                      int32_t* drain_depth, int64_t* drain_count) {
    return resolve_impl(n, m, p, ub, nroots, roots_prefix, roots_depth, targets, ntargets, budget,
                        backends, res, nullptr, 0, nullptr, drain_cap, drain_prefix, drain_depth,
                        drain_count);
}

// search.hpp:124-174 solve()'s loop, call for call (BackendSet::evaluate,
// integrate, fill_buffer), with a target schedule and a budget.
int ref_solve_trace(int n, int m, const int32_t* p, int32_t initial_ub, const int64_t* targets,
                    int ntargets, int64_t budget, int backends, orc_result* res,
                    int32_t* schedule_out, orc_round* trace, int64_t max_trace) {
    try {
        Instance inst = make_instance(n, m, p);
        BackendSet set(backends, wide_descriptor());
        std::memset(res, 0, sizeof(*res));
        Incumbent incumbent{0, std::nullopt};
        if (initial_ub >= 0) {
            incumbent.value = initial_ub;
        } else {
            Permutation identity(inst.jobs());
            for (int j = 0; j < n; ++j) identity[j] = j;
            incumbent.value = makespan(inst, identity);
            incumbent.schedule = identity;
        }
        PendingTree pending(inst.jobs());
        std::vector<Node> batch;
        batch.push_back(Node::root(inst));
        int64_t r = 0, target = 0, branched_round = 0;
        while (!batch.empty()) {
            orc_round rec{};
            rec.target = target;
            rec.branched = branched_round;
            std::vector<int> bounds = set.evaluate(inst, batch);
            rec.bounded = static_cast<int64_t>(batch.size());
            res->bounded += rec.bounded;
            IntegrateCounts counts = integrate(inst, batch, bounds, pending, incumbent);
            rec.inserted = counts.inserted;
            rec.pruned = counts.pruned;
            rec.leaves = counts.leaves;
            res->pruned += counts.pruned;
            res->leaves += counts.leaves;
            rec.incumbent = incumbent.value;
            rec.pending = static_cast<int64_t>(pending.size());
            if (trace && r < max_trace) trace[r] = rec;
            ++r;
            if (pending.empty()) break;
            if (budget > 0 && res->bounded >= budget) break;
            target = static_cast<int64_t>(target_at(targets, ntargets, r - 1));
            std::int64_t branched = 0;
            batch = fill_buffer(inst, pending, static_cast<std::size_t>(target), &branched);
            res->branched += branched;
            branched_round = branched;
        }
        res->rounds = r;
        res->optimum = incumbent.value;
        res->found = incumbent.schedule.has_value();
        res->pending = static_cast<int64_t>(pending.size());
        if (schedule_out && incumbent.schedule)
            for (int j = 0; j < n; ++j) schedule_out[j] = (*incumbent.schedule)[j];
        return 0;
    } catch (const std::exception&) {
        return -1;
    }
}

// search.hpp:124-174 -- the unmodified solve() entry point.
int ref_solve(int n, int m, const int32_t* p, int32_t initial_ub, int fixed_batch, int backends,
              int32_t* optimum, int32_t* found, int32_t* schedule_out, int64_t* stats3) {
    try {
        Instance inst = make_instance(n, m, p);
        SolveConfig config;
        if (initial_ub >= 0) config.initial_ub = initial_ub;
        config.fixed_batch = fixed_batch;
        config.backends = backends;
        config.descriptor = wide_descriptor();
        Solution s = solve(inst, config);
        *optimum = s.optimum;
        *found = s.found();
        if (s.found() && schedule_out)
            for (int j = 0; j < n; ++j) schedule_out[j] = (*s.schedule)[j];
        stats3[0] = s.stats.branched;
        stats3[1] = s.stats.bounded;
        stats3[2] = s.stats.pruned;
        return 0;
    } catch (const std::exception&) {
        return -1;
    }
}

// search.hpp:176-196
int ref_brute_force(int n, int m, const int32_t* p, int32_t* optimum, int32_t* schedule_out) {
    try {
        Instance inst = make_instance(n, m, p);
        Solution s = brute_force(inst);
        *optimum = s.optimum;
        for (int j = 0; j < n; ++j) schedule_out[j] = (*s.schedule)[j];
        return 0;
    } catch (const std::exception&) {
        return -1;
    }
}

int ref_detect_units() { return detect_units(); }

// The bench.py reference arm: the resolve_workload loop (bench.hpp:88-109,
// reference fill_buffer + BackendSet(k).evaluate + frozen prune) from the root,
//   prefill: rounds until one reaches the pool target (max 64 rounds),
//   warm:    `warm` more rounds,
//   timed:   `steps` rounds, each timed whole (selection, bounding, prune).
// Per timed round the counts go to trace[0..steps) and the seconds to secs[].
int ref_bench_rounds(int n, int m, const int32_t* p, int32_t ub, int64_t target, int warm,
                     int steps, int backends, int64_t* prefill_rounds, orc_round* trace,
                     double* secs, double max_seconds, int* steps_done) {
    try {
        Instance inst = make_instance(n, m, p);
        BackendSet set(backends, wide_descriptor());
        PendingTree pending(inst.jobs());
        pending.push(Node::root(inst));
        std::optional<int> best;
        auto round = [&](orc_round* rec) -> bool {
            if (pending.empty()) return false;
            std::int64_t branched = 0;
            std::vector<Node> batch =
                fill_buffer(inst, pending, static_cast<std::size_t>(target), &branched);
            std::vector<int> bounds = set.evaluate(inst, batch);
            orc_round r{};
            r.target = target;
            r.branched = branched;
            r.bounded = static_cast<int64_t>(batch.size());
            for (std::size_t i = 0; i < batch.size(); ++i) {
                Node& node = batch[i];
                node.lb = bounds[i];
                if (node.depth() == inst.jobs()) {
                    ++r.leaves;
                    if (node.lb < ub && (!best || node.lb < *best)) best = node.lb;
                } else if (node.lb < ub) {
                    ++r.inserted;
                    pending.push(std::move(node));
                } else {
                    ++r.pruned;
                }
            }
            r.incumbent = best ? *best : ub;
            r.pending = static_cast<int64_t>(pending.size());
            if (rec) *rec = r;
            return true;
        };
        orc_round rec{};
        int64_t pre = 0;
        while (pre < 64 && round(&rec)) {
            ++pre;
            if (rec.bounded >= target) break;
        }
        *prefill_rounds = pre;
        for (int i = 0; i < warm; ++i) round(nullptr);
        double spent = 0.0;
        *steps_done = 0;
        for (int i = 0; i < steps && (i == 0 || max_seconds <= 0 || spent < max_seconds); ++i) {
            auto t0 = std::chrono::steady_clock::now();
            orc_round r{};
            bool ok = round(&r);
            secs[i] = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            trace[i] = r;
            if (!ok) secs[i] = 0.0;
            spent += secs[i];
            *steps_done = i + 1;
            if (!ok) break;
        }
        return 0;
    } catch (const std::exception&) {
        return -1;
    }
}

// save_workload(generate_workload(...)) of the reference (workload.hpp:62-131) as text;
// returns its length (or -2 when cap is too small).
int64_t ref_workload_text(int n, int m, const int32_t* p, int32_t ub, int64_t nodes, uint32_t seed,
                          char* out, int64_t cap) {
    try {
        Instance inst = make_instance(n, m, p);
        std::string text = save_workload(generate_workload(inst, ub, CaptureCutoff::by_nodes(nodes), seed));
        if ((int64_t)text.size() + 1 > cap) return -2;
        std::memcpy(out, text.c_str(), text.size() + 1);
        return (int64_t)text.size();
    } catch (const std::exception&) {
        return -1;
    }
}

// The reference Tuner (autotune.hpp) with its trace hook, driven by the synthetic
// unimodal throughput curve tp(x) = x / (1 + (x / peak)^2) (each observation bounds
// target() nodes in target()/tp seconds) until fixed; the trace lines
// "window batch decision" go to out (newline-separated).  Returns the line count.
int ref_tuner_trace(int grain, int units, int max_batch, int window, int probes, double peak,
                    char* out, int64_t cap) {
    try {
        Tuner tuner(BackendDescriptor{grain, units, max_batch}, window, probes);
        std::string text;
        int lines = 0;
        tuner.set_trace([&](int w, int batch, double, const std::string& decision) {
            text += std::to_string(w) + " " + std::to_string(batch) + " " + decision + "\n";
            ++lines;
        });
        for (int it = 0; it < 10000 && tuner.phase() != TunerPhase::fixed; ++it) {
            const double x = tuner.target();
            const double tp = x / (1.0 + (x / peak) * (x / peak));
            tuner.observe(tuner.target(), x / tp);
        }
        if ((int64_t)text.size() + 1 > cap) return -2;
        std::memcpy(out, text.c_str(), text.size() + 1);
        return lines;
    } catch (const std::exception&) {
        return -1;
    }
}

}  // extern "C"
