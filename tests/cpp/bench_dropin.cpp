// bench_dropin.cpp -- the end-to-end speed a REFERENCE user sees: the reference's own
// explorer loop and data structures (flowbb::PendingTree of heap Nodes, fill_buffer,
// integrate / frozen prune) driving the GPU through the two drop-in entry points of
// include/flowbb_b200/gpu_backend.hpp:
//
//   gpu_round       one fused round per call (fbb_expand_bound_prune, K2) on the
//                   reference's PendingTree: pack the popped Nodes, H2D, K2, D2H of the
//                   survivors, unpack them into Nodes and push (search.hpp:64-107 shape);
//   GpuBackendSet   the reference's resolve loop (bench.hpp:88-106) with BackendSet
//                   replaced by GpuBackendSet(1): fill_buffer on the host, evaluate =
//                   fbb_bound (K1) over the packed pool, frozen prune + push on the host.
//
// Workload: Ta021 frozen at UB 2297 from the root, prefill until a round reaches the
// target, then `steps` timed rounds at that target; wall clock of the rounds (host work
// and transfers included).  Prints one JSON object.  Built by oracle/Makefile against the
// unmodified reference headers (target `dropin`), run by bench.py when present.
#include <chrono>
#include <cstdio>
#include <cstdlib>

#include "flowbb/flowbb.hpp"
#include "flowbb_b200/gpu_backend.hpp"

using namespace flowbb;
using Clock = std::chrono::steady_clock;

int main(int argc, char** argv) {
    const std::size_t target = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 262144;
    const int steps = argc > 2 ? std::atoi(argv[2]) : 20;
    const int ub = 2297;
    Instance inst = generate_instance(20, 20, 479340445);
    flowbb_b200::GpuBackend gpu;

    // ---- gpu_round on the reference PendingTree
    PendingTree pending(inst.jobs());
    pending.push(Node::root(inst));
    Incumbent inc{ub, std::nullopt};
    std::optional<int> best;
    for (int i = 0; i < 64 && !pending.empty(); ++i) {  // prefill (+ warm-up)
        auto rc = flowbb_b200::gpu_round(gpu, inst, pending, inc, target, true, &best);
        if (rc.bounded >= (std::int64_t)target && i >= 3) break;
    }
    std::int64_t r_bounded = 0;
    int r_rounds = 0;
    auto t0 = Clock::now();
    for (; r_rounds < steps && !pending.empty(); ++r_rounds)
        r_bounded += flowbb_b200::gpu_round(gpu, inst, pending, inc, target, true, &best).bounded;
    const double r_secs = std::chrono::duration<double>(Clock::now() - t0).count();

    // ---- the reference resolve loop with GpuBackendSet as the backend set
    flowbb_b200::GpuBackendSet set(1);
    PendingTree tree(inst.jobs());
    tree.push(Node::root(inst));
    auto round = [&](std::int64_t& bounded) {
        std::vector<Node> batch = fill_buffer(inst, tree, target);  // search.hpp:64-73
        std::vector<int> bounds = set.evaluate(inst, batch);
        for (std::size_t i = 0; i < batch.size(); ++i) {  // bench.hpp:96-106
            bounded += 1;
            if (batch[i].depth() == inst.jobs()) continue;
            if (bounds[i] < ub) {
                batch[i].lb = bounds[i];
                tree.push(std::move(batch[i]));
            }
        }
        return batch.size();
    };
    std::int64_t dummy = 0;
    for (int i = 0; i < 64 && !tree.empty(); ++i)
        if (round(dummy) >= target && i >= 3) break;
    std::int64_t s_bounded = 0;
    int s_rounds = 0;
    t0 = Clock::now();
    for (; s_rounds < steps && !tree.empty(); ++s_rounds) round(s_bounded);
    const double s_secs = std::chrono::duration<double>(Clock::now() - t0).count();

    std::printf("{\"target\": %zu, \"gpu_round\": {\"value\": %.1f, \"rounds\": %d, \"bounded\": %lld, "
                "\"seconds\": %.4f}, \"gpu_backend_set\": {\"value\": %.1f, \"rounds\": %d, "
                "\"bounded\": %lld, \"seconds\": %.4f}}\n",
                target, r_bounded / r_secs, r_rounds, (long long)r_bounded, r_secs, s_bounded / s_secs,
                s_rounds, (long long)s_bounded, s_secs);
    return 0;
}
