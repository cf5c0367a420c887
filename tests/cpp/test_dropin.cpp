// test_dropin.cpp -- the reference's own API driven by the GPU drop-in.
//
// Built against the UNMODIFIED reference headers (-I proj/include -I proj/tests)
// and libflowbb_b200.so by oracle/Makefile (target `dropin`, output
// oracle/_ref/dropin_test); run by tests/test_dropin.py on the GPU box.
// Mirrors the reference tests that exercise a Backend:
//   test_backend.cpp:82-98   evaluate_multi<Backend> bit-identical for k in {1,2,4,8}
//   acceptance.cpp:85-130    ta001 frontier >= 4200 nodes, batches {64,1024,4096}
//   test_search.cpp:132-174  solve loop == brute force / k-invariance (via gpu_round)
//   bench.hpp:63-114         resolve loop counts identical (via gpu_round, frozen)
#include <cstdio>
#include <random>

#include "flowbb/flowbb.hpp"
#include "flowbb_b200/gpu_backend.hpp"
#include "helpers.hpp"

using namespace flowbb;

static int failures = 0;
#define CHECK(cond, what)                                              \
    do {                                                               \
        if (!(cond)) {                                                 \
            ++failures;                                                \
            std::printf("FAIL %s (%s:%d)\n", what, __FILE__, __LINE__); \
        }                                                              \
    } while (0)

int main() {
    // 1. evaluate_multi<GpuBackend> == evaluate_batch on the ta001 frontier (acceptance C4)
    {
        Instance inst = generate_instance(20, 5, 873654221);
        PendingTree pending(inst.jobs());
        pending.push(Node::root(inst));
        std::vector<Node> batch = fill_buffer(inst, pending, 4200);
        while (batch.size() < 4200) {
            for (Node& node : batch) pending.push(std::move(node));
            batch = fill_buffer(inst, pending, 4200);
        }
        for (int size : {64, 1024, 4096}) {
            std::span<const Node> view(batch.data(), static_cast<std::size_t>(size));
            std::vector<int> sequential = evaluate_batch(inst, view);
            for (int k : {1, 2, 4, 8}) {
                flowbb_b200::GpuBackendSet set(k);
                CHECK(set.evaluate(inst, view) == sequential, "evaluate_multi<GpuBackend>");
            }
        }
        std::printf("ok evaluate_multi<GpuBackend> ta001 frontier k in {1,2,4,8}\n");
    }
    // 2. random nodes incl. leaves on random instances (helpers.hpp:22-55)
    {
        std::mt19937 rng(67);
        flowbb_b200::GpuBackend gpu;
        for (int trial = 0; trial < 40; ++trial) {
            Instance inst = testutil::random_instance(rng, 3 + trial % 30, 1 + trial % 12);
            std::vector<Node> nodes;
            for (int i = 0; i < 200; ++i) nodes.push_back(testutil::random_node(inst, rng));
            Node full = Node::root(inst);
            for (int j = 0; j < inst.jobs(); ++j) full = full.child(inst, j);
            nodes.push_back(full);
            CHECK(gpu.evaluate(inst, nodes) == evaluate_batch(inst, nodes), "random nodes");
        }
        std::printf("ok GpuBackend random nodes\n");
    }
    // 3. solve loop with gpu_round == reference solve() (counts, optimum, schedule)
    {
        std::mt19937 rng(43);
        flowbb_b200::GpuBackend gpu;
        for (int trial = 0; trial < 15; ++trial) {
            Instance inst = testutil::random_instance(rng, 5 + trial % 4, 2 + trial % 4);
            SolveConfig config;
            config.fixed_batch = 8;
            config.descriptor = BackendDescriptor{1, 1, 1 << 20};
            Solution ref = solve(inst, config);
            // search.hpp:124-174 with the fused GPU round
            Incumbent inc{0, std::nullopt};
            Permutation id(inst.jobs());
            for (int j = 0; j < inst.jobs(); ++j) id[j] = j;
            inc.value = makespan(inst, id);
            inc.schedule = id;
            PendingTree pending(inst.jobs());
            std::vector<Node> root{Node::root(inst)};
            std::vector<int> rb = gpu.evaluate(inst, root);
            std::int64_t bounded = 1, branched = 0, pruned = 0;
            integrate(inst, root, rb, pending, inc);
            if (rb[0] >= inc.value) pruned = 1;
            while (!pending.empty()) {
                auto rc = flowbb_b200::gpu_round(gpu, inst, pending, inc, 8, false);
                bounded += rc.bounded;
                branched += rc.branched;
                pruned += rc.pruned;
            }
            CHECK(inc.value == ref.optimum, "solve optimum");
            CHECK(inc.schedule == ref.schedule, "solve schedule");
            CHECK(bounded == ref.stats.bounded && branched == ref.stats.branched &&
                      pruned == ref.stats.pruned,
                  "solve counts");
            CHECK(inc.value == brute_force(inst).optimum, "brute force");
        }
        std::printf("ok gpu_round solve == reference solve on 15 instances\n");
    }
    // 4. frozen resolve of Ta021 from the optimal UB: identical per-round counts
    {
        Instance inst = generate_instance(20, 20, 479340445);
        flowbb_b200::GpuBackend gpu;
        BackendSet cpu(8, BackendDescriptor{1, 1, 1 << 30});
        PendingTree a(inst.jobs()), b(inst.jobs());
        a.push(Node::root(inst));
        b.push(Node::root(inst));
        Incumbent inc{2297, std::nullopt};
        std::optional<int> best;
        for (int round = 0; round < 12 && !a.empty(); ++round) {
            std::vector<Node> batch = fill_buffer(inst, a, 16384);
            std::vector<int> bounds = cpu.evaluate(inst, batch);
            std::int64_t ins = 0;
            for (std::size_t i = 0; i < batch.size(); ++i)
                if (batch[i].depth() < inst.jobs() && bounds[i] < 2297) {
                    batch[i].lb = bounds[i];
                    a.push(std::move(batch[i]));
                    ++ins;
                }
            auto rc = flowbb_b200::gpu_round(gpu, inst, b, inc, 16384, true, &best);
            CHECK(rc.bounded == static_cast<std::int64_t>(batch.size()), "resolve bounded");
            CHECK(rc.inserted == ins, "resolve inserted");
            CHECK(a.size() == b.size(), "resolve pending");
        }
        std::vector<Node> da = a.drain(), db = b.drain();
        bool same = da.size() == db.size();
        for (std::size_t i = 0; same && i < da.size(); ++i)
            same = da[i].prefix == db[i].prefix && da[i].heads == db[i].heads &&
                   da[i].scheduled == db[i].scheduled;
        CHECK(same, "pending trees identical after 12 rounds");
        std::printf("ok gpu_round frozen resolve Ta021 == reference (12 rounds, pending identical)\n");
    }
    // 5. generate_workload on the GPU == the reference's capture, byte for byte (workload.hpp)
    {
        flowbb_b200::GpuBackend gpu;
        Instance ta021 = generate_instance(20, 20, 479340445);
        for (std::int64_t budget : {0, 7, 500, 4000}) {
            auto cut = CaptureCutoff::by_nodes(budget);
            std::string ref = save_workload(generate_workload(ta021, 2297, cut, 42));
            std::string got = save_workload(flowbb_b200::generate_workload(gpu, ta021, 2297, cut, 42));
            CHECK(ref == got, "generate_workload Ta021");
        }
        std::mt19937 rng(5);
        for (int trial = 0; trial < 6; ++trial) {
            Instance inst = testutil::random_instance(rng, 8 + trial, 3 + trial % 4);
            int ub = solve(inst, [] { SolveConfig c; c.fixed_batch = 64; c.descriptor = BackendDescriptor{1, 1, 1 << 20}; return c; }()).optimum + 3;
            auto cut = CaptureCutoff::by_nodes(40 + 30 * trial);
            std::string ref = save_workload(generate_workload(inst, ub, cut, 1000u + trial));
            std::string got = save_workload(flowbb_b200::generate_workload(gpu, inst, ub, cut, 1000u + trial));
            CHECK(ref == got, "generate_workload random");
            // 6. run_experiment: sequential CPU vs GPU resolutions agree (bench.hpp:119-145)
            WorkloadSnapshot snap = load_workload(got);
            std::vector<BenchConfig> cfgs(3);
            cfgs[0].batch = 1;
            cfgs[1].batch = 64;
            cfgs[2].autotune = true;
            cfgs[2].descriptor = BackendDescriptor{8, 2, 4096};
            cfgs[2].window = 2;
            try {
                Report rep = flowbb_b200::run_experiment(gpu, snap, cfgs);
                CHECK(rep.rows.size() == 3, "run_experiment rows");
                BenchConfig c64;
                c64.batch = 64;
                c64.backends = 4;
                ResolutionResult cpu = resolve_workload(snap, c64);
                CHECK(rep.rows[1].nodes_bounded == cpu.nodes_bounded, "resolve nodes_bounded");
            } catch (const ResolutionMismatch&) {
                CHECK(false, "run_experiment ResolutionMismatch");
            }
        }
        std::printf("ok generate_workload byte-identical; run_experiment GPU == sequential CPU\n");
    }
    // 7. GpuGroupExplorer (fbb_group_*): frozen exhaustion over 2 and 3 members (one GPU,
    //    repeated device ids) == the reference resolve_workload; solve == reference optimum
    {
        std::mt19937 rng(91);
        for (int trial = 0; trial < 4; ++trial) {
            Instance inst = testutil::random_instance(rng, 9 + trial, 4 + trial % 3);
            SolveConfig sc;
            sc.fixed_batch = 64;
            sc.descriptor = BackendDescriptor{1, 1, 1 << 20};
            Solution ref = solve(inst, sc);
            const int ub = ref.optimum + 12;
            WorkloadSnapshot snap{inst, {Node::root(inst)}, ub, 0u, CaptureCutoff::by_nodes(0)};
            BenchConfig bc;
            bc.batch = 32;
            ResolutionResult cpu = resolve_workload(snap, bc);
            for (int G : {2, 3}) {
                flowbb_b200::GpuGroupExplorer grp(inst, std::vector<int>(G, 0));
                grp.reset(snap.nodes, ub, true);
                fbb_group_stats_t st = grp.run(32, INT64_MAX, 2, 1);
                CHECK(st.pending == 0, "group exhausted");
                CHECK(st.bounded == cpu.nodes_bounded, "group frozen bounded == reference");
                auto b = grp.best();
                CHECK(b.has_value() == cpu.best.has_value() && (!b || b->first == *cpu.best),
                      "group frozen best leaf == reference");
                flowbb_b200::GpuGroupExplorer sg(inst, std::vector<int>(G, 0));
                sg.start_solve(-1);
                fbb_group_stats_t ss = sg.run(16, INT64_MAX, 2, 1);
                auto sb = sg.best();
                CHECK(ss.pending == 0 && sb && sb->first == ref.optimum, "group solve optimum");
                CHECK(sb && makespan(inst, sb->second) == ref.optimum, "group solve schedule");
            }
        }
        std::printf("ok GpuGroupExplorer: frozen counts == reference resolve, solve optimum (G in {2,3})\n");
    }
    std::printf(failures ? "FAILED %d\n" : "ALL PASS\n", failures);
    return failures ? 1 : 0;
}
