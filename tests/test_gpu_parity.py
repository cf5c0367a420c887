"""GPU parity: the CUDA path (through the C-ABI) against the oracle and the
reference-generated golden fixtures.  Bit-exact everywhere (integer work)."""
import numpy as np
import pytest

import paper_1206_4973_b200 as fbb
from golden_util import CLASSES, instance_p, pool_children, pool_nodes, unpad

pytestmark = pytest.mark.gpu

SMALL_3x2 = np.array([3, 2, 1, 4, 2, 3], np.int32).reshape(3, 2)
SMALL_2x3 = np.array([2, 1, 3, 4, 2, 1], np.int32).reshape(2, 3)


def inst_of(p):
    return fbb.Instance(p.shape[0], p.shape[1], p)


# ---- K1: bound-only ------------------------------------------------------------------------

@pytest.mark.parametrize("name", CLASSES)
def test_k1_matches_golden_pools(instances, pools, name):
    inst = inst_of(instance_p(instances, name))
    prefixes, heads, lb = pool_nodes(pools, name)
    nodes = fbb.nodes_from_prefixes(inst, prefixes)
    assert np.array_equal(nodes.heads, heads)
    ctx = fbb.Context(inst)
    assert np.array_equal(ctx.bound(nodes), lb)


@pytest.mark.parametrize("name", CLASSES)
def test_k1_matches_golden_children(instances, pools, name):
    inst = inst_of(instance_p(instances, name))
    _, kids, _, kheads, klb = pool_children(pools, name)
    nodes = fbb.nodes_from_prefixes(inst, kids)
    assert np.array_equal(fbb.Context(inst).bound(nodes), klb)


def test_k1_small_instances_and_kats(pools):
    for s in range(12):
        p = pools[f"small{s}_p"]
        inst = inst_of(p)
        prefixes = unpad(pools[f"small{s}_nodes_prefix"], pools[f"small{s}_nodes_depth"])
        got = fbb.Context(inst).bound(fbb.nodes_from_prefixes(inst, prefixes))
        assert np.array_equal(got, pools[f"small{s}_nodes_lb"]), s
    c = fbb.Context(inst_of(SMALL_3x2))
    assert list(c.bound(fbb.nodes_from_prefixes(c.inst, [[], [1, 0, 2], [0], [1], [2]])))[:2] \
        == [10, 10]  # test_bound.cpp:77-98


def test_k1_random_pools_vs_oracle(oracle):
    rng = np.random.default_rng(2024)
    for (n, m, cnt) in [(20, 5, 5000), (20, 20, 4000), (50, 20, 600), (33, 7, 2000),
                        (64, 10, 500), (65, 3, 500), (130, 4, 200), (7, 1, 300), (1, 4, 3),
                        (2, 2, 10)]:
        p = rng.integers(1, 100, size=(n, m)).astype(np.int32)
        inst = inst_of(p)
        prefixes = [list(rng.permutation(n)[: rng.integers(0, n + 1)]) for _ in range(cnt)]
        nodes = fbb.nodes_from_prefixes(inst, prefixes)
        got = fbb.Context(inst).bound(nodes)
        ref = oracle.evaluate_batch(p, nodes.masks, nodes.heads, nodes.depth)
        assert np.array_equal(got, ref), (n, m)


def test_k1_empty_batch():
    inst = fbb.generate_instance(20, 5, 873654221)
    assert len(fbb.Context(inst).bound(fbb.NodeBatch.empty(inst, 0))) == 0


def test_backendset_bit_identical_across_k(oracle):  # test_backend.cpp:82-98, acceptance C4
    inst = fbb.generate_instance(20, 5, 873654221)
    rng = np.random.default_rng(5)
    nodes = fbb.nodes_from_prefixes(inst, [list(rng.permutation(20)[: rng.integers(0, 20)])
                                           for _ in range(4200)])
    seq = oracle.evaluate_batch(inst.p, nodes.masks, nodes.heads, nodes.depth)
    for size in (64, 1024, 4096):
        for k in (1, 2, 4, 8):
            got = fbb.BackendSet(k, fbb.BackendDescriptor(1, 1, 1 << 20)).evaluate(inst, nodes[:size])
            assert np.array_equal(got, seq[:size]), (size, k)


def test_failing_backend_poisons_round():  # test_backend.cpp:106-118
    class Failing:
        def __init__(self, fail):
            self.fail = fail

        def evaluate(self, inst, nodes):
            if self.fail:
                raise RuntimeError("simulated device fault")
            return fbb.Context(inst).bound(nodes)

    inst = inst_of(SMALL_3x2)
    nodes = fbb.nodes_from_prefixes(inst, [[0], [1], [2]])
    with pytest.raises(fbb.BackendError) as e:
        fbb.flowbb.evaluate_multi([Failing(False), Failing(True), Failing(False)], inst, nodes)
    assert e.value.backend == 1 and "simulated device fault" in str(e.value)


# ---- K2: fused expand + bound + prune ------------------------------------------------------

@pytest.mark.parametrize("name", CLASSES)
def test_k2_frozen_matches_golden_children(instances, pools, name):
    inst = inst_of(instance_p(instances, name))
    parents, kids, kid_parent, kheads, klb = pool_children(pools, name)
    order = sorted(range(len(parents)), key=lambda i: -len(parents[i]))  # pop order
    par = [parents[i] for i in order]
    kid_rows = [[k for k, pi in zip(range(len(kids)), kid_parent) if pi == i] for i in order]
    n = inst.jobs()
    ub = int(np.median(klb)) + 1
    ctx = fbb.Context(inst)
    surv, slb, best, pos, sched, counts = ctx.expand_bound_prune(
        fbb.nodes_from_prefixes(inst, par), ub, frozen=True)
    exp_pre, exp_lb, exp_heads, leaves, leaf_vals = [], [], [], 0, []
    for rows in kid_rows:
        for r in rows:
            if len(kids[r]) == n:
                leaves += 1
                leaf_vals.append(int(klb[r]))
            elif klb[r] < ub:
                exp_pre.append(kids[r])
                exp_lb.append(int(klb[r]))
                exp_heads.append(kheads[r])
    assert surv.prefixes() == exp_pre
    assert list(slb) == exp_lb
    if exp_heads:
        assert np.array_equal(surv.heads, np.array(exp_heads))
    assert list(surv.depth) == [len(x) for x in exp_pre]
    assert counts[2] == len(kids) and counts[5] == leaves
    assert counts[3] == len(exp_pre) and counts[4] == len(kids) - leaves - len(exp_pre)
    under = [v for v in leaf_vals if v < ub]
    assert best == (min(under) if under else None)
    # masks of the survivors are their prefixes' sets
    ref = fbb.nodes_from_prefixes(inst, exp_pre)
    assert np.array_equal(surv.masks, ref.masks)


def test_k2_solve_mode_prunes_with_batch_leaf_min(oracle):
    # pool = parents at depth n-2 (leaves) followed by shallower parents: internal
    # children must be pruned against min(ub, best leaf) as integrate does mid-batch
    rng = np.random.default_rng(11)
    for trial in range(6):
        n, m = 9, 4
        p = rng.integers(1, 30, size=(n, m)).astype(np.int32)
        inst = inst_of(p)
        deep = [list(rng.permutation(n)[: n - 2]) for _ in range(5)]
        shallow = [list(rng.permutation(n)[: d]) for d in (5, 4, 4, 2, 0)]
        parents = deep + shallow
        kids = []
        for pr in parents:
            kids += oracle.branch(p, pr)[0]
        kn = fbb.nodes_from_prefixes(inst, kids)
        klb = oracle.evaluate_batch(p, kn.masks, kn.heads, kn.depth)
        leaf_vals = [v for k, v in zip(kids, klb) if len(k) == n]
        ub = int(np.percentile(klb, 60))
        inc = min([ub] + leaf_vals)
        surv, slb, best, pos, sched, counts = fbb.Context(inst).expand_bound_prune(
            fbb.nodes_from_prefixes(inst, parents), ub, frozen=False)
        exp = [k for k, v in zip(kids, klb) if len(k) < n and v < inc]
        assert surv.prefixes() == exp, trial
        if min(leaf_vals) < ub:
            assert best == min(leaf_vals)
            first = next(i for i, (k, v) in enumerate(zip(kids, klb)) if len(k) == n and v == best)
            assert pos == first and sched == [int(x) for x in kids[first]]
            assert counts[6] == best
        else:
            assert best is None


@pytest.mark.parametrize("frozen", [False, True])
def test_k2_two_leaf_segments(oracle, frozen):
    # parents at depth n-1 AND at depth n-2 (two leaf segments ahead of the internal ones):
    # every leaf is evaluated, the batch minimum / first position / schedule come from
    # either segment, and internal children prune against it (integrate, search.hpp:84-107)
    rng = np.random.default_rng(17)
    for trial in range(12):
        n, m = (9, 4) if trial % 2 else (20, 20)
        p = rng.integers(1, 60, size=(n, m)).astype(np.int32)
        inst = inst_of(p)
        d1 = [list(rng.permutation(n)[: n - 1]) for _ in range(int(rng.integers(1, 6)))]
        d2 = [list(rng.permutation(n)[: n - 2]) for _ in range(int(rng.integers(1, 6)))]
        shallow = sorted([list(rng.permutation(n)[: rng.integers(0, n - 2)]) for _ in range(6)],
                         key=len, reverse=True)
        parents = d1 + d2 + shallow
        kids = []
        for pr in parents:
            kids += oracle.branch(p, pr)[0]
        kn = fbb.nodes_from_prefixes(inst, kids)
        klb = oracle.evaluate_batch(p, kn.masks, kn.heads, kn.depth)
        leaf_vals = [int(v) for k, v in zip(kids, klb) if len(k) == n]
        assert len(leaf_vals) == len(d1) + 2 * len(d2)
        # ub between the two segments' best leaves whenever possible
        ub = int(np.percentile(leaf_vals, 50 + 10 * (trial % 3))) + (trial % 2)
        inc = ub if frozen else min([ub] + leaf_vals)
        surv, slb, best, pos, sched, counts = fbb.Context(inst).expand_bound_prune(
            fbb.nodes_from_prefixes(inst, parents), ub, frozen=frozen)
        exp = [k for k, v in zip(kids, klb) if len(k) < n and v < inc]
        assert surv.prefixes() == exp, trial
        assert counts[5] == len(leaf_vals)
        under = [v for v in leaf_vals if v < ub]
        if under:
            assert best == min(under), trial
            first = next(i for i, (k, v) in enumerate(zip(kids, klb)) if len(k) == n and v == best)
            assert pos == first and sched == [int(x) for x in kids[first]], trial
        else:
            assert best is None, trial


def test_explorer_pushed_depth_n_minus_1_nodes(oracle):
    # pending nodes at depth n-1 (accepted by fbb_explorer_reset / push) are leaves' parents
    rng = np.random.default_rng(23)
    n, m = 9, 4
    p = rng.integers(1, 40, size=(n, m)).astype(np.int32)
    inst = inst_of(p)
    roots = [list(rng.permutation(n)[: d]) for d in (3, 7, 8, 8, 5, 7, 8)]
    ub = 10 ** 6
    full, gold = oracle.resolve(p, ub, roots, targets=[7], max_trace=4096)
    res = fbb.resolve_workload(inst, roots, ub, targets=[7])
    assert [tuple(r) for r in res.rounds] == [tuple(r) for r in gold]
    assert res.best == full["optimum"]


def test_k2_rejects_non_pop_order():
    inst = fbb.generate_instance(8, 3, 1234)
    ctx = fbb.Context(inst)
    with pytest.raises(ValueError):
        ctx.expand_bound_prune(fbb.nodes_from_prefixes(inst, [[0], [1, 2]]), 10_000, True)
    surv, *_ = ctx.expand_bound_prune(fbb.NodeBatch.empty(inst, 0), 10_000, True)
    assert len(surv) == 0


def test_k2_random_parents_vs_oracle(oracle):
    rng = np.random.default_rng(99)
    # covers the generic kernel (m not in {5,10,20}), v2 (n <= 64) and v3 (64 < n <= 256)
    for (n, m, cnt) in [(20, 20, 300), (20, 5, 800), (50, 20, 40), (40, 6, 200), (100, 5, 30),
                        (5, 3, 50), (3, 2, 4), (2, 3, 3), (1, 2, 1), (128, 3, 10), (129, 2, 10),
                        (65, 10, 30), (100, 20, 24), (128, 20, 8), (129, 10, 10), (200, 20, 8),
                        (200, 10, 10), (256, 5, 6), (256, 20, 3)]:
        p = rng.integers(1, 100, size=(n, m)).astype(np.int32)
        inst = inst_of(p)
        parents = sorted([list(rng.permutation(n)[: rng.integers(0, n)]) for _ in range(cnt)],
                         key=len, reverse=True)
        kids = []
        for pr in parents:
            kids += oracle.branch(p, pr)[0]
        kn = fbb.nodes_from_prefixes(inst, kids)
        klb = oracle.evaluate_batch(p, kn.masks, kn.heads, kn.depth)
        ub = int(np.percentile(klb, 50)) + 1
        surv, slb, *_ = fbb.Context(inst).expand_bound_prune(
            fbb.nodes_from_prefixes(inst, parents), ub, frozen=True)
        exp = [(k, v) for k, v in zip(kids, klb) if len(k) < n and v < ub]
        assert surv.prefixes() == [k for k, _ in exp], (n, m)
        assert list(slb) == [int(v) for _, v in exp], (n, m)


# ---- device-resident explorer ---------------------------------------------------------------

@pytest.mark.parametrize("loop", ["auto", "0"], ids=["loop_auto", "host_planned"])
@pytest.mark.parametrize("on_host", [False, True], ids=["pending_hbm", "pending_host"])
def test_explorer_resolve_traces_match_reference(instances, traces, on_host, loop, monkeypatch):
    """Multi-round calls run as device-planned graph batches by default; FBB_DEVICE_LOOP=0
    keeps every round host-planned.  Both reproduce the reference traces."""
    if loop == "0":
        monkeypatch.setenv("FBB_DEVICE_LOOP", "0")
    fbb.flowbb._ctx_cache.clear()  # contexts read the switch when created
    for tr in traces["resolve"]:
        inst = inst_of(instance_p(instances, tr["instance"]))
        res = fbb.resolve_workload(inst, tr["roots"], tr["ub"], targets=tr["targets"],
                                   budget=tr["budget"], pending_on_host=on_host)
        gold = [tuple(r) for r in tr["rounds"]]
        assert res.rounds == gold, (tr["instance"], tr["targets"][:2])
        assert res.nodes_bounded == tr["result"]["bounded"]
        assert (res.best if res.best is not None else -1) == tr["result"]["optimum"]


@pytest.mark.parametrize("loop", ["auto", "0"], ids=["loop_auto", "host_planned"])
@pytest.mark.parametrize("on_host", [False, True], ids=["pending_hbm", "pending_host"])
def test_explorer_solve_traces_match_reference(instances, traces, on_host, loop, monkeypatch):
    if loop == "0":
        monkeypatch.setenv("FBB_DEVICE_LOOP", "0")
    fbb.flowbb._ctx_cache.clear()
    for tr in traces["solve"]:
        inst = inst_of(instance_p(instances, tr["instance"]))
        ub = None if tr["initial_ub"] < 0 else tr["initial_ub"]
        sol = fbb.solve(inst, ub, targets=tr["targets"], budget=tr["budget"],
                        pending_on_host=on_host)
        gold = [tuple(r) for r in tr["rounds"]]
        assert sol.rounds == gold, tr["instance"]
        assert sol.optimum == tr["result"]["optimum"]
        assert sol.schedule == tr["schedule"]


@pytest.mark.parametrize("on_host", [False, True], ids=["pending_hbm", "pending_host"])
def test_explorer_full_solves_match_reference(traces, on_host):
    for case in traces["solve_full"]:
        p = np.asarray(case["p"], np.int32).reshape(case["n"], case["m"])
        sol = fbb.solve(inst_of(p), None, fixed_batch=case["batch"], pending_on_host=on_host)
        assert sol.optimum == case["optimum"]
        assert sol.schedule == case["schedule"]
        assert [sol.stats.branched, sol.stats.bounded, sol.stats.pruned] == case["stats"]
        assert sol.rounds == [tuple(r) for r in case["rounds"]]
        assert sol.exhausted


def test_resolution_equivalent_across_batches_and_tuner(traces):
    """test_bench.cpp:22-43,97-111 on the device explorer: a frozen-UB resolution to
    exhaustion explores the same node set whatever the pool size or the tuner does --
    same bounded count and the same best leaf."""
    for case in traces["solve_full"][:6]:
        p = np.asarray(case["p"], np.int32).reshape(case["n"], case["m"])
        inst = inst_of(p)
        ub = case["optimum"] + 1
        runs = [fbb.resolve_workload(inst, [[]], ub, batch=b) for b in (1, 8, 64, 512)]
        runs.append(fbb.resolve_workload(inst, [[]], ub, autotune=True, window=2, probes=2))
        for r in runs:
            assert r.exhausted and r.best == case["optimum"]
            assert r.nodes_bounded == runs[0].nodes_bounded


@pytest.mark.parametrize("on_host", [False, True])
def test_explorer_pending_matches_reference_drain(on_host):
    # after a budget stop, the device pending tree equals the reference's PendingTree,
    # node for node in PendingTree::drain order (pending.hpp:41-50)
    from oracle import Ref
    try:
        ref = Ref()
    except FileNotFoundError:
        pytest.skip("oracle/_ref not built on this host")
    for (n, m, seed, ub, tgt, budget) in [(20, 5, 873654221, 1279, 4096, 50_000),
                                         (20, 20, 479340445, 2297, 16384, 400_000),
                                         (50, 20, 1539989115, 3847, 8192, 100_000)]:
        inst = fbb.generate_instance(n, m, seed)
        fbb.resolve_workload(inst, [[]], ub, targets=[tgt], budget=budget, pending_on_host=on_host)
        ctx = fbb.flowbb.context_for(inst)
        got = ctx.explorer_pending()
        res, want = ref.resolve_drain(inst.p, ub, [[]], targets=[tgt], budget=budget)
        assert res["bounded"] == ctx.explorer_state()["bounded"]
        assert len(got) == len(want) == ctx.explorer_state()["pending"] > 0
        assert got == want, f"{n}x{m}: pending tree differs from the reference drain"


def test_solve_small_kats():
    sol = fbb.solve(inst_of(SMALL_3x2))
    assert sol.optimum == 10 and sol.found()
    sol = fbb.solve(inst_of(np.array([[4, 5, 6]], np.int32)))
    assert sol.optimum == 15 and sol.schedule == [0]
    sol = fbb.solve(inst_of(SMALL_3x2), initial_ub=9)
    assert not sol.found() and sol.optimum == 9
    sol = fbb.solve(inst_of(SMALL_3x2), initial_ub=11, fixed_batch=8)
    assert sol.optimum == 10 and sol.schedule == [1, 0, 2]


# ---- synthetic pools + K1 on device pointers (bounding-stress workload) -------------------------

@pytest.mark.parametrize("nm", [(20, 20), (200, 20), (100, 5)])
def test_synth_pool_and_k1_device_vs_oracle(oracle, nm):
    import torch

    from synth_ref import synth_prefix

    n, m = nm
    inst = fbb.generate_instance(n, m, 2013025619 if n == 200 else 479340445)
    ctx = fbb.Context(inst)
    cnt, seed, W = 700, 12345, (n + 63) // 64
    dm = torch.zeros(cnt * W, dtype=torch.int64, device="cuda")
    dh = torch.zeros(cnt * m, dtype=torch.int32, device="cuda")
    dd = torch.zeros(cnt, dtype=torch.int32, device="cuda")
    dp = torch.zeros(cnt * n, dtype=torch.uint8, device="cuda")
    dl = torch.zeros(cnt, dtype=torch.int32, device="cuda")
    ctx.synth_pool(seed, cnt, 0, n, dm.data_ptr(), dh.data_ptr(), dd.data_ptr(), dp.data_ptr())
    ctx.bound_device(dm.data_ptr(), dh.data_ptr(), dd.data_ptr(), cnt, dl.data_ptr())
    torch.cuda.synchronize()
    dep = dd.cpu().numpy()
    pre = dp.cpu().numpy().reshape(cnt, n)
    got = [list(map(int, pre[i, : dep[i]])) for i in range(cnt)]
    exp = [synth_prefix(n, seed, i, 0, n) for i in range(cnt)]
    assert got == exp
    ref = fbb.nodes_from_prefixes(inst, exp)
    assert np.array_equal(dh.cpu().numpy().reshape(cnt, m), ref.heads)
    assert np.array_equal(dm.cpu().numpy().view(np.uint64).reshape(cnt, W), ref.masks)
    lb = oracle.evaluate_batch(inst.p, ref.masks, ref.heads, ref.depth)
    assert np.array_equal(dl.cpu().numpy(), lb)


@pytest.mark.parametrize("nm", [(20, 20), (50, 10), (200, 20), (20, 7), (100, 5), (65, 2), (130, 3),
                                (256, 20), (33, 20), (128, 4), (9, 2)])
def test_k1_v1_v2_v3_agree(oracle, nm, monkeypatch):
    """The three K1 kernels (smem-table v1, packed-row v2, 16x2 SIMD v3) give the oracle's
    bounds; pools mix every depth (leaves included) and a ragged last tile."""
    n, m = nm
    rng = np.random.default_rng(n * 100 + m)
    inst = inst_of(rng.integers(1, 100, size=(n, m)).astype(np.int32))
    prefixes = [list(rng.permutation(n)[: rng.integers(0, n + 1)]) for _ in range(301)]
    nodes = fbb.nodes_from_prefixes(inst, prefixes)
    ref = oracle.evaluate_batch(inst.p, nodes.masks, nodes.heads, nodes.depth)
    got = {}
    for sel in ("v1", "v2", "v3"):
        monkeypatch.setenv("FBB_K1", sel)
        ctx = fbb.Context(inst)
        kern = ctx.kernels()
        got[sel] = ctx.bound(nodes)
        ctx.close()
        if sel == "v3" and m <= 20:
            assert "k1v3_kernel" in kern, kern
    for sel in got:
        assert np.array_equal(got[sel], ref), sel


def test_k2_generic_and_specialised_agree(monkeypatch):
    """The generic K2 and the register-row kernels (v2 n<=64, v3 n<=256) give identical
    survivors, bounds and counts on the same parents."""
    rng = np.random.default_rng(5)
    for n, m in [(20, 20), (50, 20), (100, 10)]:
        inst = inst_of(rng.integers(1, 100, size=(n, m)).astype(np.int32))
        parents = sorted([list(rng.permutation(n)[: rng.integers(0, n - 2)]) for _ in range(60)],
                         key=len, reverse=True)
        pb = fbb.nodes_from_prefixes(inst, parents)
        outs = []
        for sel in ("generic", "auto"):
            monkeypatch.setenv("FBB_K2", sel)
            ctx = fbb.Context(inst)
            surv, slb, best, pos, sched, counts = ctx.expand_bound_prune(pb, 10**6, frozen=True)
            k = int(np.median(slb)) if len(slb) else 0
            s2, l2, *_ = ctx.expand_bound_prune(pb, k, frozen=True)
            outs.append((surv.prefixes(), list(slb), counts, s2.prefixes(), list(l2)))
            ctx.close()
        assert outs[0] == outs[1], (n, m)


@pytest.mark.parametrize("nm_sel", [((20, 20), "auto"), ((30, 10), "auto"), ((50, 20), "auto"),
                                    ((100, 20), "auto"), ((70, 5), "auto"), ((20, 7), "auto"),
                                    ((20, 20), "generic")],
                         ids=lambda v: f"{v[0][0]}x{v[0][1]}-{v[1]}")
def test_host_tree_row_formats_match_hbm(nm_sel, monkeypatch):
    """The host-resident pending tree in its compact form (prefixes only: every K2 kernel
    folds heads and masks from the prefix when it stages a parent, and place_kernel moves
    only the prefix bytes up to the child depth) and in the full-row form both reproduce
    the HBM-resident explorer round for round, pending tree included."""
    (n, m), sel = nm_sel
    monkeypatch.setenv("FBB_K2", sel)
    rng = np.random.default_rng(n * 31 + m)
    inst = inst_of(rng.integers(1, 100, size=(n, m)).astype(np.int32))
    ub = fbb.makespan(inst, list(range(n))) - 1
    out = {}
    for mode in ("hbm", "host", "host_full"):
        monkeypatch.setenv("FBB_HOST_ROWS", "full" if mode == "host_full" else "compact")
        ctx = fbb.Context(inst)
        ctx.explorer_set_residency(mode != "hbm")
        ctx.explorer_reset(fbb.NodeBatch.root(inst), ub, frozen=True)
        rounds = ctx.explorer_run([64, 1024, 4096, 16384], 40, 400_000)
        out[mode] = (rounds, ctx.explorer_pending(), ctx.explorer_state()["bounded"])
        ctx.close()
    assert len(out["hbm"][0]) > 3
    assert out["host"] == out["hbm"] and out["host_full"] == out["hbm"]


@pytest.mark.parametrize("on_host,rows", [(False, "full"), (True, "full"), (True, "compact")],
                         ids=["pending_hbm", "pending_host_full", "pending_host_compact"])
def test_device_planned_loop_matches_reference(instances, traces, on_host, rows, monkeypatch):
    """The batched, device-planned explorer loop (FBB_DEVICE_LOOP=1, one CUDA graph per
    batch) reproduces the reference's per-round traces like the host-planned one, with the
    tree in HBM or in pinned host memory (full rows, or prefix-only rows)."""
    monkeypatch.setenv("FBB_DEVICE_LOOP", "1")
    monkeypatch.setenv("FBB_HOST_ROWS", rows)
    for tr in traces["resolve"][:4]:
        inst = inst_of(instance_p(instances, tr["instance"]))
        ctx = fbb.Context(inst)  # a fresh context picks up the environment
        ctx.explorer_set_residency(on_host)
        ctx.explorer_reset(fbb.nodes_from_prefixes(inst, tr["roots"]), tr["ub"], frozen=True)
        rounds = ctx.explorer_run(tr["targets"], 1 << 20, tr["budget"])
        assert rounds == [tuple(r) for r in tr["rounds"]], tr["instance"]
        ctx.close()
    for case in traces["solve_full"][:5]:
        p = np.asarray(case["p"], np.int32).reshape(case["n"], case["m"])
        ctx = fbb.Context(inst_of(p))
        ctx.explorer_set_residency(on_host)
        r0 = ctx.explorer_start_solve(None)
        rounds = ctx.explorer_run([case["batch"]], 1 << 20)
        st = ctx.explorer_state()
        assert [r0] + rounds == [tuple(r) for r in case["rounds"]]
        assert st["incumbent"] == case["optimum"] and st["schedule"] == case["schedule"]
        ctx.close()


@pytest.mark.parametrize("persist", ["1", "0"], ids=["persistent", "graph"])
def test_persistent_batch_matches_reference(instances, traces, persist, monkeypatch):
    """Single-wave batches on an HBM tree run as ONE cooperative launch of the persistent K2
    (plan, leaves, K2 with direct placement and close per round inside it, grid barriers
    between; FBB_PERSIST=0: the conditional-graph batch): resolve and solve traces, leaf
    rounds and schedules included, equal the reference's.  The launch count proves which
    path ran (persistent: one launch for a whole batch)."""
    monkeypatch.setenv("FBB_DEVICE_LOOP", "1")
    monkeypatch.setenv("FBB_PERSIST", persist)
    ran_persistent = False
    for tr in traces["resolve"]:
        inst = inst_of(instance_p(instances, tr["instance"]))
        ctx = fbb.Context(inst)
        if "batch=1" not in ctx.kernels() or max(tr["targets"]) > 16384:
            ctx.close()
            continue
        ctx.explorer_reset(fbb.nodes_from_prefixes(inst, tr["roots"]), tr["ub"], frozen=True)
        rounds, tim = ctx.explorer_run(tr["targets"], 1 << 20, tr["budget"], timing=True)
        assert rounds == [tuple(r) for r in tr["rounds"]], tr["instance"]
        if persist == "1" and len(tim) > 2:
            assert sum(t["launches"] for t in tim) < len(tim)  # not 5 kernels per round
            ran_persistent = True
        ctx.close()
    for case in traces["solve_full"]:
        p = np.asarray(case["p"], np.int32).reshape(case["n"], case["m"])
        ctx = fbb.Context(inst_of(p))
        r0 = ctx.explorer_start_solve(None)
        rounds = ctx.explorer_run([case["batch"]], 1 << 20)
        st = ctx.explorer_state()
        assert [r0] + rounds == [tuple(r) for r in case["rounds"]]
        assert st["incumbent"] == case["optimum"] and st["schedule"] == case["schedule"]
        ctx.close()
    assert ran_persistent or persist == "0"


# ---- >= 1 M-node traces at 50x20, 100x20, 200x20 (tests/golden/make_traces_large.py) ----------

def _large_traces():
    import json
    import os

    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "traces_large.json")
    with open(path) as f:
        return json.load(f)["resolve"]


@pytest.mark.parametrize("mode", ["hbm", "host", "device_loop"])
def test_explorer_large_traces_match_reference(instances, mode, monkeypatch):
    """Per-round counts over >= 1 M bounded nodes (fixed pools and a tuner-shaped doubling
    schedule) equal the reference explorer's at 50x20 (K2 v2 wide), 100x20 and 200x20
    (K2 v3): HBM tree, host-resident tree, and the graph-captured device-planned loop."""
    if mode == "device_loop":
        monkeypatch.setenv("FBB_DEVICE_LOOP", "1")
        monkeypatch.setenv("FBB_HOST_ROWS", "full")
    for tr in _large_traces():
        inst = inst_of(instance_p(instances, tr["instance"]))
        ctx = fbb.Context(inst)
        ctx.explorer_set_residency(mode == "host")
        ctx.explorer_reset(fbb.NodeBatch.root(inst), tr["ub"], frozen=True)
        rounds = ctx.explorer_run(tr["targets"], 1 << 20, tr["budget"])
        assert rounds == [tuple(r) for r in tr["rounds"]], (tr["instance"], tr["targets"][:2], mode)
        assert ctx.explorer_state()["bounded"] == tr["result"]["bounded"] >= 1_000_000
        ctx.close()


def test_tuner_schedule_replays_on_the_reference():
    """Config 3 parity (SURVEY 7 hard part 4): the adaptive tuner (autotune.hpp:35-156 with
    the B200 descriptor) picks each round's pool size from measured device time, so its
    schedule is not reproducible -- but once recorded, the reference explorer driven with
    the same per-round targets (oracle/_ref, the reference headers compiled in place) must
    produce identical per-round counts on Ta051 (50x20, frozen UB)."""
    import os

    from oracle import REF_SO, Ref

    if not os.path.exists(REF_SO):
        pytest.skip("oracle/_ref not built")
    inst = fbb.generate_instance(50, 20, 1539989115)
    ctx = fbb.Context(inst)
    ctx.explorer_reset(fbb.NodeBatch.root(inst), 3847, frozen=True)
    tuner = fbb.Tuner(ctx.descriptor(), 1, 2)
    rounds, total = [], 0
    while total < 600_000:
        r, t = ctx.explorer_run([tuner.target()], 1, timing=True)
        if not r:
            break
        tuner.observe(r[0][2], max(t[0]["round_ms"], 1e-6) / 1e3)
        rounds += r
        total += r[0][2]
    targets = [r[0] for r in rounds]
    assert len(set(targets)) >= 2  # the tuner moved the pool size
    ref = Ref()
    res, gold, _ = ref.resolve(inst.p, 3847, [[]], targets=targets, budget=total,
                               backends=ref.detect_units(), max_trace=1 << 12)
    assert rounds == [tuple(x) for x in gold]
    assert res["bounded"] == total
    ctx.close()


@pytest.mark.parametrize("device_loop", ["0", "1"])
def test_direct_placement_matches_staged(device_loop, monkeypatch):
    """Single-wave pools: K2 writes its survivors straight to the bucket rows after a
    grid-wide count (Pool::direct) instead of staging them for place_kernel.  Same rounds
    and the same pending tree as the staged path, at pool sizes on both sides of the
    one-wave limit, in solve mode (leaf rounds, mid-batch incumbent) and frozen mode."""
    monkeypatch.setenv("FBB_DEVICE_LOOP", device_loop)
    inst = fbb.generate_instance(20, 20, 479340445)
    out = {}
    for direct in ("0", "1"):
        monkeypatch.setenv("FBB_DIRECT", direct)
        ctx = fbb.Context(inst)
        res = []
        for targets in ([512], [4096], [16384, 40000, 4096], [100000]):
            ctx.explorer_reset(fbb.NodeBatch.root(inst), 2297, frozen=True)
            res.append((ctx.explorer_run(targets, 40), ctx.explorer_pending()))
        r0 = ctx.explorer_start_solve(None)
        res.append(([r0] + ctx.explorer_run([2048], 60), ctx.explorer_state()["schedule"]))
        out[direct] = res
        ctx.close()
    assert out["0"] == out["1"]


def test_kernel_variants_selected():
    """The specialised kernels are the ones that run on the benchmark instances (a failed
    kernel configuration would otherwise fall back to the generic kernels silently)."""
    want = {(20, 20, 479340445): ("k1v3_kernel", "k2_v2_kernel<20,20,2>"),
            (20, 5, 873654221): ("K1=", "k2_v2_kernel<20,5,3>"),
            (50, 20, 1539989115): ("k1v3_kernel", "k2_v2_kernel<64,20,2>"),
            (100, 20, 450926852): ("k1v3_kernel", "k2_v3_kernel<4,20>"),
            (200, 20, 2013025619): ("k1v3_kernel", "k2_v3_kernel<8,20>")}
    for (n, m, seed), (k1, k2) in want.items():
        ks = fbb.Context(fbb.generate_instance(n, m, seed)).kernels()
        assert k1 in ks and k2 in ks, ks
