"""The multi-GPU driver over DEVICE explorers (parallel.DevicePort -> fbb_explorer_run /
take / push / set_incumbent / best), world 2.

The box has one GPU, so both ranks share cuda:0 and the collectives run over gloo
(the transfers still go through torch tensors of the dtypes NCCL accepts -- the
strict wrapper of test_multiproc enforces NCCL's type map).  Frozen exhaustion is
partition-invariant (bench.hpp:60-62): the ranks' bounded/pruned/leaves totals must
equal one device explorer's and the C oracle's resolve from the root; in solve mode
(search.hpp:124-174 with the paper's UB exchange) the global best
must be the oracle's optimum and its schedule must achieve it."""
import os
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def _worker(rank, world, port, p, ub, frozen, roots_by_rank, target, every, q):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from test_multiproc import strict_nccl_dtypes

    strict_nccl_dtypes()
    import paper_1206_4973_b200 as fbb
    from paper_1206_4973_b200.parallel import DevicePort, ParallelExplorer

    inst = fbb.Instance(p.shape[0], p.shape[1], p)
    ctx = fbb.Context(inst, 0)
    roots = roots_by_rank[rank]
    ctx.explorer_reset(fbb.nodes_from_prefixes(inst, roots) if roots else fbb.NodeBatch.empty(inst),
                       ub, frozen=frozen)
    px = ParallelExplorer(DevicePort(ctx, frozen), p.shape[0], balance_every=1,
                          exchange_every=every)
    res = px.run([target])
    st = ctx.explorer_state()
    q.put((rank, res.bounded, res.best, res.schedule, res.transfers, res.exhausted,
           sum(r[2] for r in res.rounds), st["pruned"], st["leaves"], st["bounded"]))
    ctx.close()
    dist.destroy_process_group()


def _run(world, p, ub, frozen, roots_by_rank, target, every):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29700 + (os.getpid() % 500) + 3 * every + (0 if frozen else 1)
    procs = [ctx.Process(target=_worker,
                         args=(r, world, port, p, ub, frozen, roots_by_rank, target, every, q))
             for r in range(world)]
    for pr in procs:
        pr.start()
    out = sorted(q.get(timeout=600) for _ in range(world))
    for pr in procs:
        pr.join(timeout=120)
        assert pr.exitcode == 0
    return out


@pytest.mark.parametrize("every", [1, 4])
def test_device_ranks_frozen_exhaustion_matches_single_explorer(every, oracle):
    """All work starts on rank 0; take/push feed rank 1; the totals over both ranks equal
    the oracle's resolve from the root and one device explorer's exhaustion."""
    import paper_1206_4973_b200 as fbb

    rng = np.random.default_rng(21)
    p = rng.integers(1, 60, size=(11, 6)).astype(np.int32)
    opt, _, _ = oracle.solve(p, -1, targets=[256])
    ub = opt["optimum"] + 25
    ref, _ = oracle.resolve(p, ub, [[]], targets=[64])
    inst = fbb.Instance(11, 6, p)
    one = fbb.resolve_workload(inst, [[]], ub, targets=[64])
    assert one.nodes_bounded == ref["bounded"]
    out = _run(2, p, ub, True, [[[]], []], 64, every)
    assert all(o[1] == ref["bounded"] for o in out)            # gathered total on every rank
    assert sum(o[6] for o in out) == ref["bounded"]            # per-rank rounds add up
    assert sum(o[9] for o in out) == ref["bounded"]            # device counters agree
    assert sum(o[7] for o in out) == ref["pruned"]
    assert sum(o[8] for o in out) == ref["leaves"]
    assert all(o[5] for o in out)                              # exhausted everywhere
    assert out[1][6] > 0 and out[0][4] > 0                     # rank 1 was fed by rank 0
    best = ref["optimum"] if ref["found"] else None
    assert all(o[2] == best for o in out)


def test_device_ranks_solve_reaches_the_oracle_optimum(oracle):
    """Solve mode from the identity makespan + 1: the UB min-allreduce lowers the other
    rank's pruning bound (fbb_explorer_set_incumbent); the global best equals the oracle's
    optimum and the broadcast schedule achieves it."""
    rng = np.random.default_rng(8)
    p = rng.integers(1, 60, size=(10, 5)).astype(np.int32)
    opt, _, _ = oracle.solve(p, -1, targets=[256])
    ident = oracle.makespan(p, list(range(10)))
    kids = [list(map(int, k)) for k in oracle.branch(p, [])[0]]
    out = _run(2, p, ident + 1, False, [kids[0::2], kids[1::2]], 32, 2)
    assert {o[2] for o in out} == {opt["optimum"]}
    s = out[0][3]
    assert s is not None and sorted(s) == list(range(10))
    assert oracle.makespan(p, s) == opt["optimum"]


@pytest.mark.timeout(600)
def test_group_members_sharing_a_gpu_with_single_wave_pools():
    """Two group members on one GPU run K2 concurrently; with ~200-chunk pools each round is
    single-wave (direct placement: its CTAs wait for each other), but the two grids together
    exceed the device.  The cooperative launch gang-schedules each grid, so neither can hold
    SMs while waiting for its own unscheduled CTAs.  Totals to a node budget's exhaustion
    equal one context's (frozen exploration is partition-invariant)."""
    import paper_1206_4973_b200 as fbb

    inst = fbb.generate_instance(20, 20, 479340445)
    ub = 2230  # below the optimum 2297: a tree the GPU exhausts in seconds
    one = fbb.Context(inst)
    one.explorer_reset(fbb.NodeBatch.root(inst), ub, frozen=True)
    one.explorer_run([30000], 1 << 20)
    st1 = one.explorer_state()
    one.close()
    assert st1["pending"] == 0
    grp = fbb.DeviceGroup(inst, [0, 0])
    grp.reset(fbb.NodeBatch.root(inst), ub, frozen=True)
    gs = grp.run(30000, rounds_per_step=2, balance_every=1)
    assert gs["pending"] == 0 and gs["bounded"] == st1["bounded"]
    assert gs["pruned"] == st1["pruned"] and gs["leaves"] == st1["leaves"]
    grp.close()
