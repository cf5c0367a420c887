"""The N>1 path of bench.py on CPU: world_size-2 gloo.

Frozen-UB exploration is partition-invariant (bench.hpp:60-62: the explored node
set does not depend on batch size or backend count), which is what lets bench.py
shard the frontier across GPUs with no data-path collective.  Here each gloo rank
takes its split_slices share of a frontier, resolves it with the oracle, and the
all-reduced totals must equal one rank resolving the whole frontier; the best leaf
is reduced with MIN (the incumbent min-allreduce of solve mode)."""
import os
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _worker(rank, world, port, p, ub, frontier, q):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import Oracle
    import paper_1206_4973_b200 as fbb

    off, ln = fbb.split_slices(len(frontier), world)[rank]
    res, _ = Oracle().resolve(p, ub, frontier[off:off + ln], targets=[64])
    t = torch.tensor([res["bounded"], res["pruned"], res["leaves"]], dtype=torch.int64)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    best = torch.tensor([res["optimum"] if res["found"] else 2**31 - 1], dtype=torch.int64)
    dist.all_reduce(best, op=dist.ReduceOp.MIN)
    if rank == 0:
        q.put((t.tolist(), int(best.item())))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_frontier_partition_is_count_invariant(world, oracle):
    rng = np.random.default_rng(3)
    p = rng.integers(1, 40, size=(9, 4)).astype(np.int32)
    opt, _, _ = oracle.solve(p, -1, targets=[64])
    ub = opt["optimum"] + 6
    import paper_1206_4973_b200 as fbb

    full, _ = oracle.resolve(p, ub, [[]], targets=[64])
    # frontier: the root's children with lb < ub (the first round's survivors)
    kids, _ = oracle.branch(p, [])
    frontier = [k for k in kids if oracle.lower_bound(p, k) < ub]
    single, _ = oracle.resolve(p, ub, frontier, targets=[64])
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() % 1000)
    procs = [ctx.Process(target=_worker, args=(r, world, port, p, ub, frontier, q))
             for r in range(world)]
    for pr in procs:
        pr.start()
    tot, best = q.get(timeout=120)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    assert tot == [single["bounded"], single["pruned"], single["leaves"]]
    assert best == (single["optimum"] if single["found"] else 2**31 - 1)
    # and the frontier resolution + the root round equals the full resolve from the root
    assert single["bounded"] + len(kids) == full["bounded"]
    assert fbb.split_slices(len(frontier), world)[0][0] == 0
