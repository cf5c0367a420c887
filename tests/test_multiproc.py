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


# ---- the multi-GPU driver (paper_1206_4973_b200.parallel) over gloo ---------------------------

# torch's NCCL process group accepts only these element types (c10d NCCLUtils.hpp
# getNcclDataType: kChar, kByte, kBool, kInt, kLong, kHalf, kFloat, kDouble, kBFloat16 and
# the float8 types); gloo is laxer, so the CPU tests enforce NCCL's map themselves.
NCCL_DTYPES = {torch.int8, torch.uint8, torch.bool, torch.int32, torch.int64, torch.float16,
               torch.float32, torch.float64, torch.bfloat16}


def strict_nccl_dtypes():
    """Wraps the torch.distributed calls the multi-GPU driver uses so that a tensor NCCL
    would reject raises here too (the round-1 int16 rebalancing rows passed gloo and would
    have failed their first NCCL send)."""
    def wrap(fn):
        def checked(*a, **kw):
            for x in a:
                for t in (x if isinstance(x, (list, tuple)) else [x]):
                    if isinstance(t, torch.Tensor) and t.dtype not in NCCL_DTYPES:
                        raise TypeError(f"{fn.__name__}: dtype {t.dtype} is not supported by NCCL")
            return fn(*a, **kw)
        return checked
    saved = {}
    for name in ("send", "recv", "all_gather", "all_reduce", "broadcast"):
        saved[name] = getattr(dist, name)
        setattr(dist, name, wrap(saved[name]))
    return saved


def _parallel_worker(rank, world, port, p, ub, frozen, roots_by_rank, target, q, every=1):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    strict_nccl_dtypes()
    from model_port import OraclePort
    from oracle import Oracle
    from paper_1206_4973_b200.parallel import ParallelExplorer

    ex = ParallelExplorer(OraclePort(Oracle(), p, ub, frozen, roots_by_rank[rank]), p.shape[0],
                          balance_every=1, exchange_every=every)
    res = ex.run([target])
    q.put((rank, res.bounded, res.best, res.schedule, res.transfers, res.exhausted,
           sum(r[2] for r in res.rounds)))
    dist.destroy_process_group()


def _run_parallel(world, p, ub, frozen, roots_by_rank, target=16, every=1):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29600 + (os.getpid() % 1000) + 7 * every
    procs = [ctx.Process(target=_parallel_worker,
                         args=(r, world, port, p, ub, frozen, roots_by_rank, target, q, every))
             for r in range(world)]
    for pr in procs:
        pr.start()
    out = sorted(q.get(timeout=300) for _ in range(world))
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    return out


def test_plan_transfers_is_deterministic_and_conserving():
    from paper_1206_4973_b200.parallel import plan_transfers

    assert plan_transfers([100, 0], 10, 1000) == [(0, 1, 50)]
    assert plan_transfers([5, 5, 5], 10, 1000) == []            # nobody rich enough
    plan = plan_transfers([0, 400, 3, 90], 10, 64)
    assert plan == [(1, 0, 64), (3, 2, 43)]                      # one donation per donor
    assert plan_transfers([0, 400], 10, 64) == [(1, 0, 64)]     # capped


def test_strict_dtype_wrapper_rejects_int16():
    """The dtype guard itself: an int16 tensor (what round 1 sent) is refused."""
    calls = []
    orig = dist.send
    dist.send = lambda *a, **k: calls.append(a)
    saved = strict_nccl_dtypes()
    try:
        with pytest.raises(TypeError):
            dist.send(torch.zeros(3, dtype=torch.int16), 1)
        dist.send(torch.zeros(3, dtype=torch.int32), 1)
        assert len(calls) == 1
    finally:
        for name, fn in saved.items():
            setattr(dist, name, fn)
        dist.send = orig


@pytest.mark.parametrize("world,every", [(2, 1), (2, 3)])
def test_parallel_frozen_exploration_is_partition_invariant(world, every, oracle):
    """Frozen UB, all work on rank 0 at the start: rebalancing feeds rank 1, and the total
    bounded count over ranks equals the single-explorer resolve (bench.hpp:60-62)."""
    rng = np.random.default_rng(11)
    p = rng.integers(1, 30, size=(8, 4)).astype(np.int32)
    opt, _, _ = oracle.solve(p, -1, targets=[64])
    ub = opt["optimum"] + 8
    single, _ = oracle.resolve(p, ub, [[]], targets=[16])
    out = _run_parallel(world, p, ub, True, [[[]], []], every=every)
    assert all(o[1] == single["bounded"] for o in out)          # gathered total, every rank
    assert sum(o[6] for o in out) == single["bounded"]          # per-rank work adds up
    assert all(o[5] for o in out)                               # exhausted everywhere
    assert out[1][6] > 0 and out[0][4] > 0                      # rank 1 got work
    best = single["optimum"] if single["found"] else None
    assert all(o[2] == best for o in out)


@pytest.mark.parametrize("world", [2])
def test_parallel_solve_reaches_the_optimum_with_ub_exchange(world, oracle):
    """Solve mode: each rank prunes with the min-allreduced incumbent; the global best
    is the brute-force optimum and its schedule (from the finding rank) achieves it."""
    rng = np.random.default_rng(5)
    p = rng.integers(1, 30, size=(7, 3)).astype(np.int32)
    opt, sched, _ = oracle.solve(p, -1, targets=[64])
    ident = oracle.makespan(p, list(range(7)))
    # the root's children split across the ranks
    kids, _ = oracle.branch(p, [])
    kids = [list(map(int, k)) for k in kids]
    out = _run_parallel(world, p, ident + 1, False, [kids[0::2], kids[1::2]])
    vals = {o[2] for o in out}
    assert vals == {opt["optimum"]}
    s = out[0][3]
    assert s is not None and oracle.makespan(p, s) == opt["optimum"]


def test_library_and_python_transfer_plans_agree():
    """The in-library group (csrc/group.cpp) and the multi-process driver (parallel.py)
    compute the same deterministic rebalancing plan from the same pending sizes."""
    import ctypes as C

    import paper_1206_4973_b200 as fbb
    from paper_1206_4973_b200.parallel import plan_transfers

    L = fbb.load_library()
    rng = np.random.default_rng(17)
    for trial in range(400):
        G = int(rng.integers(1, 9))
        pend = rng.integers(0, 3, size=G) * rng.integers(0, 5000, size=G)
        low, cap = int(rng.integers(1, 600)), int(rng.integers(1, 2000))
        out = np.zeros(3 * G, np.int64)
        cnt = C.c_int(0)
        assert L.fbb_plan_transfers(np.ascontiguousarray(pend, np.int64), G, low, cap, out,
                                    C.byref(cnt)) == 0
        lib = [tuple(int(x) for x in out[3 * i:3 * i + 3]) for i in range(cnt.value)]
        assert lib == plan_transfers([int(x) for x in pend], low, cap), (pend, low, cap)
