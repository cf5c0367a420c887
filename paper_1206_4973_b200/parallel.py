"""Multi-GPU exploration: one process per GPU over torch.distributed.

The paper splits each pool across the GPUs of one host and merges the results
(PAPER.md:290-308); the reference models that as `split_slices` -> k concurrent
backends -> `merge_slices` (backend.hpp:73-158).  On an NVSwitch box the cheaper
equivalent is to split the *pending tree*: every rank owns a device-resident
explorer over its own subtrees (frozen exploration is partition-invariant,
bench.hpp:60-62: the explored node set does not depend on who explores which
subtree), and per round the ranks exchange only

  * the incumbent: min-allreduce of one int per rank (solve mode; a leaf found on
    one GPU prunes on all of them from the next round on), and
  * the pending sizes, from which every rank computes the same rebalancing plan:
    a starving rank receives the shallowest pending nodes (the roots of the
    largest unexplored subtrees) of the richest rank, as (depth, prefix) rows.

Both ride on ONE all_gather of a [incumbent, pending, bounded] triple per rank per
exchange step of `exchange_every` rounds (NCCL over NVLink on GPUs, gloo in the
CPU tests); rebalancing adds a send/recv pair per transfer every `balance_every`
steps.  Every tensor that crosses a collective is int32 or int64: torch's NCCL
backend has no 16-bit integer type.  The explorer behind a
rank is any object with the `ExplorerPort` methods -- the device explorer in
production (`DevicePort`), a CPU model in the tests.
"""
from __future__ import annotations

import time
from dataclasses import dataclass, field
from typing import List, Optional, Protocol, Sequence

import numpy as np

INT32_MAX = 2**31 - 1


class ExplorerPort(Protocol):
    def run(self, target: int, max_rounds: int):  # -> list of round tuples (may be empty)
        ...

    def pending(self) -> int:
        ...

    def take(self, k: int) -> List[List[int]]:
        ...

    def push(self, prefixes: Sequence[Sequence[int]]) -> None:
        ...

    def incumbent(self) -> int:  # current pruning bound
        ...

    def set_incumbent(self, v: int) -> None:
        ...

    def best(self):  # (value, schedule) of this rank's own best leaf, or (None, None)
        ...


class DevicePort:
    """ExplorerPort over a device context (fbb_explorer_*).

    `run` hands R rounds to ONE fbb_explorer_run call (host-planned rounds back to back
    on the library's stream, no Python between them); the pending size and incumbent
    come from the last round record and are tracked across take/push, so a rank makes
    one explorer_state call at construction and none per round."""

    def __init__(self, ctx, frozen: bool):
        self.ctx, self.frozen = ctx, frozen
        self.last_timing = None
        self.last_timings = []
        st = ctx.explorer_state()
        self._pend = st["pending"]
        self._inc = st["incumbent"]

    def run(self, target: int, max_rounds: int = 1):
        if self._pend <= 0:
            self.last_timings, self.last_timing = [], None
            return []
        r, t = self.ctx.explorer_run([target], max_rounds, timing=True)
        self.last_timings = t
        self.last_timing = t[-1] if t else None
        if r:
            self._inc, self._pend = int(r[-1][6]), int(r[-1][7])
        return r

    def round(self, target: int):
        r = self.run(target, 1)
        return r[0] if r else None

    def pending(self) -> int:
        return self._pend

    def take(self, k: int):
        out = self.ctx.explorer_take(k)
        self._pend -= len(out)
        return out

    def push(self, prefixes):
        self.ctx.explorer_push(prefixes)
        self._pend += len(prefixes)

    def incumbent(self) -> int:
        return self._inc if not self.frozen else INT32_MAX

    def set_incumbent(self, v: int) -> None:
        if not self.frozen and v < self._inc:
            self.ctx.explorer_set_incumbent(v)
            self._inc = int(v)

    def best(self):
        return self.ctx.explorer_best()


def plan_transfers(pending: Sequence[int], low: int, cap: int):
    """Deterministic rebalancing plan from the gathered pending sizes: every rank whose
    pending is below `low` (ascending) receives from the richest rank that still has
    more than 2*low and has not donated this step, half the difference (<= cap).
    Returns [(donor, receiver, count)]; identical on every rank."""
    est = list(pending)
    donated = set()
    plan = []
    for rcv in sorted(range(len(est)), key=lambda r: (est[r], r)):
        if est[rcv] >= low:
            break
        donors = [d for d in range(len(est)) if d not in donated and d != rcv and est[d] > 2 * low]
        if not donors:
            break
        d = max(donors, key=lambda r: (est[r], -r))
        k = min(cap, (est[d] - est[rcv]) // 2)
        if k <= 0:
            continue
        plan.append((d, rcv, k))
        est[d] -= k
        est[rcv] += k
        donated.add(d)
    return plan


@dataclass
class ParallelResult:
    rounds: list = field(default_factory=list)   # this rank's round tuples
    bounded: int = 0                              # all ranks
    transfers: int = 0                            # nodes moved between ranks
    exchange_seconds: float = 0.0                 # this rank's time in collectives
    best: Optional[int] = None                    # global best leaf (min over ranks)
    best_rank: int = -1
    schedule: Optional[list] = None
    exhausted: bool = False


class ParallelExplorer:
    """Runs synchronous exchange steps on every rank: `exchange_every` explorer rounds
    (one fbb_explorer_run call on a device port), then the rank exchange above.

    Exchanging every R rounds instead of every round keeps the collective (a ~20-50 us
    all_gather plus its host sync) off R-1 of every R rounds of ~120 us; the price is
    that an incumbent found on one rank prunes on the others up to R rounds later
    (solve mode only -- still exact, since the incumbent only lowers), and that a rank
    whose tree runs dry idles until the next exchange feeds it."""

    def __init__(self, port: ExplorerPort, n_jobs: int, group=None, device=None,
                 balance_every: int = 4, low_water: Optional[int] = None, max_transfer: int = 1 << 16,
                 exchange_every: int = 1):
        import torch
        import torch.distributed as dist

        self.port, self.n, self.group = port, n_jobs, group
        self.torch, self.dist = torch, dist
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.device = device if device is not None else "cpu"
        self.balance_every = max(1, balance_every)
        self.exchange_every = max(1, exchange_every)
        self.low_water = low_water
        self.max_transfer = max_transfer
        self.res = ParallelResult()
        self._bounded_local = 0
        self._round = 0

    # -- collectives ---------------------------------------------------------------------------
    def _gather(self, inc: int, pend: int, bounded: int):
        t = self.torch
        mine = t.tensor([inc, pend, bounded], dtype=t.int64, device=self.device)
        out = [t.zeros(3, dtype=t.int64, device=self.device) for _ in range(self.world)]
        self.dist.all_gather(out, mine, group=self.group)
        rows = t.stack(out).cpu().numpy()
        return rows[:, 0], rows[:, 1], rows[:, 2]

    def _rebalance(self, pending, target):
        low = self.low_water if self.low_water is not None else max(1, target // max(1, self.n))
        plan = plan_transfers([int(x) for x in pending], low, self.max_transfer)
        t = self.torch
        for donor, rcv, k in plan:
            if self.rank == donor:
                nodes = self.port.take(k)
                # int32 rows: torch's NCCL backend has no 16-bit integer type (c10d
                # NCCLUtils datatype map: int8/uint8/int32/int64/float types only)
                buf = np.full((k, self.n + 1), -1, np.int32)
                for i, pr in enumerate(nodes):
                    buf[i, 0] = len(pr)
                    buf[i, 1:1 + len(pr)] = pr
                self.dist.send(t.from_numpy(buf).to(self.device), rcv, group=self.group)
            elif self.rank == rcv:
                buf = t.zeros((k, self.n + 1), dtype=t.int32, device=self.device)
                self.dist.recv(buf, donor, group=self.group)
                rows = buf.cpu().numpy()
                self.port.push([list(map(int, r[1:1 + r[0]])) for r in rows if r[0] >= 0])
            self.res.transfers += k

    # -- driver --------------------------------------------------------------------------------
    def _run_local(self, target: int, rounds: int):
        if self.port.pending() <= 0:
            return []
        run = getattr(self.port, "run", None)
        if run is not None:
            return list(run(target, rounds))
        out = []  # a port with a one-round interface only
        while len(out) < rounds and self.port.pending() > 0:
            rec = self.port.round(target)
            if rec is None:
                break
            out.append(rec)
        return out

    def step(self, target: int) -> bool:
        """`exchange_every` rounds on every rank, then one exchange; False once every
        rank's pending is empty."""
        for rec in self._run_local(target, self.exchange_every):
            self.res.rounds.append(tuple(rec))
            self._bounded_local += int(rec[2])
        t0 = time.perf_counter()
        inc, pend, bnd = self._gather(self.port.incumbent(), self.port.pending(), self._bounded_local)
        g = int(inc.min())
        if g < self.port.incumbent():
            self.port.set_incumbent(g)
        self.res.bounded = int(bnd.sum())
        self._round += 1
        if int(pend.sum()) == 0:
            self.res.exchange_seconds += time.perf_counter() - t0
            self.res.exhausted = True
            return False
        if self.world > 1 and self._round % self.balance_every == 0:
            self._rebalance(pend, target)
        self.res.exchange_seconds += time.perf_counter() - t0
        return True

    def run(self, targets, max_rounds: int = 1 << 40, budget: int = 0) -> ParallelResult:
        targets = list(np.atleast_1d(targets))
        r = 0
        while r < max_rounds:
            tgt = int(targets[min(r, len(targets) - 1)])
            if not self.step(tgt):
                break
            r += 1
            if budget and self.res.bounded >= budget:
                break
        return self.finish()

    def finish(self) -> ParallelResult:
        """Global best leaf: min over ranks of (value, rank); its schedule is broadcast."""
        t = self.torch
        v, sched = self.port.best()
        mine = t.tensor([v if v is not None else INT32_MAX, self.rank], dtype=t.int64,
                        device=self.device)
        out = [t.zeros(2, dtype=t.int64, device=self.device) for _ in range(self.world)]
        self.dist.all_gather(out, mine, group=self.group)
        rows = sorted(tuple(int(x) for x in o.cpu().tolist()) for o in out)
        best, who = rows[0]
        self.res.best = None if best == INT32_MAX else best
        self.res.best_rank = who if best != INT32_MAX else -1
        if self.res.best is not None:
            buf = t.full((self.n,), -1, dtype=t.int32, device=self.device)
            if self.rank == who and sched is not None:
                buf = t.tensor(sched, dtype=t.int32, device=self.device)
            self.dist.broadcast(buf, who, group=self.group)
            s = [int(x) for x in buf.cpu().tolist()]
            self.res.schedule = s if s and s[0] >= 0 else None
        return self.res
