"""A CPU model of one rank's explorer for the multi-process tests (TEST INFRASTRUCTURE).

`OraclePort` implements parallel.ExplorerPort with the reference's round semantics
(fill_buffer search.hpp:64-73, branch :40-59, integrate :84-107 / frozen prune
bench.hpp:96-106, PendingTree pending.hpp:13-56) on top of the C oracle's branch and
lower_bound, so the rank-exchange protocol of paper_1206_4973_b200.parallel can run
under gloo on CPU exactly as it runs over NCCL with device explorers."""
from __future__ import annotations

INT32_MAX = 2**31 - 1


class OraclePort:
    def __init__(self, oracle, p, ub, frozen, roots):
        self.orc, self.p, self.frozen = oracle, p, frozen
        self.n = p.shape[0]
        self.ub = int(ub)
        self.buckets = [[] for _ in range(self.n + 1)]
        self.best_v, self.sched = None, None
        for pr in roots:
            self.buckets[len(pr)].append(list(pr))

    def pending(self):
        return sum(len(b) for b in self.buckets)

    def incumbent(self):
        return INT32_MAX if self.frozen else self.ub

    def set_incumbent(self, v):
        if not self.frozen:
            self.ub = min(self.ub, int(v))

    def best(self):
        return self.best_v, (self.sched if not self.frozen else None)

    def take(self, k):
        out = []
        for d in range(self.n + 1):
            while self.buckets[d] and len(out) < k:
                out.append(self.buckets[d].pop())
        return out

    def push(self, prefixes):
        for pr in prefixes:
            self.buckets[len(pr)].append(list(pr))

    def round(self, target):
        n = self.n
        batch, branched = [], 0
        for d in range(n, -1, -1):  # fill_buffer: deepest first, LIFO, until >= target
            while self.buckets[d] and len(batch) < target:
                parent = self.buckets[d].pop()
                branched += 1
                kids, _ = self.orc.branch(self.p, parent)
                batch += [list(map(int, k)) for k in kids]
            if len(batch) >= target:
                break
        if not batch:
            return None
        leaves = inserted = pruned = 0
        for child in batch:
            lb = self.orc.lower_bound(self.p, child)
            if len(child) == n:
                leaves += 1
                if self.frozen:
                    if lb < self.ub and (self.best_v is None or lb < self.best_v):
                        self.best_v = lb
                elif lb < self.ub:
                    self.ub, self.best_v, self.sched = lb, lb, child
            elif lb < self.ub:
                inserted += 1
                self.buckets[len(child)].append(child)
            else:
                pruned += 1
        inc = (self.best_v if self.best_v is not None else self.ub) if self.frozen else self.ub
        return (target, branched, len(batch), inserted, pruned, leaves, inc, self.pending())
