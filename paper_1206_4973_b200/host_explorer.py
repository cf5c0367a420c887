"""Host-pending explorer: the paper's Type-1 model through the C-ABI with HOST buffers.

The control thread keeps the reference's PendingTree (pending.hpp:13-56: per-depth
stacks, deepest first, LIFO) in host memory as flat numpy stacks, selects each pool
exactly like fill_buffer (search.hpp:64-73), and hands the parents to the GPU in one
fbb_expand_bound_prune call (include/flowbb_b200.h), which returns only the surviving
children, stably compacted; they are pushed back in batch order (integrate,
search.hpp:84-107 / frozen prune, bench.hpp:96-106).  This is the drop-in round a
reference user gets by replacing `fill_buffer -> BackendSet::evaluate -> integrate`,
and it is what bench.py times as the end-to-end (`e2e`) number: every step copies the
parents host->device and the survivors device->host (pinned buffers when available).
"""
from __future__ import annotations

import ctypes as C
import time

import numpy as np

from ._lib import RoundRec, check
from .flowbb import Context, Instance, NodeBatch, nodes_from_prefixes, nwords


def _pinned(shape, dtype):
    """Page-locked numpy buffer (torch pin_memory) when CUDA is present, else plain."""
    try:
        import torch

        if torch.cuda.is_available():
            t = torch.empty(int(np.prod(shape)) * np.dtype(dtype).itemsize, dtype=torch.uint8,
                            pin_memory=True)
            return t.numpy().view(dtype).reshape(shape)
    except Exception:
        pass
    return np.empty(shape, dtype)


class _Stack:
    def __init__(self, n, m, W, cap=1024):
        self.n, self.m, self.W = n, m, W
        self.masks = np.zeros((cap, W), np.uint64)
        self.heads = np.zeros((cap, m), np.int32)
        self.prefix = np.zeros((cap, max(n, 1)), np.uint8)
        self.size = 0

    def reserve(self, want):
        if want <= len(self.heads):
            return
        cap = max(want, 2 * len(self.heads))
        for name in ("masks", "heads", "prefix"):
            old = getattr(self, name)
            new = np.zeros((cap,) + old.shape[1:], old.dtype)
            new[: self.size] = old[: self.size]
            setattr(self, name, new)

    def push(self, masks, heads, prefix):
        k = len(heads)
        self.reserve(self.size + k)
        self.masks[self.size:self.size + k] = masks
        self.heads[self.size:self.size + k] = heads
        self.prefix[self.size:self.size + k] = prefix
        self.size += k


class HostExplorer:
    """resolve_workload / solve rounds with the pending tree on the host."""

    def __init__(self, ctx: Context, max_pool: int = 1 << 20):
        self.ctx = ctx
        self.n, self.m, self.W = ctx.n, ctx.m, ctx.W
        self.stacks = [_Stack(self.n, self.m, self.W) for _ in range(self.n + 1)]
        self.incumbent = 0
        self.frozen = True
        self.found = False
        self.best = None
        self.schedule = None
        self._alloc(max_pool)

    def _alloc(self, cap):
        n, m, W = self.n, self.m, self.W
        self.cap = cap
        self.in_masks = _pinned((cap, W), np.uint64)
        self.in_heads = _pinned((cap, m), np.int32)
        self.in_depth = _pinned((cap,), np.int32)
        self.in_prefix = _pinned((cap, max(n, 1)), np.uint8)
        kids = cap * n
        self.kcap = kids
        self.out_masks = _pinned((kids, W), np.uint64)
        self.out_heads = _pinned((kids, m), np.int32)
        self.out_depth = _pinned((kids,), np.int32)
        self.out_prefix = _pinned((kids, max(n, 1)), np.uint8)
        self.out_lb = _pinned((kids,), np.int32)
        self.sched = np.zeros(max(n, 1), np.int32)

    def pending(self) -> int:
        return sum(s.size for s in self.stacks)

    def reset(self, nodes, ub: int, frozen: bool = True):
        """bench.hpp:83-84: push the snapshot nodes in order."""
        if not isinstance(nodes, NodeBatch):
            nodes = nodes_from_prefixes(self.ctx.inst, nodes)
        for s in self.stacks:
            s.size = 0
        for i in range(len(nodes)):
            d = int(nodes.depth[i])
            self.stacks[d].push(nodes.masks[i:i + 1], nodes.heads[i:i + 1], nodes.prefix[i:i + 1])
        self.incumbent, self.frozen = int(ub), frozen
        self.found, self.best, self.schedule = False, None, None

    def round(self, target: int):
        """One round; returns (round tuple, seconds, h2d_bytes, d2h_bytes)."""
        t0 = time.perf_counter()
        n, m, W = self.n, self.m, self.W
        # fill_buffer (search.hpp:64-73): deepest bucket first, LIFO, until >= target
        segs, have, npar = [], 0, 0
        for d in range(n, -1, -1):
            if have >= target:
                break
            st = self.stacks[d]
            if st.size == 0:
                continue
            r = n - d
            k = min(st.size, -(-(target - have) // r))
            segs.append((d, k))
            have += k * r
            npar += k
        if npar == 0:
            return None
        if npar > self.cap or have > self.kcap:
            self._alloc(max(npar, have // max(1, n - 1) + 1, 2 * self.cap))
        o = 0
        for d, k in segs:
            st = self.stacks[d]
            lo = st.size - k
            sl = slice(lo, st.size)
            self.in_masks[o:o + k] = st.masks[sl][::-1]
            self.in_heads[o:o + k] = st.heads[sl][::-1]
            self.in_prefix[o:o + k] = st.prefix[sl][::-1]
            self.in_depth[o:o + k] = d
            st.size = lo
            o += k
        L = self.ctx.L
        oc, lbest, lpos, rec = C.c_int64(0), C.c_int32(0), C.c_int64(0), RoundRec()
        rc = L.fbb_expand_bound_prune(
            self.ctx.h, self.in_masks.reshape(-1), self.in_heads.reshape(-1), self.in_depth,
            self.in_prefix.reshape(-1), npar, self.incumbent, 1 if self.frozen else 0,
            self.out_masks.reshape(-1), self.out_heads.reshape(-1), self.out_depth,
            self.out_prefix.reshape(-1), self.out_lb, C.byref(oc), C.byref(lbest), C.byref(lpos),
            self.sched, C.byref(rec))
        check(self.ctx.h, rc, self.ctx.device)
        k = oc.value
        # push survivors in batch order (they arrive grouped by depth, deepest first)
        if k:
            dep = self.out_depth[:k]
            cuts = np.flatnonzero(np.diff(dep)) + 1
            starts = np.concatenate(([0], cuts))
            ends = np.concatenate((cuts, [k]))
            for a, b in zip(starts, ends):
                self.stacks[int(dep[a])].push(self.out_masks[a:b], self.out_heads[a:b],
                                              self.out_prefix[a:b])
        if lbest.value != 2**31 - 1:
            v = lbest.value
            if self.frozen:
                if v < self.incumbent and (self.best is None or v < self.best):
                    self.best, self.found = v, True
            elif v < self.incumbent:
                self.incumbent, self.best, self.found = v, v, True
                self.schedule = [int(x) for x in self.sched[:n]]
        inc = (self.best if self.found else self.incumbent) if self.frozen else self.incumbent
        tup = (int(target), rec.branched, rec.bounded, rec.inserted, rec.pruned, rec.leaves, inc,
               self.pending())
        h2d = npar * (W * 8 + m * 4 + 4 + n)
        d2h = k * (W * 8 + m * 4 + 4 + n + 4) + 64
        return tup, time.perf_counter() - t0, h2d, d2h


def resolve_host(inst: Instance, nodes, ub: int, targets, budget: int = 0, device: int = 0,
                 max_rounds: int = 1 << 30):
    """resolve_workload (bench.hpp:63-114) with the host-pending explorer."""
    from .flowbb import context_for

    ex = HostExplorer(context_for(inst, device))
    ex.reset(nodes, ub, frozen=True)
    rounds, bounded = [], 0
    targets = list(np.atleast_1d(targets))
    while ex.pending() and len(rounds) < max_rounds:
        t = int(targets[min(len(rounds), len(targets) - 1)])
        tup, *_ = ex.round(t)
        rounds.append(tup)
        bounded += tup[2]
        if budget and bounded >= budget:
            break
    return rounds, ex
