"""Python mirror of the reference flowbb C++ API over the C-ABI.

Each class / function cites the reference symbol it stands in for (paths relative
to the reference's proj/include/flowbb/).  All compute goes through
libflowbb_b200.so; nothing here evaluates a bound.
"""
from __future__ import annotations

import ctypes as C
import enum
import threading
import time
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from ._lib import (FBB_OK, BackendError, Descriptor, GroupStats, RoundRec, _i64p, check,
                   last_error, load_library)

# ---------------------------------------------------------------------------------------------
# L0: instance model (instance.hpp)
# ---------------------------------------------------------------------------------------------


class Instance:
    """instance.hpp:28-74: n jobs, m machines, p job-major (p[j][k])."""

    def __init__(self, jobs: int, machines: int, times):
        p = np.asarray(times, dtype=np.int64).reshape(jobs, machines)
        if jobs < 1 or machines < 1:
            raise ValueError("instance dimensions must be positive")
        if (p < 0).any():
            raise ValueError("negative processing time")
        self.p = np.ascontiguousarray(p.astype(np.int32))
        # instance.hpp:38-45: tails[j][k] = sum_{u>k} p[j][u]
        rev = np.cumsum(self.p[:, ::-1], axis=1)[:, ::-1]
        self.tails = np.ascontiguousarray(rev - self.p)

    def jobs(self) -> int:
        return self.p.shape[0]

    def machines(self) -> int:
        return self.p.shape[1]

    def __eq__(self, other):
        return isinstance(other, Instance) and np.array_equal(self.p, other.p)

    def key(self) -> bytes:
        return self.p.tobytes() + bytes(str(self.p.shape), "ascii")


def generate_instance(jobs: int, machines: int, seed: int) -> Instance:
    """instance.hpp:227-265: Taillard's generator (Lehmer 16807 mod 2^31-1, Schrage split),
    times U[1,99] drawn machine-major.  Host-side input generation."""
    if jobs < 1 or machines < 1:
        raise ValueError("instance dimensions must be positive")
    if seed <= 0 or seed >= 2147483647:
        raise ValueError("Taillard seed must be in (0, 2^31-1)")
    M, A, Q, R = 2147483647, 16807, 127773, 2836
    state = seed
    p = np.zeros((jobs, machines), np.int32)
    for k in range(machines):
        for j in range(jobs):
            kq = state // Q
            state = A * (state % Q) - R * kq
            if state < 0:
                state += M
            p[j, k] = 1 + int((state / M) * 99)
    return Instance(jobs, machines, p)


def makespan(inst: Instance, perm: Sequence[int]) -> int:
    """instance.hpp:92-96 (host-side utility; not on the accelerated path)."""
    h = np.zeros(inst.machines(), np.int64)
    for j in perm:
        prev = 0
        for k in range(inst.machines()):
            prev = max(prev, int(h[k])) + int(inst.p[j, k])
            h[k] = prev
    return int(h[-1])


# ---------------------------------------------------------------------------------------------
# L1: node batches (node.hpp), structure-of-arrays
# ---------------------------------------------------------------------------------------------


def nwords(n: int) -> int:
    return (n + 63) // 64


@dataclass
class NodeBatch:
    """A position-aligned batch of Node (node.hpp:28-53) as SoA:
    masks (cnt, W) uint64, heads (cnt, m) int32, depth (cnt,) int32, prefix (cnt, n) uint8."""

    masks: np.ndarray
    heads: np.ndarray
    depth: np.ndarray
    prefix: np.ndarray

    def __len__(self):
        return int(self.depth.shape[0])

    def __getitem__(self, sl):
        if isinstance(sl, int):
            sl = slice(sl, sl + 1)
        return NodeBatch(self.masks[sl], self.heads[sl], self.depth[sl], self.prefix[sl])

    def prefixes(self):
        return [list(map(int, self.prefix[i, : self.depth[i]])) for i in range(len(self))]

    @staticmethod
    def empty(inst: Instance, count: int = 0) -> "NodeBatch":
        n, m = inst.p.shape
        return NodeBatch(np.zeros((count, nwords(n)), np.uint64), np.zeros((count, m), np.int32),
                         np.zeros(count, np.int32), np.zeros((count, max(n, 1)), np.uint8))

    @staticmethod
    def root(inst: Instance) -> "NodeBatch":
        """Node::root (node.hpp:37-42)."""
        return NodeBatch.empty(inst, 1)

    @staticmethod
    def concat(parts: Sequence["NodeBatch"]) -> "NodeBatch":
        return NodeBatch(np.concatenate([p.masks for p in parts]),
                         np.concatenate([p.heads for p in parts]),
                         np.concatenate([p.depth for p in parts]),
                         np.concatenate([p.prefix for p in parts]))


def nodes_from_prefixes(inst: Instance, prefixes: Sequence[Sequence[int]]) -> NodeBatch:
    """Folds Node::child (node.hpp:44-52, child_heads instance.hpp:81-89) over each prefix,
    vectorised over the batch (host-side input preparation)."""
    n, m = inst.p.shape
    cnt = len(prefixes)
    out = NodeBatch.empty(inst, cnt)
    if cnt == 0:
        return out
    depth = np.array([len(pr) for pr in prefixes], np.int32)
    if (depth > n).any():
        raise ValueError("prefix longer than the job count")
    pre = np.zeros((cnt, max(n, 1)), np.int64)
    for i, pr in enumerate(prefixes):
        if len(set(pr)) != len(pr) or any(j < 0 or j >= n for j in pr):
            raise ValueError(f"invalid prefix {pr}")
        pre[i, : len(pr)] = pr
    heads = np.zeros((cnt, m), np.int64)
    masks = np.zeros((cnt, nwords(n)), np.uint64)
    p = inst.p.astype(np.int64)
    for i in range(int(depth.max())):
        act = depth > i
        jobs = pre[act, i]
        h = heads[act]
        prev = np.zeros(len(jobs), np.int64)
        for k in range(m):
            prev = np.maximum(prev, h[:, k]) + p[jobs, k]
            h[:, k] = prev
        heads[act] = h
        w = (jobs >> 6).astype(np.int64)
        bits = np.left_shift(np.uint64(1), (jobs & 63).astype(np.uint64))
        rows = np.nonzero(act)[0]
        np.bitwise_or.at(masks, (rows, w), bits)
    out.masks[:] = masks
    out.heads[:] = heads.astype(np.int32)
    out.depth[:] = depth
    out.prefix[:] = pre.astype(np.uint8)
    return out


# ---------------------------------------------------------------------------------------------
# L3: backend boundary (backend.hpp)
# ---------------------------------------------------------------------------------------------


@dataclass
class BackendDescriptor:
    """backend.hpp:27-33 (grain, base_units, max_batch)."""

    grain: int = 256
    base_units: int = 1
    max_batch: int = 65536


class Context:
    """One device context over one instance (fbb_create, include/flowbb_b200.h)."""

    def __init__(self, inst: Instance, device: int = 0):
        L = self.L = load_library()
        self.inst = inst
        self.device = device
        self.n, self.m = inst.p.shape
        self.W = nwords(self.n)
        self._lock = threading.Lock()
        h = L.fbb_create(device, np.ascontiguousarray(inst.p.ravel()), self.n, self.m)
        if not h:
            status, _, msg = last_error(None)
            if status == -1:
                raise ValueError(msg)
            raise BackendError(device, msg, status)
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            self.L.fbb_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc):
        check(self.h, rc, self.device)

    def descriptor(self) -> BackendDescriptor:
        d = Descriptor()
        self._check(self.L.fbb_descriptor(self.h, C.byref(d)))
        return BackendDescriptor(d.grain, d.base_units, d.max_batch)

    def kernels(self) -> str:
        """The kernel variants this context launches (fbb_kernels)."""
        buf = C.create_string_buffer(256)
        self._check(self.L.fbb_kernels(self.h, buf, 256))
        return buf.value.decode()

    # K1 ----------------------------------------------------------------------------------
    def bound(self, batch: NodeBatch) -> np.ndarray:
        cnt = len(batch)
        out = np.zeros(max(cnt, 1), np.int32)
        if cnt == 0:
            return out[:0]
        with self._lock:
            self._check(self.L.fbb_bound(self.h, np.ascontiguousarray(batch.masks.ravel()),
                                         np.ascontiguousarray(batch.heads.ravel()),
                                         np.ascontiguousarray(batch.depth), cnt, out))
        return out

    def bound_device(self, d_masks: int, d_heads: int, d_depth: int, count: int, d_lb: int,
                     stream: int = 0):
        """K1 on device pointers (fbb_bound_device), asynchronous on `stream`."""
        self._check(self.L.fbb_bound_device(self.h, d_masks, d_heads, d_depth, int(count), d_lb,
                                            stream or None))

    def synth_pool(self, seed: int, count: int, min_depth: int, max_depth: int, d_masks: int,
                   d_heads: int, d_depth: int, d_prefix: int = 0, stream: int = 0):
        """Synthetic random nodes generated on the device (fbb_synth_pool)."""
        self._check(self.L.fbb_synth_pool(self.h, int(seed) & (2**64 - 1), int(count),
                                          int(min_depth), int(max_depth), d_masks, d_heads,
                                          d_depth, d_prefix or None, stream or None))

    # K2 ----------------------------------------------------------------------------------
    def expand_bound_prune(self, parents: NodeBatch, ub: int, frozen: bool):
        """Returns (survivors NodeBatch, survivor lbs, leaf_best or None, leaf_pos,
        leaf_schedule or None, round counts tuple)."""
        n, m, W = self.n, self.m, self.W
        cnt = len(parents)
        cap = max(1, int(((n - parents.depth.astype(np.int64)).sum()) if cnt else 1))
        om = np.zeros(cap * W, np.uint64)
        oh = np.zeros(cap * m, np.int32)
        od = np.zeros(cap, np.int32)
        op = np.zeros(cap * n, np.uint8)
        ol = np.zeros(cap, np.int32)
        oc = C.c_int64(0)
        lbest = C.c_int32(0)
        lpos = C.c_int64(0)
        sched = np.zeros(max(n, 1), np.int32)
        rec = RoundRec()
        pm = np.ascontiguousarray(parents.masks.ravel()) if cnt else np.zeros(W, np.uint64)
        ph = np.ascontiguousarray(parents.heads.ravel()) if cnt else np.zeros(m, np.int32)
        pd = np.ascontiguousarray(parents.depth) if cnt else np.zeros(1, np.int32)
        pp = np.ascontiguousarray(parents.prefix.ravel()) if cnt else np.zeros(n, np.uint8)
        with self._lock:
            self._check(self.L.fbb_expand_bound_prune(
                self.h, pm, ph, pd, pp, cnt, int(ub), 1 if frozen else 0, om, oh, od, op, ol,
                C.byref(oc), C.byref(lbest), C.byref(lpos), sched, C.byref(rec)))
        k = oc.value
        surv = NodeBatch(om.reshape(cap, W)[:k].copy(), oh.reshape(cap, m)[:k].copy(),
                         od[:k].copy(), op.reshape(cap, n)[:k].copy())
        best = lbest.value if lbest.value != 2**31 - 1 else None
        return (surv, ol[:k].copy(), best, lpos.value,
                [int(x) for x in sched] if best is not None else None, rec.as_tuple())

    # explorer (pending tree in HBM, or in pinned host memory) ------------------------------
    def explorer_set_residency(self, on_host: bool):
        """Pending tree in device memory (False) or pinned host memory (True: every round
        uploads its parents and receives only the survivors).  Clears the tree."""
        self._check(self.L.fbb_explorer_set_residency(self.h, 1 if on_host else 0))

    def explorer_reset(self, nodes: NodeBatch, ub: int, frozen: bool = True):
        cnt = len(nodes)
        pre = np.ascontiguousarray(nodes.prefix.ravel()) if cnt else np.zeros(1, np.uint8)
        dep = np.ascontiguousarray(nodes.depth) if cnt else np.zeros(1, np.int32)
        self._check(self.L.fbb_explorer_reset(self.h, pre, dep, cnt, int(ub), 1 if frozen else 0))

    def explorer_start_solve(self, ub: Optional[int] = None):
        rec = RoundRec()
        self._check(self.L.fbb_explorer_start_solve(self.h, -1 if ub is None else int(ub),
                                                    C.byref(rec)))
        return rec.as_tuple()

    def explorer_run(self, targets, max_rounds: int, budget: int = 0, timing: bool = False):
        """Runs rounds on the device explorer; returns the per-round count tuples
        (and, with timing=True, the per-round device timings)."""
        t = np.ascontiguousarray(np.atleast_1d(np.asarray(targets, np.int64)))
        recs = (RoundRec * max(min(max_rounds, 1 << 20), 1))()
        done = C.c_int64(0)
        self._check(self.L.fbb_explorer_run(self.h, t, len(t), min(max_rounds, 1 << 20), budget,
                                            C.cast(recs, C.c_void_p), C.byref(done)))
        rounds = [recs[i].as_tuple() for i in range(done.value)]
        if timing:
            return rounds, [recs[i].timing() for i in range(done.value)]
        return rounds

    def explorer_set_incumbent(self, ub: int):
        self._check(self.L.fbb_explorer_set_incumbent(self.h, int(ub)))

    def explorer_best(self):
        """(value, schedule) of this context's own best leaf, or (None, None)."""
        v = C.c_int32(0)
        sched = np.zeros(max(self.n, 1), np.int32)
        found = self.L.fbb_explorer_best(self.h, C.byref(v), sched)
        if found < 0:
            self._check(found)
        if not found:
            return None, None
        return v.value, [int(x) for x in sched[: self.n]]

    def explorer_take(self, k: int):
        """Removes up to k pending nodes (shallowest buckets first); returns their prefixes."""
        k = max(0, int(k))
        pre = np.zeros(max(k, 1) * self.n, np.uint8)
        dep = np.zeros(max(k, 1), np.int32)
        got = C.c_int64(0)
        self._check(self.L.fbb_explorer_take(self.h, k, pre, dep, C.byref(got)))
        pre = pre.reshape(-1, self.n)
        return [list(map(int, pre[i, : dep[i]])) for i in range(got.value)]

    def explorer_push(self, prefixes):
        if not prefixes:
            return
        batch = nodes_from_prefixes(self.inst, prefixes)
        self._check(self.L.fbb_explorer_push(self.h, np.ascontiguousarray(batch.prefix.ravel()),
                                             np.ascontiguousarray(batch.depth), len(batch)))

    def explorer_state(self):
        inc = C.c_int32(0)
        found = C.c_int32(0)
        sched = np.zeros(max(self.n, 1), np.int32)
        pend = C.c_int64(0)
        tot = np.zeros(4, np.int64)
        self._check(self.L.fbb_explorer_state(self.h, C.byref(inc), C.byref(found), sched,
                                              C.byref(pend), tot))
        return {"incumbent": inc.value, "found": bool(found.value),
                "schedule": [int(x) for x in sched] if found.value else None,
                "pending": pend.value, "branched": int(tot[0]), "bounded": int(tot[1]),
                "pruned": int(tot[2]), "leaves": int(tot[3])}

    def explorer_pending(self):
        cnt = C.c_int64(0)
        self.L.fbb_explorer_pending(self.h, np.zeros(1, np.uint8), np.zeros(1, np.int32), 0,
                                    C.byref(cnt))
        k = cnt.value
        pre = np.zeros(max(k, 1) * self.n, np.uint8)
        dep = np.zeros(max(k, 1), np.int32)
        self._check(self.L.fbb_explorer_pending(self.h, pre, dep, k, C.byref(cnt)))
        pre = pre.reshape(-1, self.n)
        return [list(map(int, pre[i, : dep[i]])) for i in range(k)]


_ctx_cache: dict = {}
_ctx_lock = threading.Lock()


def context_for(inst: Instance, device: int = 0) -> Context:
    key = (inst.key(), device)
    with _ctx_lock:
        ctx = _ctx_cache.get(key)
        if ctx is None:
            if len(_ctx_cache) > 16:
                _ctx_cache.clear()
            ctx = _ctx_cache[key] = Context(inst, device)
        return ctx


class GpuBackend:
    """Models the reference Backend concept (backend.hpp:50-69, test_backend.cpp:14-22):
    descriptor() and evaluate(inst, nodes) -> position-aligned lower bounds."""

    def __init__(self, descriptor: Optional[BackendDescriptor] = None, device: int = 0):
        self.device = device
        self._descriptor = descriptor

    def descriptor(self) -> BackendDescriptor:
        if self._descriptor is None:
            raise ValueError("descriptor is only known once an instance is bound; pass one")
        return self._descriptor

    def evaluate(self, inst: Instance, nodes: NodeBatch) -> np.ndarray:
        return context_for(inst, self.device).bound(nodes)


def split_slices(total: int, k: int):
    """backend.hpp:71-84: contiguous slices; the first total % k get one more."""
    if k < 1:
        raise ValueError("backend count must be positive")
    base, extra = divmod(total, k)
    out, off = [], 0
    for i in range(k):
        ln = base + (1 if i < extra else 0)
        out.append((off, ln))
        off += ln
    return out


def merge_slices(slice_results, slices):
    """backend.hpp:86-100: concatenation in slice order; length mismatch = BackendError(i)."""
    parts = []
    for i, res in enumerate(slice_results):
        if len(res) != slices[i][1]:
            raise BackendError(i, "slice result length mismatch")
        parts.append(np.asarray(res, np.int32))
    return np.concatenate(parts) if parts else np.zeros(0, np.int32)


def evaluate_multi(backends, inst: Instance, batch: NodeBatch) -> np.ndarray:
    """backend.hpp:102-138: split, evaluate the slices concurrently (one host thread per
    backend), merge in order; the first failing slice poisons the round."""
    if not backends:
        raise ValueError("empty backend set")
    if len(batch) == 0:
        return np.zeros(0, np.int32)
    k = len(backends)
    if k == 1:
        return np.asarray(backends[0].evaluate(inst, batch), np.int32)
    slices = split_slices(len(batch), k)
    with ThreadPoolExecutor(max_workers=k) as ex:
        futs = [ex.submit(backends[i].evaluate, inst, batch[off:off + ln])
                for i, (off, ln) in enumerate(slices)]
        results, failed, failure = [None] * k, -1, ""
        for i, f in enumerate(futs):
            try:
                results[i] = f.result()
            except Exception as e:  # noqa: BLE001
                if failed < 0:
                    failed, failure = i, str(e)
    if failed >= 0:
        raise BackendError(failed, failure)
    return merge_slices(results, slices)


class BackendSet:
    """backend.hpp:140-158 over GPUs: backend i runs on device devices[i % len(devices)]."""

    def __init__(self, count: int, descriptor: Optional[BackendDescriptor] = None,
                 devices: Optional[Sequence[int]] = None):
        if count < 1:
            raise ValueError("backend count must be positive")
        devices = list(devices) if devices else [0]
        self.backends = [GpuBackend(descriptor, devices[i % len(devices)]) for i in range(count)]

    def size(self) -> int:
        return len(self.backends)

    def descriptor(self) -> BackendDescriptor:
        return self.backends[0].descriptor()

    def evaluate(self, inst: Instance, batch: NodeBatch) -> np.ndarray:
        return evaluate_multi(self.backends, inst, batch)


# ---------------------------------------------------------------------------------------------
# L5: tuner (autotune.hpp)
# ---------------------------------------------------------------------------------------------


class DeviceGroup:
    """fbb_group_*: the multi-device explorer inside one process (the paper's split of one
    host's pools over its GPUs; BackendSet(k) over k devices,
    backend.hpp:142-158).  Member i is a full context (`context(i)`); the library runs
    every member's rounds on its own host thread and exchanges the incumbent (solve) and
    pending subtrees between steps.  Device ids may repeat (tests on one GPU)."""

    def __init__(self, inst: Instance, devices: Sequence[int]):
        L = self.L = load_library()
        self.inst = inst
        self.n, self.m = inst.p.shape
        devs = np.ascontiguousarray(np.asarray(list(devices), np.int32))
        h = L.fbb_group_create(devs, len(devs), np.ascontiguousarray(inst.p.ravel()), self.n, self.m)
        if not h:
            status, _, msg = last_error(None)
            if status == -1:
                raise ValueError(msg or "invalid group")
            raise BackendError(int(devs[0]) if len(devs) else -1, msg, status)
        self.h = h
        self.devices = [int(d) for d in devs]

    def close(self):
        if getattr(self, "h", None):
            self.L.fbb_group_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc):
        if rc != FBB_OK:
            member = C.c_int(-1)
            buf = C.create_string_buffer(512)
            status = self.L.fbb_group_last_error(self.h, C.byref(member), buf, 512)
            msg = buf.value.decode(errors="replace")
            if status == -1:
                raise ValueError(msg)
            raise BackendError(member.value, msg, status)

    def size(self) -> int:
        return self.L.fbb_group_size(self.h)

    def reset(self, nodes, ub: int, frozen: bool = True):
        """Splits the nodes (NodeBatch or prefixes) into size() contiguous slices."""
        if not isinstance(nodes, NodeBatch):
            nodes = nodes_from_prefixes(self.inst, nodes) if len(nodes) else NodeBatch.empty(self.inst)
        cnt = len(nodes)
        pre = np.ascontiguousarray(nodes.prefix.ravel()) if cnt else np.zeros(1, np.uint8)
        dep = np.ascontiguousarray(nodes.depth) if cnt else np.zeros(1, np.int32)
        self._check(self.L.fbb_group_reset(self.h, pre, dep, cnt, int(ub), 1 if frozen else 0))

    def start_solve(self, ub: Optional[int] = None):
        self._check(self.L.fbb_group_start_solve(self.h, -1 if ub is None else int(ub)))

    def run(self, target: int, max_steps: int = 1 << 40, rounds_per_step: int = 4,
            balance_every: int = 1, budget: int = 0) -> dict:
        st = GroupStats()
        self._check(self.L.fbb_group_run(self.h, int(target), int(max_steps), int(rounds_per_step),
                                         int(balance_every), int(budget), C.byref(st)))
        return st.as_dict()

    def best(self):
        """(value, schedule) of the group's best leaf, or (None, None)."""
        v = C.c_int32(0)
        sched = np.zeros(max(self.n, 1), np.int32)
        found = self.L.fbb_group_best(self.h, C.byref(v), sched)
        if found < 0:
            self._check(found)
        if not found:
            return None, None
        return v.value, [int(x) for x in sched[: self.n]]


class TunerPhase(enum.IntEnum):
    doubling = 0
    refining = 1
    fixed = 2


class Tuner:
    """autotune.hpp:35-156 through fbb_tuner_* (host C++ state machine)."""

    def __init__(self, descriptor: BackendDescriptor, window: int, probes_per_side: int = 2):
        self.L = load_library()
        h = self.L.fbb_tuner_create(int(descriptor.grain), int(descriptor.base_units),
                                    int(descriptor.max_batch), int(window), int(probes_per_side))
        if not h:
            raise ValueError("invalid tuner configuration")
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            self.L.fbb_tuner_destroy(self.h)
            self.h = None

    def target(self) -> int:
        return int(self.L.fbb_tuner_target(self.h))

    def observe(self, nodes_bounded: int, elapsed_seconds: float) -> None:
        if self.L.fbb_tuner_observe(self.h, int(nodes_bounded), float(elapsed_seconds)) != FBB_OK:
            raise ValueError("elapsed time must be positive")

    def phase(self) -> TunerPhase:
        return TunerPhase(self.L.fbb_tuner_phase(self.h))

    def best_batch(self) -> int:
        return int(self.L.fbb_tuner_best_batch(self.h))

    def best_throughput(self) -> float:
        return float(self.L.fbb_tuner_best_throughput(self.h))

    def set_trace(self, fn) -> None:
        """Tuner::set_trace (autotune.hpp): fn(window, batch, throughput, decision) per
        closed window; None disables it."""
        from ._lib import TRACE_FN

        self._trace = TRACE_FN(lambda _u, w, b, tp, d: fn(w, b, tp, d.decode())) if fn else None
        self.L.fbb_tuner_set_trace(self.h, self._trace or TRACE_FN(), None)


# ---------------------------------------------------------------------------------------------
# L4/L6: explorer drivers (search.hpp solve, bench.hpp resolve_workload)
# ---------------------------------------------------------------------------------------------


@dataclass
class SearchStats:
    """search.hpp:21-26"""

    branched: int = 0
    bounded: int = 0
    pruned: int = 0
    elapsed_seconds: float = 0.0


@dataclass
class Solution:
    """search.hpp:28-35"""

    optimum: int = 0
    schedule: Optional[list] = None
    stats: SearchStats = field(default_factory=SearchStats)
    rounds: list = field(default_factory=list)
    exhausted: bool = True  # False when a node budget stopped the run

    def found(self) -> bool:
        return self.schedule is not None


@dataclass
class ResolutionResult:
    """bench.hpp:53-58"""

    best: Optional[int] = None
    nodes_bounded: int = 0
    elapsed_seconds: float = 0.0
    batch_used: int = 0
    rounds: list = field(default_factory=list)
    exhausted: bool = True


def _drive(ctx: Context, targets, autotune, window, probes, budget, max_rounds, tuner=None):
    """Round loop on the device explorer: fixed target schedule (one C call), or the
    tuner observing each round's wall time (search.hpp:155-165).  `tuner`: one that
    already observed earlier rounds (solve's root round)."""
    if not autotune:
        return ctx.explorer_run(targets, max_rounds, budget), None
    if tuner is None:
        tuner = Tuner(ctx.descriptor(), window, probes)
    rounds = []
    while len(rounds) < max_rounds:
        t0 = time.perf_counter()
        rec = ctx.explorer_run([tuner.target()], 1, budget)
        el = time.perf_counter() - t0
        if not rec:
            break
        rounds.extend(rec)
        tuner.observe(rec[0][2], max(el, 1e-9))
    return rounds, tuner


def resolve_workload(inst: Instance, nodes, incumbent_value: int, batch: Optional[int] = None,
                     autotune: bool = False, window: int = 5, probes: int = 2, budget: int = 0,
                     targets=None, device: int = 0, max_rounds: int = 1 << 40,
                     pending_on_host: bool = False) -> ResolutionResult:
    """bench.hpp:63-114 with the incumbent frozen at `incumbent_value`, on the device
    explorer.  `nodes`: NodeBatch or list of prefixes (the snapshot list L, pushed in order).
    `targets` (per-round pool targets) replays a recorded schedule; `budget` stops after the
    first round whose cumulative bounded count reaches it.  `pending_on_host` keeps the
    pending tree in pinned host memory (parents uploaded, survivors returned per round)."""
    ctx = context_for(inst, device)
    ctx.explorer_set_residency(pending_on_host)
    if not isinstance(nodes, NodeBatch):
        nodes = nodes_from_prefixes(inst, nodes)
    if targets is None:
        targets = [batch if batch else ctx.descriptor().grain * ctx.descriptor().base_units]
    t0 = time.perf_counter()
    ctx.explorer_reset(nodes, incumbent_value, frozen=True)
    rounds, tuner = _drive(ctx, targets, autotune, window, probes, budget, max_rounds)
    st = ctx.explorer_state()
    res = ResolutionResult()
    res.elapsed_seconds = time.perf_counter() - t0
    res.best = st["incumbent"] if st["found"] else None
    res.nodes_bounded = st["bounded"]
    res.rounds = rounds
    res.exhausted = st["pending"] == 0
    res.batch_used = tuner.best_batch() if tuner else int(np.atleast_1d(targets)[-1])
    return res


def solve(inst: Instance, initial_ub: Optional[int] = None, fixed_batch: Optional[int] = None,
          autotune: bool = False, window: int = 5, probes: int = 2, budget: int = 0,
          targets=None, device: int = 0, max_rounds: int = 1 << 40,
          pending_on_host: bool = False) -> Solution:
    """search.hpp:124-174 on the device explorer (strict-improvement incumbent, mid-batch
    updates, deepest-first LIFO selection)."""
    ctx = context_for(inst, device)
    ctx.explorer_set_residency(pending_on_host)
    # the tuner exists before the root round and observes it (batch of 1), as
    # search.hpp:139-165 does: its first window closes on the reference's iteration
    tuner = Tuner(ctx.descriptor(), window, probes) if autotune else None
    t0 = time.perf_counter()
    r0 = ctx.explorer_start_solve(initial_ub)
    if tuner is not None:
        tuner.observe(r0[2], max(time.perf_counter() - t0, 1e-9))
    if targets is None:
        d = ctx.descriptor()
        targets = [fixed_batch if fixed_batch else d.grain * d.base_units]
    rounds, _ = _drive(ctx, targets, autotune, window, probes, budget, max_rounds, tuner)
    st = ctx.explorer_state()
    sol = Solution()
    sol.optimum = st["incumbent"]
    sol.schedule = st["schedule"]
    sol.stats = SearchStats(st["branched"], st["bounded"], st["pruned"],
                            time.perf_counter() - t0)
    sol.rounds = [r0] + rounds
    sol.exhausted = st["pending"] == 0
    return sol
