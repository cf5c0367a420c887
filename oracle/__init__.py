"""ctypes bindings for the parity checkers (TEST INFRASTRUCTURE ONLY).

`Oracle` wraps oracle/liboracle.so, the C restatement of the reference hot path
(oracle/flowbb_oracle.c).  `Ref` wraps oracle/_ref/libflowbb_ref.so, the
reference's own headers compiled in place (oracle/ref_shim.cpp); it exists only
where /root/reference was present at build time.

Only tests/, __graft_entry__.smoke() and bench.py's reference / cpu_baseline legs
may import this package.  The product path (paper_1206_4973_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libflowbb_ref.so")
REF_SRC = "/root/reference/proj"

_i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")


class Round(C.Structure):
    """orc_round (oracle/flowbb_oracle.h)."""

    _fields_ = [
        ("target", C.c_int64),
        ("branched", C.c_int64),
        ("bounded", C.c_int64),
        ("inserted", C.c_int64),
        ("pruned", C.c_int64),
        ("leaves", C.c_int64),
        ("incumbent", C.c_int32),
        ("pad", C.c_int32),
        ("pending", C.c_int64),
    ]

    def as_tuple(self):
        return (self.target, self.branched, self.bounded, self.inserted, self.pruned,
                self.leaves, self.incumbent, self.pending)


class Result(C.Structure):
    """orc_result (oracle/flowbb_oracle.h)."""

    _fields_ = [
        ("branched", C.c_int64),
        ("bounded", C.c_int64),
        ("pruned", C.c_int64),
        ("leaves", C.c_int64),
        ("rounds", C.c_int64),
        ("optimum", C.c_int32),
        ("found", C.c_int32),
        ("pending", C.c_int64),
    ]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


ROUND_FIELDS = ("target", "branched", "bounded", "inserted", "pruned", "leaves", "incumbent",
                "pending")


def build(ref: bool | None = None) -> None:
    """make -C oracle (liboracle.so; _ref when the reference sources exist)."""
    targets = ["liboracle.so"]
    if ref is None:
        ref = os.path.isdir(REF_SRC)
    if ref:
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE, *targets], check=True)


def nwords(n: int) -> int:
    return (n + 63) // 64


def _targets(targets):
    t = np.ascontiguousarray(np.atleast_1d(np.asarray(targets, dtype=np.int64)))
    return t, len(t)


class Oracle:
    """The C restatement."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build(ref=False)
        L = self.lib = C.CDLL(path)
        L.orc_generate_instance.argtypes = [C.c_int, C.c_int, C.c_int32, _i32p]
        L.orc_generate_instance.restype = C.c_int
        L.orc_tails.argtypes = [C.c_int, C.c_int, _i32p, _i32p]
        L.orc_child_heads.argtypes = [C.c_int, C.c_int, _i32p, _i32p, C.c_int, _i32p]
        L.orc_makespan.argtypes = [C.c_int, C.c_int, _i32p, _i32p, C.c_int]
        L.orc_makespan.restype = C.c_int32
        L.orc_johnson_two_machine.argtypes = [_i32p, _i32p, _i32p, C.c_int, C.c_int32, C.c_int32]
        L.orc_johnson_two_machine.restype = C.c_int32
        L.orc_lb_one_machine.argtypes = [C.c_int, C.c_int, _i32p, _u64p, _i32p]
        L.orc_lb_one_machine.restype = C.c_int32
        L.orc_lb_machine_pair.argtypes = [C.c_int, C.c_int, _i32p, _u64p, _i32p, C.c_int, C.c_int]
        L.orc_lb_machine_pair.restype = C.c_int32
        L.orc_lower_bound.argtypes = [C.c_int, C.c_int, _i32p, _u64p, _i32p, C.c_int]
        L.orc_lower_bound.restype = C.c_int32
        L.orc_evaluate_batch.argtypes = [C.c_int, C.c_int, _i32p, C.c_int64, _u64p, _i32p, _i32p,
                                         _i32p]
        L.orc_node_from_prefix.argtypes = [C.c_int, C.c_int, _i32p, _i32p, C.c_int, _u64p, _i32p]
        L.orc_branch.argtypes = [C.c_int, C.c_int, _i32p, _i32p, C.c_int, _i32p, _u64p, _i32p,
                                 _i32p]
        L.orc_branch.restype = C.c_int
        L.orc_solve.argtypes = [C.c_int, C.c_int, _i32p, C.c_int32, _i64p, C.c_int, C.c_int64,
                                C.POINTER(Result), _i32p, C.c_void_p, C.c_int64]
        L.orc_resolve.argtypes = [C.c_int, C.c_int, _i32p, C.c_int32, C.c_int64, _i32p, _i32p,
                                  _i64p, C.c_int, C.c_int64, C.POINTER(Result), C.c_void_p,
                                  C.c_int64]

    # -- instance ---------------------------------------------------------------------------
    def generate_instance(self, n, m, seed):
        p = np.zeros(n * m, np.int32)
        if self.lib.orc_generate_instance(n, m, seed, p) != 0:
            raise ValueError("Taillard seed must be in (0, 2^31-1)")
        return p.reshape(n, m)

    def tails(self, p):
        n, m = p.shape
        t = np.zeros(n * m, np.int32)
        self.lib.orc_tails(n, m, np.ascontiguousarray(p, np.int32).ravel(), t)
        return t.reshape(n, m)

    def child_heads(self, p, heads, job):
        n, m = p.shape
        out = np.zeros(m, np.int32)
        self.lib.orc_child_heads(n, m, np.ascontiguousarray(p, np.int32).ravel(),
                                 np.ascontiguousarray(heads, np.int32), job, out)
        return out

    def makespan(self, p, perm):
        n, m = p.shape
        perm = np.ascontiguousarray(perm, np.int32)
        return int(self.lib.orc_makespan(n, m, np.ascontiguousarray(p, np.int32).ravel(), perm,
                                         len(perm)))

    # -- bound ------------------------------------------------------------------------------
    def johnson(self, jobs, ra, rb):
        jobs = np.asarray(jobs, np.int32).reshape(-1, 3)
        a, lag, b = (np.ascontiguousarray(jobs[:, i]) for i in range(3))
        return int(self.lib.orc_johnson_two_machine(a, lag, b, len(jobs), ra, rb))

    def node(self, p, prefix):
        n, m = p.shape
        mask = np.zeros(nwords(n), np.uint64)
        heads = np.zeros(m, np.int32)
        pre = np.zeros(max(n, 1), np.int32)
        pre[: len(prefix)] = prefix
        self.lib.orc_node_from_prefix(n, m, np.ascontiguousarray(p, np.int32).ravel(), pre,
                                      len(prefix), mask, heads)
        return mask, heads

    def nodes(self, p, prefixes, depths):
        """Batch of nodes (SoA) from padded prefixes (count x n) and depths."""
        n, m = p.shape
        cnt = len(depths)
        masks = np.zeros((cnt, nwords(n)), np.uint64)
        heads = np.zeros((cnt, m), np.int32)
        pf = np.ascontiguousarray(p, np.int32).ravel()
        for i in range(cnt):
            mk = np.zeros(nwords(n), np.uint64)
            hd = np.zeros(m, np.int32)
            self.lib.orc_node_from_prefix(n, m, pf, np.ascontiguousarray(prefixes[i], np.int32),
                                          int(depths[i]), mk, hd)
            masks[i] = mk
            heads[i] = hd
        return masks, heads

    def lb_one_machine(self, p, prefix):
        n, m = p.shape
        mask, heads = self.node(p, prefix)
        return int(self.lib.orc_lb_one_machine(n, m, np.ascontiguousarray(p, np.int32).ravel(),
                                               mask, heads))

    def lb_machine_pair(self, p, prefix, k, l):
        n, m = p.shape
        mask, heads = self.node(p, prefix)
        return int(self.lib.orc_lb_machine_pair(n, m, np.ascontiguousarray(p, np.int32).ravel(),
                                                mask, heads, k, l))

    def lower_bound(self, p, prefix):
        n, m = p.shape
        mask, heads = self.node(p, prefix)
        return int(self.lib.orc_lower_bound(n, m, np.ascontiguousarray(p, np.int32).ravel(),
                                            mask, heads, len(prefix)))

    def evaluate_batch(self, p, masks, heads, depth):
        n, m = p.shape
        cnt = len(depth)
        out = np.zeros(cnt, np.int32)
        self.lib.orc_evaluate_batch(n, m, np.ascontiguousarray(p, np.int32).ravel(), cnt,
                                    np.ascontiguousarray(masks, np.uint64).ravel(),
                                    np.ascontiguousarray(heads, np.int32).ravel(),
                                    np.ascontiguousarray(depth, np.int32), out)
        return out

    def branch(self, p, prefix):
        n, m = p.shape
        pre = np.zeros(n, np.int32)
        pre[: len(prefix)] = prefix
        cp = np.zeros(n * n, np.int32)
        cm = np.zeros(n * nwords(n), np.uint64)
        ch = np.zeros(n * m, np.int32)
        cd = np.zeros(n, np.int32)
        c = self.lib.orc_branch(n, m, np.ascontiguousarray(p, np.int32).ravel(), pre, len(prefix),
                                cp, cm, ch, cd)
        if c < 0:
            raise RuntimeError("cannot branch a complete node")
        cp = cp.reshape(n, n)
        return [list(cp[i, : cd[i]]) for i in range(c)], ch.reshape(n, m)[:c].copy()

    # -- explorer ---------------------------------------------------------------------------
    def solve(self, p, initial_ub=-1, targets=(1,), budget=0, max_trace=0):
        n, m = p.shape
        t, nt = _targets(targets)
        res = Result()
        sched = np.zeros(n, np.int32)
        trace = (Round * max_trace)() if max_trace else None
        self.lib.orc_solve(n, m, np.ascontiguousarray(p, np.int32).ravel(), initial_ub, t, nt,
                           budget, C.byref(res), sched,
                           C.cast(trace, C.c_void_p) if trace is not None else None, max_trace)
        rounds = [trace[i].as_tuple() for i in range(min(res.rounds, max_trace))] if trace else []
        return res.as_dict(), ([int(x) for x in sched] if res.found else None), rounds

    def resolve(self, p, ub, roots, targets=(1,), budget=0, max_trace=0):
        n, m = p.shape
        pre, dep = pack_prefixes(n, roots)
        t, nt = _targets(targets)
        res = Result()
        trace = (Round * max_trace)() if max_trace else None
        self.lib.orc_resolve(n, m, np.ascontiguousarray(p, np.int32).ravel(), ub, len(roots), pre,
                             dep, t, nt, budget, C.byref(res),
                             C.cast(trace, C.c_void_p) if trace is not None else None, max_trace)
        rounds = [trace[i].as_tuple() for i in range(min(res.rounds, max_trace))] if trace else []
        return res.as_dict(), rounds


def pack_prefixes(n, prefixes):
    """Padded prefixes (cnt x n, -1 filled) and depths; never zero-sized for ctypes."""
    cnt = len(prefixes)
    pre = np.full((max(cnt, 1), max(n, 1)), -1, np.int32)
    dep = np.zeros(max(cnt, 1), np.int32)
    for i, pr in enumerate(prefixes):
        pre[i, : len(pr)] = pr
        dep[i] = len(pr)
    return np.ascontiguousarray(pre.ravel()), dep


class Ref:
    """The reference headers compiled in place (oracle/_ref)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            if os.path.isdir(REF_SRC):
                build(ref=True)
            else:
                raise FileNotFoundError(f"{path} (reference not compiled on this host)")
        L = self.lib = C.CDLL(path)
        L.ref_generate_instance.argtypes = [C.c_int, C.c_int, C.c_int32, _i32p]
        L.ref_random_instance.argtypes = [C.c_uint32, C.c_int, C.c_int, C.c_int, C.c_int, _i32p]
        L.ref_random_nodes.argtypes = [C.c_int, C.c_int, _i32p, C.c_uint32, C.c_int64, _i32p,
                                       _i32p]
        L.ref_evaluate.argtypes = [C.c_int, C.c_int, _i32p, C.c_int64, _i32p, _i32p, C.c_int,
                                   _i32p, _i32p]
        L.ref_lb_one_machine.argtypes = [C.c_int, C.c_int, _i32p, _i32p, C.c_int]
        L.ref_lb_one_machine.restype = C.c_int32
        L.ref_lb_machine_pair.argtypes = [C.c_int, C.c_int, _i32p, _i32p, C.c_int, C.c_int,
                                          C.c_int]
        L.ref_lb_machine_pair.restype = C.c_int32
        L.ref_johnson.argtypes = [_i32p, _i32p, _i32p, C.c_int, C.c_int32, C.c_int32]
        L.ref_johnson.restype = C.c_int32
        L.ref_branch.argtypes = [C.c_int, C.c_int, _i32p, _i32p, C.c_int, _i32p, _i32p, _i32p]
        L.ref_resolve.argtypes = [C.c_int, C.c_int, _i32p, C.c_int32, C.c_int64, _i32p, _i32p,
                                  _i64p, C.c_int, C.c_int64, C.c_int, C.POINTER(Result),
                                  C.c_void_p, C.c_int64, C.POINTER(C.c_double)]
        L.ref_resolve_drain.argtypes = [C.c_int, C.c_int, _i32p, C.c_int32, C.c_int64, _i32p,
                                        _i32p, _i64p, C.c_int, C.c_int64, C.c_int,
                                        C.POINTER(Result), C.c_int64, _i32p, _i32p,
                                        C.POINTER(C.c_int64)]
        L.ref_solve_trace.argtypes = [C.c_int, C.c_int, _i32p, C.c_int32, _i64p, C.c_int,
                                      C.c_int64, C.c_int, C.POINTER(Result), _i32p, C.c_void_p,
                                      C.c_int64]
        L.ref_solve.argtypes = [C.c_int, C.c_int, _i32p, C.c_int32, C.c_int, C.c_int,
                                C.POINTER(C.c_int32), C.POINTER(C.c_int32), _i32p, _i64p]
        L.ref_brute_force.argtypes = [C.c_int, C.c_int, _i32p, C.POINTER(C.c_int32), _i32p]
        L.ref_detect_units.restype = C.c_int
        L.ref_bench_rounds.argtypes = [C.c_int, C.c_int, _i32p, C.c_int32, C.c_int64, C.c_int,
                                       C.c_int, C.c_int, C.POINTER(C.c_int64), C.c_void_p,
                                       np.ctypeslib.ndpointer(dtype=np.float64,
                                                              flags="C_CONTIGUOUS"),
                                       C.c_double, C.POINTER(C.c_int)]

    def bench_rounds(self, p, ub, target, warm, steps, backends, max_seconds=0.0):
        """Prefill-until-full, `warm` untimed rounds, up to `steps` timed rounds of the
        reference resolve loop (stopping once `max_seconds` > 0 of them have elapsed);
        returns (prefill_rounds, [round tuples], [seconds])."""
        n, m = p.shape
        pre = C.c_int64(0)
        done = C.c_int(0)
        trace = (Round * max(steps, 1))()
        secs = np.zeros(max(steps, 1), np.float64)
        rc = self.lib.ref_bench_rounds(n, m, np.ascontiguousarray(p, np.int32).ravel(), ub, target,
                                       warm, steps, backends, C.byref(pre),
                                       C.cast(trace, C.c_void_p), secs, float(max_seconds),
                                       C.byref(done))
        if rc != 0:
            raise RuntimeError("ref_bench_rounds failed")
        k = done.value
        return pre.value, [trace[i].as_tuple() for i in range(k)], list(secs[:k])

    def detect_units(self):
        return int(self.lib.ref_detect_units())

    def workload_text(self, p, ub, nodes, seed):
        """The reference's save_workload(generate_workload(inst, ub, by_nodes(nodes), seed))."""
        n, m = p.shape
        buf = C.create_string_buffer(1 << 24)
        self.lib.ref_workload_text.argtypes = [C.c_int, C.c_int, _i32p, C.c_int32, C.c_int64,
                                               C.c_uint32, C.c_char_p, C.c_int64]
        self.lib.ref_workload_text.restype = C.c_int64
        k = self.lib.ref_workload_text(n, m, np.ascontiguousarray(p, np.int32).ravel(), ub, nodes,
                                       seed, buf, 1 << 24)
        if k < 0:
            raise RuntimeError("ref_workload_text failed")
        return buf.raw[:k].decode()

    def tuner_trace(self, grain, units, max_batch, window, probes, peak):
        """The reference Tuner's trace lines ("window batch decision") on the synthetic
        curve x / (1 + (x / peak)^2), driven until fixed (ref_tuner_trace)."""
        buf = C.create_string_buffer(1 << 16)
        self.lib.ref_tuner_trace.argtypes = [C.c_int] * 5 + [C.c_double, C.c_char_p, C.c_int64]
        k = self.lib.ref_tuner_trace(grain, units, max_batch, window, probes, peak, buf, 1 << 16)
        if k < 0:
            raise RuntimeError("ref_tuner_trace failed")
        return buf.value.decode().splitlines()

    def generate_instance(self, n, m, seed):
        p = np.zeros(n * m, np.int32)
        if self.lib.ref_generate_instance(n, m, seed, p) != 0:
            raise ValueError("bad seed")
        return p.reshape(n, m)

    def random_instance(self, seed, n, m, low=1, high=99):
        p = np.zeros(n * m, np.int32)
        self.lib.ref_random_instance(seed, n, m, low, high, p)
        return p.reshape(n, m)

    def random_nodes(self, p, seed, count):
        n, m = p.shape
        pre = np.zeros(count * n, np.int32)
        dep = np.zeros(count, np.int32)
        self.lib.ref_random_nodes(n, m, np.ascontiguousarray(p, np.int32).ravel(), seed, count,
                                  pre, dep)
        pre = pre.reshape(count, n)
        return [list(pre[i, : dep[i]]) for i in range(count)]

    def evaluate(self, p, prefixes, backends=1):
        n, m = p.shape
        pre, dep = pack_prefixes(n, prefixes)
        cnt = len(prefixes)
        lb = np.zeros(max(cnt, 1), np.int32)
        hd = np.zeros(max(cnt, 1) * m, np.int32)
        rc = self.lib.ref_evaluate(n, m, np.ascontiguousarray(p, np.int32).ravel(), cnt, pre, dep,
                                   backends, lb, hd)
        if rc != 0:
            raise RuntimeError("ref_evaluate failed")
        return lb[:cnt].copy(), hd.reshape(-1, m)[:cnt].copy()

    def lb_one_machine(self, p, prefix):
        n, m = p.shape
        pre = np.zeros(n, np.int32)
        pre[: len(prefix)] = prefix
        return int(self.lib.ref_lb_one_machine(n, m, np.ascontiguousarray(p, np.int32).ravel(),
                                               pre, len(prefix)))

    def lb_machine_pair(self, p, prefix, k, l):
        n, m = p.shape
        pre = np.zeros(n, np.int32)
        pre[: len(prefix)] = prefix
        return int(self.lib.ref_lb_machine_pair(n, m, np.ascontiguousarray(p, np.int32).ravel(),
                                                pre, len(prefix), k, l))

    def johnson(self, jobs, ra, rb):
        jobs = np.asarray(jobs, np.int32).reshape(-1, 3)
        a, lag, b = (np.ascontiguousarray(jobs[:, i]) for i in range(3))
        return int(self.lib.ref_johnson(a, lag, b, len(jobs), ra, rb))

    def branch(self, p, prefix):
        n, m = p.shape
        pre = np.zeros(n, np.int32)
        pre[: len(prefix)] = prefix
        cp = np.zeros(n * n, np.int32)
        cd = np.zeros(n, np.int32)
        ch = np.zeros(n * m, np.int32)
        c = self.lib.ref_branch(n, m, np.ascontiguousarray(p, np.int32).ravel(), pre, len(prefix),
                                cp, cd, ch)
        if c < 0:
            raise RuntimeError("cannot branch a complete node")
        cp = cp.reshape(n, n)
        return [list(cp[i, : cd[i]]) for i in range(c)], ch.reshape(n, m)[:c].copy()

    def resolve(self, p, ub, roots, targets=(1,), budget=0, backends=1, max_trace=0):
        n, m = p.shape
        pre, dep = pack_prefixes(n, roots)
        t, nt = _targets(targets)
        res = Result()
        secs = C.c_double(0)
        trace = (Round * max_trace)() if max_trace else None
        rc = self.lib.ref_resolve(n, m, np.ascontiguousarray(p, np.int32).ravel(), ub, len(roots),
                                  pre, dep, t, nt, budget, backends, C.byref(res),
                                  C.cast(trace, C.c_void_p) if trace is not None else None,
                                  max_trace, C.byref(secs))
        if rc != 0:
            raise RuntimeError("ref_resolve failed")
        rounds = [trace[i].as_tuple() for i in range(min(res.rounds, max_trace))] if trace else []
        return res.as_dict(), rounds, secs.value

    def resolve_drain(self, p, ub, roots, targets=(1,), budget=0, backends=1, cap=1 << 22):
        """resolve() stopped by `budget`, then PendingTree::drain (pending.hpp:41-50) of what
        is left: (result dict, [prefix of every pending node, drain order])."""
        n, m = p.shape
        pre, dep = pack_prefixes(n, roots)
        t, nt = _targets(targets)
        res = Result()
        dp = np.zeros(cap * n, np.int32)
        dd = np.zeros(cap, np.int32)
        cnt = C.c_int64(0)
        rc = self.lib.ref_resolve_drain(n, m, np.ascontiguousarray(p, np.int32).ravel(), ub,
                                        len(roots), pre, dep, t, nt, budget, backends,
                                        C.byref(res), cap, dp, dd, C.byref(cnt))
        if rc != 0:
            raise RuntimeError(f"ref_resolve_drain failed ({rc}, pending {cnt.value})")
        dp = dp.reshape(cap, n)
        return res.as_dict(), [list(map(int, dp[i, : dd[i]])) for i in range(cnt.value)]

    def solve_trace(self, p, initial_ub=-1, targets=(1,), budget=0, backends=1, max_trace=0):
        n, m = p.shape
        t, nt = _targets(targets)
        res = Result()
        sched = np.zeros(n, np.int32)
        trace = (Round * max_trace)() if max_trace else None
        rc = self.lib.ref_solve_trace(n, m, np.ascontiguousarray(p, np.int32).ravel(), initial_ub,
                                      t, nt, budget, backends, C.byref(res), sched,
                                      C.cast(trace, C.c_void_p) if trace is not None else None,
                                      max_trace)
        if rc != 0:
            raise RuntimeError("ref_solve_trace failed")
        rounds = [trace[i].as_tuple() for i in range(min(res.rounds, max_trace))] if trace else []
        return res.as_dict(), ([int(x) for x in sched] if res.found else None), rounds

    def solve(self, p, initial_ub=-1, fixed_batch=1, backends=1):
        n, m = p.shape
        opt = C.c_int32()
        found = C.c_int32()
        sched = np.zeros(n, np.int32)
        stats = np.zeros(3, np.int64)
        rc = self.lib.ref_solve(n, m, np.ascontiguousarray(p, np.int32).ravel(), initial_ub,
                                fixed_batch, backends, C.byref(opt), C.byref(found), sched, stats)
        if rc != 0:
            raise RuntimeError("ref_solve failed")
        return opt.value, ([int(x) for x in sched] if found.value else None), tuple(int(x) for x in stats)

    def brute_force(self, p):
        n, m = p.shape
        opt = C.c_int32()
        sched = np.zeros(n, np.int32)
        if self.lib.ref_brute_force(n, m, np.ascontiguousarray(p, np.int32).ravel(),
                                    C.byref(opt), sched) != 0:
            raise ValueError("brute_force refuses instances with more than 10 jobs")
        return opt.value, [int(x) for x in sched]
