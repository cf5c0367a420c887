"""Steady-state per-round split, device-resident vs host-resident pending tree
(the bench's value vs e2e legs): wall, library host time, sync wait, device round,
K2, bytes over the host link.  Usage: python scripts/diag_e2e.py [ta021|ta081|...] [target]"""
import os
import statistics as st
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1206_4973_b200 as fbb

INST = {"ta021": (20, 20, 479340445, 2297), "ta081": (100, 20, 450926852, 6202),
        "ta051": (50, 20, 1539989115, 3847), "ta101": (200, 20, 2013025619, 11195),
        "ta001": (20, 5, 873654221, 1279)}
name = sys.argv[1] if len(sys.argv) > 1 else "ta021"
T = int(sys.argv[2]) if len(sys.argv) > 2 else 262144
n, m, seed, ub = INST[name]
inst = fbb.generate_instance(n, m, seed)
ctx = fbb.Context(inst, 0)
ctx.explorer_reset(fbb.NodeBatch.root(inst), ub, frozen=True)
for _ in range(32):
    r = ctx.explorer_run([T], 1)
    if r[0][2] >= T:
        break
snap = fbb.nodes_from_prefixes(inst, ctx.explorer_pending())
for host in (False, True):
    ctx.explorer_set_residency(host)
    ctx.explorer_reset(snap, ub, frozen=True)
    ctx.explorer_run([T] * 5, 5)  # warm
    w0 = time.perf_counter()
    r, t = ctx.explorer_run([T] * 100, 100, timing=True)
    wall = (time.perf_counter() - w0) * 1e3 / len(r)
    bounded = sum(x[2] for x in r) / len(r)
    f = {k: st.mean(x[k] for x in t) for k in t[0]}
    print(f"{'host' if host else 'dev '} wall/round {wall:.3f} ms  {bounded / wall / 1e6:.3f} G/s  " +
          "  ".join(f"{k} {v:.3f}" if isinstance(v, float) else f"{k} {v:.0f}" for k, v in f.items()),
          flush=True)
