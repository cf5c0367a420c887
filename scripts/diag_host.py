"""Per-round timing of the host-resident explorer vs the device-resident one."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1206_4973_b200 as fbb

INST = {"ta021": (20, 20, 479340445, 2297), "ta081": (100, 20, 450926852, 6202),
        "ta051": (50, 20, 1539989115, 3847)}
n, m, seed, ub = INST[sys.argv[1] if len(sys.argv) > 1 else "ta021"]
inst = fbb.generate_instance(n, m, seed)
ctx = fbb.Context(inst, 0)
T = 262144
ctx.explorer_reset(fbb.NodeBatch.root(inst), ub, frozen=True)
for _ in range(16):
    r = ctx.explorer_run([T], 1)
    if r[0][2] >= T:
        break
snap = fbb.nodes_from_prefixes(inst, ctx.explorer_pending())
for host in (False, True):
    ctx.explorer_set_residency(host)
    ctx.explorer_reset(snap, ub, frozen=True)
    out = []
    for i in range(6):
        w0 = time.perf_counter()
        r, t = ctx.explorer_run([T], 1, timing=True)
        w = time.perf_counter() - w0
        out.append((round(1e3 * w, 3), round(t[0]["host_ms"], 3), round(t[0]["sync_ms"], 3),
                    round(t[0]["round_ms"], 3), round(t[0]["k2_ms"], 3), t[0]["h2d_bytes"],
                    t[0]["d2h_bytes"], r[0][3]))
    print("host" if host else "dev ", out, flush=True)
