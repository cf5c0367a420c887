"""Per-round timing of the host-resident explorer vs the device-resident one."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1206_4973_b200 as fbb

inst = fbb.generate_instance(20, 20, 479340445)
ctx = fbb.Context(inst, 0)
T = 262144
ctx.explorer_reset(fbb.NodeBatch.root(inst), 2297, frozen=True)
for _ in range(8):
    r = ctx.explorer_run([T], 1)
    if r[0][2] >= T:
        break
snap = fbb.nodes_from_prefixes(inst, ctx.explorer_pending())
for host in (False, True, False, True):
    ctx.explorer_set_residency(host)
    ctx.explorer_reset(snap, 2297, frozen=True)
    out = []
    for i in range(8):
        w0 = time.perf_counter()
        r, t = ctx.explorer_run([T], 1, timing=True)
        w = time.perf_counter() - w0
        out.append((round(1e3 * w, 3), round(t[0]["host_ms"], 3), round(t[0]["sync_ms"], 3),
                    round(t[0]["round_ms"], 3), t[0]["h2d_bytes"], t[0]["d2h_bytes"]))
    print("host" if host else "dev ", out, flush=True)
# raw copy speed from pinned
a = torch.empty(3 << 20, dtype=torch.uint8, pin_memory=True)
b = torch.empty(3 << 20, dtype=torch.uint8, device="cuda")
for _ in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter(); b.copy_(a); torch.cuda.synchronize()
    t1 = time.perf_counter(); a.copy_(b); torch.cuda.synchronize(); t2 = time.perf_counter()
    print("torch 3MiB H2D %.3f ms D2H %.3f ms" % (1e3 * (t1 - t0), 1e3 * (t2 - t1)))
