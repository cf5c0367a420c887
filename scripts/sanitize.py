"""Small workloads for compute-sanitizer (memcheck / racecheck / synccheck): every kernel
path -- K1 v1/v2, K2 v2 (both occupancies), v3, generic, leaves, place, the explorer
with its tree in HBM and in host memory, the device-planned loop (graph batches and the
persistent batch kernel) -- on inputs
small enough for the sanitizer, each checked against the oracle."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_1206_4973_b200 as fbb
from oracle import Oracle

orc = Oracle()
rng = np.random.default_rng(1)
for n, m in [(20, 20), (20, 5), (50, 20), (100, 20), (12, 7)]:
    p = rng.integers(1, 100, size=(n, m)).astype(np.int32)
    inst = fbb.Instance(n, m, p)
    ctx = fbb.Context(inst)
    pre = [list(rng.permutation(n)[: rng.integers(0, n + 1)]) for _ in range(64)]
    nodes = fbb.nodes_from_prefixes(inst, pre)
    assert np.array_equal(ctx.bound(nodes), orc.evaluate_batch(p, nodes.masks, nodes.heads, nodes.depth))
    par = sorted([list(rng.permutation(n)[: rng.integers(0, n - 2)]) for _ in range(24)], key=len,
                 reverse=True)
    surv, slb, *_ = ctx.expand_bound_prune(fbb.nodes_from_prefixes(inst, par), 10**6, frozen=True)
    # tree in HBM, in host memory (compact prefix rows at n <= 32), and host full rows;
    # deep enough at n <= 20 to reach the leaf kernels
    for mode in ("hbm", "host", "host_full"):
        os.environ["FBB_HOST_ROWS"] = "full" if mode == "host_full" else "compact"
        ctx.explorer_set_residency(mode != "hbm")
        ctx.explorer_reset(fbb.NodeBatch.root(inst), 10**6, frozen=True)
        ctx.explorer_run([2048], n + 2 if n <= 20 else 3)
    ctx.close()
    # direct placement (single-wave pools: K2 grid-wide count + direct bucket writes) and the
    # device-planned graph batches, in solve mode (leaf rounds, incumbent updates)
    # (FBB_PERSIST: the persistent batch kernel -- one cooperative launch per batch, grid
    # barriers between the rounds -- or the conditional-graph batch)
    for dl, ps in (("0", "1"), ("1", "1"), ("1", "0")):
        os.environ["FBB_DEVICE_LOOP"] = dl
        os.environ["FBB_PERSIST"] = ps
        ctx = fbb.Context(inst)
        ctx.explorer_set_residency(False)
        ctx.explorer_start_solve(None)
        ctx.explorer_run([256, 1024], 12)
        ctx.close()
    os.environ["FBB_DEVICE_LOOP"] = "0"
    print("ok", n, m, flush=True)
# the in-library multi-device group (two members on one device)
inst = fbb.generate_instance(12, 6, 123)
grp = fbb.DeviceGroup(inst, [0, 0])
grp.reset(fbb.NodeBatch.root(inst), 10**6, frozen=True)
grp.run(512, max_steps=3, rounds_per_step=2)
grp.close()
print("ok group", flush=True)
