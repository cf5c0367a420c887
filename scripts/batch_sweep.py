"""Ta021 pool-size sweep (BASELINE configs[1]) in the way an explorer call runs in the
paper's regime: K rounds per fbb_explorer_run call.  Two planners side by side:
host-planned (FBB_DEVICE_LOOP=0: one stream sync per round) and device-planned
(FBB_DEVICE_LOOP=1: the batch is one conditional-WHILE CUDA graph).  A step = one call of
B rounds, L2 flushed between steps (untimed); rate = bounded nodes / wall clock of the
calls (host->device state upload, the rounds, the summary download included), plus the
device-only rate from the rounds' own timings.  Prints one JSON line per (target, planner).

usage: python scripts/batch_sweep.py [targets...]   (env BATCH=rounds per call, STEPS,
PLANNERS=01 / 0 / 1)"""
import json
import os
import sys
import time

sys.path.insert(0, os.getcwd())

import torch

TARGETS = [int(x) for x in sys.argv[1:]] or [4096, 8192, 16384, 32768, 65536, 131072, 262144]
B = int(os.environ.get("BATCH", "32"))
STEPS = int(os.environ.get("STEPS", "20"))


def run(T, planner):
    os.environ["FBB_DEVICE_LOOP"] = planner
    import paper_1206_4973_b200 as fbb

    inst = fbb.generate_instance(20, 20, 479340445)
    ctx = fbb.Context(inst, 0)
    ctx.explorer_reset(fbb.NodeBatch.root(inst), 2297, frozen=True)
    for _ in range(64):  # prefill until a round reaches the target
        r = ctx.explorer_run([T], 1)
        if not r or r[0][2] >= T:
            break
    for _ in range(3):
        ctx.explorer_run([T], B)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda:0")
    wall, dev, k2, bounded, rounds = 0.0, 0.0, 0.0, 0, 0
    for s in range(STEPS):
        flush.fill_(s % 7)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r, t = ctx.explorer_run([T], B, timing=True)
        wall += time.perf_counter() - t0
        dev += sum(x["round_ms"] for x in t) / 1e3
        k2 += sum(x["k2_ms"] for x in t) / 1e3
        bounded += sum(x[2] for x in r)
        rounds += len(r)
    ctx.close()
    return {"target": T, "planner": "device" if planner == "1" else "host", "rounds": rounds,
            "rounds_per_call": B, "bounded": bounded, "wall_rate": bounded / wall,
            "device_rate": bounded / dev if dev > 0 else None,
            "us_per_round_wall": 1e6 * wall / max(1, rounds),
            "us_per_round_device": 1e6 * dev / max(1, rounds),
            "us_per_round_k2": 1e6 * k2 / max(1, rounds)}


if __name__ == "__main__":
    for T in TARGETS:
        for pl in os.environ.get("PLANNERS", "01"):
            print(json.dumps(run(T, pl)), flush=True)
