"""Diagnostics: run the solve traces one by one; time explorer rounds (wall vs device)."""
import json
import sys
import time

sys.path.insert(0, ".")
import numpy as np

import paper_1206_4973_b200 as fbb

mode = sys.argv[1]
if mode == "solve":
    tr = json.load(open("tests/golden/traces.json"))
    ins = json.load(open("tests/golden/instances.json"))
    for t in tr["solve"]:
        d = ins[t["instance"]]
        inst = fbb.Instance(d["n"], d["m"], d["p"])
        ub = None if t["initial_ub"] < 0 else t["initial_ub"]
        print("solve", t["instance"], ub, t["targets"], flush=True)
        sol = fbb.solve(inst, ub, targets=t["targets"], budget=t["budget"])
        gold = [tuple(r) for r in t["rounds"]]
        print(" rounds ok" if sol.rounds == gold else f" MISMATCH at {next(i for i,(a,b) in enumerate(zip(sol.rounds, gold)) if a!=b)}", flush=True)
elif mode == "timing":
    import torch
    inst = fbb.generate_instance(20, 20, 479340445)
    ctx = fbb.Context(inst)
    ctx.explorer_reset(fbb.NodeBatch.root(inst), 2297, True)
    for _ in range(8):
        ctx.explorer_run([262144], 1)
    torch.cuda.synchronize()
    for k in range(3):
        t0 = time.perf_counter()
        r, tm = ctx.explorer_run([262144], 10, timing=True)
        el = time.perf_counter() - t0
        print(f"10 rounds in one call: wall {el*1e3/10:.3f} ms/round, device {sum(x['round_ms'] for x in tm)/10:.3f} ms/round, k2 {sum(x['k2_ms'] for x in tm)/10:.3f}", flush=True)
    for k in range(3):
        t0 = time.perf_counter()
        for _ in range(10):
            r, tm = ctx.explorer_run([262144], 1, timing=True)
        el = time.perf_counter() - t0
        print(f"1 round per call: wall {el*1e3/10:.3f} ms/round", flush=True)

if mode == "seq":
    # the pytest order: resolve traces (budgets capped) then solve traces
    tr = json.load(open("tests/golden/traces.json"))
    ins = json.load(open("tests/golden/instances.json"))
    cap = int(sys.argv[2]) if len(sys.argv) > 2 else 100000
    for t in tr["resolve"]:
        d = ins[t["instance"]]
        inst = fbb.Instance(d["n"], d["m"], d["p"])
        print("resolve", t["instance"], t["targets"][:2], flush=True)
        res = fbb.resolve_workload(inst, t["roots"], t["ub"], targets=t["targets"], budget=min(cap, t["budget"]))
        gold = [tuple(r) for r in t["rounds"]]
        print(" ok" if res.rounds == gold[:len(res.rounds)] else " MISMATCH", flush=True)
    for t in tr["solve"]:
        d = ins[t["instance"]]
        inst = fbb.Instance(d["n"], d["m"], d["p"])
        ub = None if t["initial_ub"] < 0 else t["initial_ub"]
        print("solve", t["instance"], ub, t["targets"], flush=True)
        sol = fbb.solve(inst, ub, targets=t["targets"], budget=min(cap, t["budget"]))
        gold = [tuple(r) for r in t["rounds"]]
        print(" ok" if sol.rounds == gold[:len(sol.rounds)] else " MISMATCH", flush=True)

if mode == "ta001":
    tr = json.load(open("tests/golden/traces.json"))
    ins = json.load(open("tests/golden/instances.json"))
    for kind in ("resolve", "solve"):
        for t in tr[kind]:
            if t["instance"] not in ("ta001",):
                continue
            d = ins[t["instance"]]
            inst = fbb.Instance(d["n"], d["m"], d["p"])
            print(kind, t["instance"], t["targets"][:2], flush=True)
            if kind == "resolve":
                res = fbb.resolve_workload(inst, t["roots"], t["ub"], targets=t["targets"], budget=t["budget"])
                rounds = res.rounds
            else:
                ub = None if t["initial_ub"] < 0 else t["initial_ub"]
                rounds = fbb.solve(inst, ub, targets=t["targets"], budget=t["budget"]).rounds
            gold = [tuple(r) for r in t["rounds"]]
            print(" ok" if rounds == gold else " MISMATCH", flush=True)
