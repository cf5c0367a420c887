"""Generates tests/golden/traces_large.json: per-round traces of the REFERENCE explorer
(oracle/_ref = the reference headers compiled in place, resolve_workload loop of
bench.hpp:63-114 with a frozen UB) at >= 1 M bounded nodes for the 50x20, 100x20 and
200x20 Taillard instances, with fixed and tuner-shaped (doubling, then fixed) target
schedules.  TEST INFRASTRUCTURE; run here (where /root/reference exists):

    python tests/golden/make_traces_large.py
"""
from __future__ import annotations

import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

from make_golden import FROZEN_UB, TAILLARD  # noqa: E402
from oracle import Ref  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "traces_large.json")


def main():
    ref = Ref()
    nthreads = os.cpu_count() or 1
    out = {"resolve": []}
    t_start = time.time()

    def add(name, targets, budget):
        n, m, seed = TAILLARD[name]
        p = ref.generate_instance(n, m, seed)
        t0 = time.time()
        res, rounds, _ = ref.resolve(p, FROZEN_UB[name], [[]], targets=targets, budget=budget,
                                     backends=nthreads, max_trace=1 << 16)
        out["resolve"].append({"instance": name, "ub": FROZEN_UB[name], "targets": list(targets),
                               "budget": budget, "roots": [[]], "result": res, "rounds": rounds})
        print(name, targets[:3], budget, res["bounded"], len(rounds), round(time.time() - t0, 1),
              flush=True)

    # fixed pools (config 3/4/5 instances)
    add("ta051", [65536], 1_000_000)
    add("ta081", [131072], 1_000_000)
    add("ta101", [262144], 1_000_000)
    # tuner-shaped: doubling from grain x units of the B200 descriptor, then fixed (config 3)
    add("ta051", [37888] * 3 + [75776] * 3 + [151552] * 3 + [303104] * 3 + [151552], 1_500_000)
    with open(OUT, "w") as f:
        json.dump(out, f, separators=(",", ":"))
    print("done", round(time.time() - t_start, 1), "s")


if __name__ == "__main__":
    main()
