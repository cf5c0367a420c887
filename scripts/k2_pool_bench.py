"""Times K2 on one fixed pool (Ta021 frontier, pop order) through fbb_expand_bound_prune."""
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import numpy as np

import paper_1206_4973_b200 as fbb

INST = {"ta021": (20, 20, 479340445, 2297), "ta081": (100, 20, 450926852, 6202),
        "ta051": (50, 20, 1539989115, 3847), "ta101": (200, 20, 2013025619, 11195)}
n, m, seed, UB = INST[os.environ.get("FBB_POOL_INSTANCE", "ta021")]
inst = fbb.generate_instance(n, m, seed)
ctx = fbb.Context(inst, 0)
ctx.explorer_reset(fbb.NodeBatch.root(inst), UB, frozen=True)
for _ in range(5):
    ctx.explorer_run([262144], 1)
pend = ctx.explorer_pending()               # drain order: shallow first
pop = sorted(pend, key=len, reverse=True)   # deepest first
kids, par = 0, []
for pr in pop:
    par.append(pr)
    kids += n - len(pr)
    if kids >= 262144:
        break
parents = fbb.nodes_from_prefixes(inst, par)
for i in range(int(sys.argv[1]) if len(sys.argv) > 1 else 5):
    t0 = time.perf_counter()
    surv, slb, *_ , rec = ctx.expand_bound_prune(parents, UB, frozen=True)
    print(len(par), kids, len(surv),
          "%.3f ms" % (1e3 * (time.perf_counter() - t0)))
