"""Times K2 on one fixed pool (Ta021 frontier, pop order) through fbb_expand_bound_prune."""
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import numpy as np

import paper_1206_4973_b200 as fbb

inst = fbb.generate_instance(20, 20, 479340445)
ctx = fbb.Context(inst, 0)
ctx.explorer_reset(fbb.NodeBatch.root(inst), 2297, frozen=True)
for _ in range(5):
    ctx.explorer_run([262144], 1)
pend = ctx.explorer_pending()               # drain order: shallow first
pop = sorted(pend, key=len, reverse=True)   # deepest first
kids, par = 0, []
for pr in pop:
    par.append(pr)
    kids += 20 - len(pr)
    if kids >= 262144:
        break
parents = fbb.nodes_from_prefixes(inst, par)
for i in range(int(sys.argv[1]) if len(sys.argv) > 1 else 5):
    t0 = time.perf_counter()
    surv, slb, *_ , rec = ctx.expand_bound_prune(parents, 2297, frozen=True)
    print(len(par), kids, len(surv),
          "%.3f ms" % (1e3 * (time.perf_counter() - t0)))
