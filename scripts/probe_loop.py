import os, sys
sys.path.insert(0, os.getcwd())
import paper_1206_4973_b200 as fbb
inst = fbb.generate_instance(20, 20, 479340445)
ctx = fbb.Context(inst, 0)
print(ctx.kernels())
ctx.explorer_reset(fbb.NodeBatch.root(inst), 2297, frozen=True)
for _ in range(10):
    r = ctx.explorer_run([4096], 1)
r, t = ctx.explorer_run([4096], 32, timing=True)
print(len(r), sum(x["round_ms"] for x in t) / len(t) * 1e3, sum(x["k2_ms"] for x in t) / len(t) * 1e3)
lead = sum(x["place_ms"] for x in t) / len(t) * 1e3
print("us/round: total %.1f lead-in %.1f K2 %.1f" % (sum(x["round_ms"] for x in t) / len(t) * 1e3, lead,
      sum(x["k2_ms"] for x in t) / len(t) * 1e3))
for T in (16384, 262144):
    r, t = ctx.explorer_run([T], 32, timing=True)
    print(T, "us/round: total %.1f lead-in %.1f K2 %.1f" % (sum(x["round_ms"] for x in t) / len(t) * 1e3,
          sum(x["place_ms"] for x in t) / len(t) * 1e3, sum(x["k2_ms"] for x in t) / len(t) * 1e3))
