"""Where an e2e (host-resident tree) round's device time goes: FBB_PDL=0 gives event-timed
K2 and place (+ summary); prints per-round averages for the HBM and the host tree."""
import os
import sys

sys.path.insert(0, os.getcwd())
import paper_1206_4973_b200 as fbb

T = int(sys.argv[1]) if len(sys.argv) > 1 else 262144
inst = fbb.generate_instance(20, 20, 479340445)
for host in (False, True):
    ctx = fbb.Context(inst, 0)
    ctx.explorer_set_residency(host)
    ctx.explorer_reset(fbb.NodeBatch.root(inst), 2297, frozen=True)
    for _ in range(12):
        ctx.explorer_run([T], 1)
    tim = []
    for _ in range(40):
        r, t = ctx.explorer_run([T], 1, timing=True)
        tim += t
    k = len(tim)
    avg = lambda f: sum(x[f] for x in tim) / k * 1e3  # noqa: E731
    print(f"host={host} T={T}: round {avg('round_ms'):.1f} us  K2 {avg('k2_ms'):.1f}  place+summary "
          f"{avg('place_ms'):.1f}  h2d {sum(x['h2d_bytes'] for x in tim) // k} B  d2h "
          f"{sum(x['d2h_bytes'] for x in tim) // k} B")
    ctx.close()
