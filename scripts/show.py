"""Prints the key fields of bench JSON lines (gpurun_out/*.json)."""
import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.load(open(f))
    except Exception as e:  # noqa: BLE001
        print(f, "unreadable:", e)
        continue
    e2e = (d.get("e2e") or {}).get("value") or 0.0
    rf = d.get("roofline") or {}
    print(f"{f}: value {d['value']/1e6:.1f} M/s  ms/step {d['ms_per_step']:.4f}  "
          f"wall {d.get('wall_value', 0)/1e6:.1f} M/s  e2e {e2e/1e6:.1f}  "
          f"frac {rf.get('frac', 0):.3f} k2share {rf.get('k2_share_of_round', 0):.3f}")
    if "wall_breakdown_ms_per_step" in d:
        print("   ", {k: round(v, 4) for k, v in d["wall_breakdown_ms_per_step"].items()})
