"""Table of scripts/batch_sweep.py lines (stdin)."""
import json
import sys

print("| target | planner | us/round wall | us/round device | us K2 | device M/s | wall M/s |")
print("|---|---|---|---|---|---|---|")
for line in sys.stdin:
    try:
        d = json.loads(line)
    except Exception:
        print(line.strip())
        continue
    print(f"| {d['target']} | {d['planner']} | {d['us_per_round_wall']:.1f} | {d['us_per_round_device']:.1f} | "
          f"{d.get('us_per_round_k2', 0):.1f} | {d['device_rate'] / 1e6:.1f} | {d['wall_rate'] / 1e6:.1f} |")
