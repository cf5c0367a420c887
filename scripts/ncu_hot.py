"""Hot spots of one kernel in an ncu --set full report (--import-source): total warp
instructions, stall-sample totals by reason, and the top SASS lines by stall samples.
python scripts/ncu_hot.py REPORT [TOP]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, data = rows[1], [r for r in rows[2:] if len(r) == len(rows[1])]
ie, src, st = hdr.index("Instructions Executed"), hdr.index("Source"), \
    hdr.index("Warp Stall Sampling (All Samples)")
num = lambda s: int(s) if s.isdigit() else 0  # noqa: E731
tot_i = sum(num(r[ie]) for r in data)
tot_s = sum(num(r[st]) for r in data)
print(f"{rows[0][1][:90]}\nwarp instructions {tot_i}, stall samples {tot_s}")
cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
sums = sorted(((sum(num(r[i]) for r in data), hdr[i]) for i in cols), reverse=True)
print("stalls:", ", ".join(f"{h[6:]} {100.0 * v / max(tot_s, 1):.1f}%" for v, h in sums[:8]))
for r in sorted(data, key=lambda r: -num(r[st]))[:top]:
    print(f"{r[0][-5:]} {num(r[ie]):>11} {num(r[st]):>7}  {r[src].strip()}")
