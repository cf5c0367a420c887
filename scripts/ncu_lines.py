"""Per-source-line totals of an ncu --set full report: warp instructions executed and stall
samples of each CUDA source line of one kernel, via the SASS page and nvdisasm -g line info
of the same build.  python scripts/ncu_lines.py REPORT OBJECT.o KERNEL_SUBSTRING [TOP]"""
import collections
import csv
import glob
import io
import os
import re
import subprocess
import sys
import tempfile

rep, obj, pat = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
out = subprocess.run(["ncu", "-i", rep, "-k", "regex:" + re.split(r"<|IL", pat)[0], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, data = rows[1], [r for r in rows[2:] if len(r) == len(rows[1])]
ie, st = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
num = lambda s: int(s) if s.isdigit() else 0  # noqa: E731
base = min(int(r[0], 16) for r in data)
prof = {int(r[0], 16) - base: (num(r[ie]), num(r[st])) for r in data}
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=tmp, capture_output=True)
cubin = glob.glob(os.path.join(tmp, "*.cubin"))[0]
dis = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
line, on, src = None, False, {}
per = collections.defaultdict(lambda: [0, 0])
for ln in dis.splitlines():
    if ln.strip().startswith(".text.") or re.match(r"^\s*\.section\s+\.text\.", ln):
        on = pat in ln
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        line = (os.path.basename(m.group(1)), int(m.group(2)))
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
    if on and m and line:
        off = int(m.group(1), 16)
        if off in prof:
            per[line][0] += prof[off][0]
            per[line][1] += prof[off][1]
ti = sum(v[0] for v in per.values()) or 1
ts = sum(v[1] for v in per.values()) or 1
print(f"{pat}: {ti} warp instructions, {ts} stall samples mapped")
for (f, l), (i, s) in sorted(per.items(), key=lambda kv: -kv[1][1])[:top]:
    print(f"{f}:{l:<5} inst {100.0 * i / ti:5.1f}%  stall {100.0 * s / ts:5.1f}%")
