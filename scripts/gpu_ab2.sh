#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for V in head new occ2; do
unset FBB_LIB FBB_K2_OCC
if [ $V = head ]; then export FBB_LIB=$GRAFT_REPO_ROOT/libflowbb_b200_head.so; fi
if [ $V = occ2 ]; then export FBB_K2_OCC=2; fi
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active --clock-control none -k regex:k2_v2 -s 5 -c 1 --csv \
   --log-file gpurun_out/kp_$V.csv python scripts/k2_pool_bench.py 2 > /dev/null 2>&1
python - <<PY
import csv
rows=list(csv.reader(open("gpurun_out/kp_$V.csv")))
h=None; d={}
for r in rows:
    if "Metric Name" in r: h=r; continue
    if h and len(r)==len(h): d.setdefault(int(r[h.index("ID")]),{})[r[h.index("Metric Name")].split('.')[0][:26]]=r[h.index("Metric Value")]
print("$V", d)
PY
for I in ta021 ta051 ta001; do timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 100 --instance $I > gpurun_out/q_$I.json 2>/dev/null; echo -n "$V "; python scripts/show.py gpurun_out/q_$I.json | head -1; done
done
