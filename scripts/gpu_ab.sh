#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for V in old new; do
case $V in old) D=_ab_old;; new) D=.;; esac
(cd $D && timeout 600 ncu --metrics gpu__time_duration.sum,sm__cycles_active.max,sm__cycles_active.avg,sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:k2_v2 -s 5 -c 3 --csv \
   --log-file $GRAFT_REPO_ROOT/gpurun_out/kp_$V.csv python $GRAFT_REPO_ROOT/scripts/k2_pool_bench.py 3 > $GRAFT_REPO_ROOT/gpurun_out/kp_$V.txt 2>&1)
echo "$V"; tail -1 gpurun_out/kp_$V.txt; python - <<PY
import csv
rows=list(csv.reader(open("gpurun_out/kp_$V.csv")))
h=None; d={}
for r in rows:
    if "Metric Name" in r: h=r; continue
    if h and len(r)==len(h): d.setdefault(int(r[h.index("ID")]),{})[r[h.index("Metric Name")].split('.')[0][:30]]=r[h.index("Metric Value")]
for k in sorted(d): print(k, d[k])
PY
done
timeout 600 python bench.py --no-cpu-baseline --steps 100 > gpurun_out/q_ta021.json 2>/dev/null; python scripts/show.py gpurun_out/q_ta021.json
timeout 600 python bench.py --no-cpu-baseline --steps 100 --instance ta051 > gpurun_out/q_ta051.json 2>/dev/null; python scripts/show.py gpurun_out/q_ta051.json
