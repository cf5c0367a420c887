#!/bin/bash
mkdir -p gpurun_out
for V in old new; do
case $V in old) D=_ab_old;; var) D=_ab_var;; var2) D=_ab_var2;; new) D=.;; esac
(cd $D && timeout 600 ncu --metrics gpu__time_duration.sum,sm__cycles_active.max,sm__cycles_active.avg --clock-control none -k regex:k2_v2 -s 5 -c 3 --csv \
   --log-file $GRAFT_REPO_ROOT/gpurun_out/kp_$V.csv python $GRAFT_REPO_ROOT/scripts/k2_pool_bench.py 3 > $GRAFT_REPO_ROOT/gpurun_out/kp_$V.txt 2>&1)
echo "$V"; tail -1 gpurun_out/kp_$V.txt; python - <<PY
import csv
rows=list(csv.reader(open("gpurun_out/kp_$V.csv")))
h=None; d={}
for r in rows:
    if "Metric Name" in r: h=r; continue
    if h and len(r)==len(h): d.setdefault(int(r[h.index("ID")]),{})[r[h.index("Metric Name")]]=r[h.index("Metric Value")]
for k in sorted(d): print(k, d[k])
PY
done
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
export FBB_NO_CLOCKS=1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
   --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
python scripts/summarize_launches.py gpurun_out/launches.csv 2>/dev/null | head -5
