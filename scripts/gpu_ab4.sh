#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for I in ta021 ta051 ta001 ta081; do timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 100 --instance $I > gpurun_out/q_$I.json 2>/dev/null; python scripts/show.py gpurun_out/q_$I.json | head -1; done
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:k2_v2 -s 5 -c 1 --csv --log-file gpurun_out/kp.csv python scripts/k2_pool_bench.py 2 > /dev/null 2>&1
grep -E "gpu__time|inst_executed|issue_active" gpurun_out/kp.csv | awk -F'","' '{print $(NF-2), $NF}'
timeout 600 python bench.py --no-cpu-baseline --steps 100 > gpurun_out/q_e2e.json 2>/dev/null; python scripts/show.py gpurun_out/q_e2e.json | head -1
