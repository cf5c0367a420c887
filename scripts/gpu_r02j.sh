#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "k1 or synth or backendset" > gpurun_out/pytest_j.txt 2>&1; tail -2 gpurun_out/pytest_j.txt
FBB_DIRECT=0 timeout 300 python bench.py --instance ta001 --no-cpu-baseline --no-e2e > gpurun_out/j_ta001_nodirect.json 2>/dev/null
timeout 300 python bench.py --instance ta001 --no-cpu-baseline --no-e2e > gpurun_out/j_ta001.json 2>/dev/null
FBB_DIRECT=0 timeout 300 python bench.py --instance ta001 --no-cpu-baseline --no-e2e > gpurun_out/j_ta001_nodirect2.json 2>/dev/null
for I in ta021 ta051 ta101; do timeout 600 python bench.py --mode bound --instance $I --steps 10 --no-cpu-baseline --no-e2e > gpurun_out/j_bound_$I.json 2>/dev/null; done
python scripts/show.py gpurun_out/j_*.json
timeout 900 ncu --set full --clock-control none -k regex:"k1v3" -s 1 -c 1 \
   -o gpurun_out/prof_k1v3_ta101_split -f python bench.py --mode bound --instance ta101 --steps 2 --warmup 1 --pool 1000000 --no-e2e --no-cpu-baseline > /dev/null 2>&1
ncu -i gpurun_out/prof_k1v3_ta101_split.ncu-rep --page raw --csv 2>/dev/null | python -c "
import csv,sys
r=list(csv.reader(sys.stdin)); h=r[0]
for k in ['gpu__time_duration.sum','l1tex__data_pipe_lsu_wavefronts_mem_shared.sum','l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum','smsp__issue_active.avg.pct_of_peak_sustained_active']:
    print(k, r[2][h.index(k)])"
