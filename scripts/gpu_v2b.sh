#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.txt 2>&1; tail -3 gpurun_out/pytest_gpu.txt
timeout 600 python scripts/diag.py seq 3000000 > gpurun_out/diag_seq.txt 2>&1; grep -c " ok" gpurun_out/diag_seq.txt; grep -E "MISMATCH|Error" gpurun_out/diag_seq.txt | head -3
for T in 262144 524288; do timeout 300 python bench.py --no-cpu-baseline --no-e2e --target $T > gpurun_out/bench_$T.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/bench_$T.json')); print('T=$T', round(d['value']/1e6,1), 'M/s dev', round(d['wall_value']/1e6,1), 'wall ms/step', round(d['ms_per_step'],4), 'k2share', round(d['roofline']['k2_share_of_round'],3))"; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k2_ -s 6 -c 1 \
     -o gpurun_out/prof_k2v2b -f python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_v2b.log 2>&1
tail -1 gpurun_out/ncu_v2b.log
