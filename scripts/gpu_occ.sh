#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.txt 2>&1; tail -2 gpurun_out/pytest_gpu.txt
for O in 2 3; do for T in 262144 524288; do FBB_K2_OCC=$O timeout 300 python bench.py --no-cpu-baseline --no-e2e --target $T > gpurun_out/bench_o${O}_$T.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/bench_o${O}_$T.json')); print('OCC=$O T=$T', round(d['value']/1e6,1), 'M/s dev', round(d['wall_value']/1e6,1), 'wall; ms/step', round(d['ms_per_step'],4), 'k2share', round(d['roofline']['k2_share_of_round'],3), d['clocks'])"; done; done
FBB_K2_OCC=3 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k2_ -s 6 -c 1 \
     -o gpurun_out/prof_k2occ3 -f python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_occ3.log 2>&1
tail -1 gpurun_out/ncu_occ3.log
