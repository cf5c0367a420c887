#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for I in ta021 ta051 ta001; do timeout 600 python bench.py --no-cpu-baseline --steps 100 --instance $I > gpurun_out/q_$I.json 2>/dev/null; python scripts/show.py gpurun_out/q_$I.json; done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k2_v2" -s 5 -c 1 \
   -o gpurun_out/prof_k2v2_pool -f python scripts/k2_pool_bench.py 2 > /dev/null 2>&1
ls gpurun_out/prof_k2v2_pool*
