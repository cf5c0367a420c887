#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.txt 2>&1; tail -3 gpurun_out/pytest_gpu.txt
timeout 300 python scripts/diag_host.py 2>&1 | tail -6
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/q_ta021.json 2> gpurun_out/q_ta021.err; tail -2 gpurun_out/q_ta021.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
   --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
python scripts/summarize_launches.py gpurun_out/launches.csv
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"place|k2_v2" -s 12 -c 2 \
   -o gpurun_out/prof_place -f python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_place.log 2>&1
tail -1 gpurun_out/ncu_place.log
