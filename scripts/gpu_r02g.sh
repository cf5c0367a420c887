#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/pytest_g.txt 2>&1; tail -3 gpurun_out/pytest_g.txt
for T in 4096 16384 262144; do
  timeout 300 python bench.py --target $T --steps 200 --no-cpu-baseline > gpurun_out/e2e_$T.json 2>/dev/null
  FBB_DEVICE_LOOP=1 timeout 300 python bench.py --target $T --steps 200 --no-cpu-baseline > gpurun_out/e2edl_$T.json 2>/dev/null
done
python scripts/show.py gpurun_out/e2e*.json
FBB_DEVICE_LOOP=1 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv \
   --log-file gpurun_out/launches_small_dl_4096.csv python bench.py --target 4096 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
python scripts/summarize_launches.py gpurun_out/launches_small_dl_4096.csv 2>&1 | tail -10
