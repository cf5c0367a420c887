#!/bin/bash
# r02: direct placement (single-wave pools) parity + small-pool sweep
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "direct_placement" > gpurun_out/pytest_direct.txt 2>&1; tail -3 gpurun_out/pytest_direct.txt
grep -q passed gpurun_out/pytest_direct.txt || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "traces or device_planned or explorer" > gpurun_out/pytest_explorer.txt 2>&1; tail -3 gpurun_out/pytest_explorer.txt
for T in 4096 16384 32768 65536; do
  timeout 120 python bench.py --target $T --steps 200 --no-cpu-baseline --no-e2e > gpurun_out/sweep_$T.json 2>/dev/null
  FBB_DEVICE_LOOP=1 timeout 120 python bench.py --target $T --steps 200 --no-cpu-baseline --no-e2e > gpurun_out/sweepdl_$T.json 2>/dev/null
done
python scripts/show.py gpurun_out/sweep*.json
FBB_DEVICE_LOOP=1 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv \
   --log-file gpurun_out/launches_small_dl_4096.csv python bench.py --target 4096 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
python scripts/summarize_launches.py gpurun_out/launches_small_dl_4096.csv 2>&1 | tail -10
