#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "device_planned or direct_placement or resolve_traces" > gpurun_out/pytest_s.txt 2>&1; tail -2 gpurun_out/pytest_s.txt
FBB_DEVICE_LOOP=1 timeout 300 ncu --graph-profiling node --metrics gpu__time_duration.sum --clock-control none -c 80 --csv \
   --log-file gpurun_out/launches_dl_262k.csv python bench.py --steps 6 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
python scripts/summarize_launches.py gpurun_out/launches_dl_262k.csv | tail -10
