#!/bin/bash
# Where a small-pool round's time goes: kernel durations (ncu, serialised) and the event /
# device-clock split (FBB_PDL=0: events around K2 and place) at 4K and 16K children.
mkdir -p gpurun_out
for T in 4096 16384; do
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
     --log-file gpurun_out/launches_small_$T.csv python bench.py --target $T --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
  FBB_PDL=0 timeout 300 python bench.py --target $T --steps 200 --no-cpu-baseline --no-e2e > gpurun_out/sweep_nopdl_$T.json 2>/dev/null
done
python scripts/summarize_launches.py gpurun_out/launches_small_4096.csv 2>&1 | tail -15
python scripts/summarize_launches.py gpurun_out/launches_small_16384.csv 2>&1 | tail -15
python scripts/show.py gpurun_out/sweep_nopdl_*.json
FBB_DEVICE_LOOP=1 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv \
   --log-file gpurun_out/launches_small_dl_4096.csv python bench.py --target 4096 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
python scripts/summarize_launches.py gpurun_out/launches_small_dl_4096.csv 2>&1 | tail -15
