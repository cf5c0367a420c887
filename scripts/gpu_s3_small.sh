#!/bin/bash
# r02 session 3: small pools -- batch sweep (host-planned / device-planned incl. the persistent
# batch kernel), per-round breakdown, and the launch list of 4 K-child batches
mkdir -p gpurun_out
STEPS=20 timeout 600 python scripts/batch_sweep.py 4096 8192 16384 32768 65536 131072 262144 > gpurun_out/batch_sweep.jsonl 2> gpurun_out/batch_sweep.err
python scripts/show_sweep.py < gpurun_out/batch_sweep.jsonl > gpurun_out/batch_sweep.md; cat gpurun_out/batch_sweep.md
FBB_PERSIST=0 STEPS=20 timeout 600 python scripts/batch_sweep.py 4096 16384 32768 2>/dev/null | python scripts/show_sweep.py > gpurun_out/batch_sweep_graph.md; cat gpurun_out/batch_sweep_graph.md
FBB_LOOP_DEBUG=1 timeout 120 python scripts/probe_loop.py 2>&1 | grep -v grow > gpurun_out/probe_loop.txt; grep "per round" gpurun_out/probe_loop.txt | tail -3
BATCH=32 STEPS=3 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 100 --csv \
   --log-file gpurun_out/launches_batch4k.csv python scripts/batch_sweep.py 4096 > /dev/null 2>&1
python scripts/summarize_launches.py gpurun_out/launches_batch4k.csv | tail -10
