#!/bin/bash
mkdir -p gpurun_out
timeout 600 python bench.py --instance ta101 --no-cpu-baseline --steps 100 > gpurun_out/q_ta101.json 2>/dev/null; python scripts/show.py gpurun_out/q_ta101.json
timeout 600 python bench.py --instance ta051 --tuner --no-cpu-baseline --steps 100 > gpurun_out/q_ta051_tuner.json 2>/dev/null; python scripts/show.py gpurun_out/q_ta051_tuner.json
python -c "import json; d=json.load(open('gpurun_out/q_ta051_tuner.json')); print(d['config']); print(sorted(set(r[0] for r in d['rounds'])))"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k2_v3" -s 4 -c 1 \
   -o gpurun_out/prof_k2v3_ta081 -f python bench.py --instance ta081 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_v3.log 2>&1
tail -1 gpurun_out/ncu_v3.log
