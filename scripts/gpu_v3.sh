#!/bin/bash
# v3 (n > 64) check: GPU parity tests, the 100x20 / 200x20 / 50x20 bench lines, one ncu capture of v3.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for I in ${INSTANCES:-ta081 ta101 ta051}; do timeout 600 python bench.py --instance $I --no-cpu-baseline --no-e2e > gpurun_out/v3_$I.json 2> gpurun_out/v3_$I.err; done
python scripts/show.py gpurun_out/v3_*.json
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k2_v3" -s 5 -c 1 \
   -o gpurun_out/prof_k2v3_ta081 -f python bench.py --instance ta081 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_v3.log 2>&1
tail -1 gpurun_out/ncu_v3.log
