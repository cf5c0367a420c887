#!/bin/bash
# ncu --set full (with source) of the hot kernels: K2 v2 (Ta021), K2 v3 (Ta081), K1 (Ta021, Ta101 bound-only)
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k2_v2" -s 5 -c 1 \
   -o gpurun_out/prof_k2v2 -f python scripts/k2_pool_bench.py 2 > gpurun_out/ncu_k2v2.log 2>&1; tail -1 gpurun_out/ncu_k2v2.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k2_v3" -s 5 -c 1 \
   -o gpurun_out/prof_k2v3 -f python bench.py --instance ta081 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_k2v3.log 2>&1; tail -1 gpurun_out/ncu_k2v3.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k1" -s 1 -c 1 \
   -o gpurun_out/prof_k1_ta101 -f python bench.py --mode bound --instance ta101 --steps 2 --warmup 1 --pool 500000 --no-e2e --no-cpu-baseline > gpurun_out/ncu_k1a.log 2>&1; tail -1 gpurun_out/ncu_k1a.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k1" -s 1 -c 1 \
   -o gpurun_out/prof_k1_ta021 -f python bench.py --mode bound --instance ta021 --steps 2 --warmup 1 --pool 2000000 --no-e2e --no-cpu-baseline > gpurun_out/ncu_k1b.log 2>&1; tail -1 gpurun_out/ncu_k1b.log
ls -la gpurun_out
