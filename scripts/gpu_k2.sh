#!/bin/bash
# K2 variant comparison: tests, bench (v2 vs generic), ncu of the v2 kernel.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.txt 2>&1; tail -3 gpurun_out/pytest_gpu.txt
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_v2.json 2> gpurun_out/bench_v2.err; tail -2 gpurun_out/bench_v2.err
FBB_K2=generic timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_v1.json 2> gpurun_out/bench_v1.err
for T in 65536 131072 524288; do timeout 300 python bench.py --no-cpu-baseline --no-e2e --target $T > gpurun_out/bench_v2_$T.json 2>&1; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k2_ -s 6 -c 2 \
     -o gpurun_out/prof_k2v2 -f python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_v2.log 2>&1
tail -2 gpurun_out/ncu_v2.log
