#!/bin/bash
# Quick GPU check: parity tests, bench (twice: clocks on / off), launch list.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.txt 2>&1; tail -3 gpurun_out/pytest_gpu.txt
for I in ${INSTANCES:-ta021}; do
  timeout 600 python bench.py --instance $I --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/q_$I.json 2> gpurun_out/q_$I.err; tail -2 gpurun_out/q_$I.err
  FBB_NO_CLOCKS=1 timeout 600 python bench.py --instance $I --no-cpu-baseline --no-e2e ${BENCH_ARGS} > gpurun_out/q2_$I.json 2>> gpurun_out/q_$I.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
   --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
python scripts/summarize_launches.py gpurun_out/launches.csv
