#!/bin/bash
# r02: integer issue-rate microbenchmark, GPU tests (multi-rank, group, CLI, drop-in), small-pool sweep
mkdir -p gpurun_out
timeout 120 scripts/micro/intpeak > gpurun_out/intpeak.json 2> gpurun_out/intpeak.err; cat gpurun_out/intpeak.json
timeout 1500 python -m pytest tests -m gpu -q ${PYTEST_ARGS} > gpurun_out/pytest_gpu.txt 2>&1; tail -5 gpurun_out/pytest_gpu.txt
for T in 4096 16384 65536; do
  timeout 300 python bench.py --target $T --steps 200 --no-cpu-baseline --no-e2e > gpurun_out/sweep_$T.json 2>/dev/null
  FBB_DEVICE_LOOP=1 timeout 300 python bench.py --target $T --steps 200 --no-cpu-baseline --no-e2e > gpurun_out/sweepdl_$T.json 2>/dev/null
done
python scripts/show.py gpurun_out/sweep*.json
