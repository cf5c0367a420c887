#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "direct_placement or kernel_variants or device_planned or traces" > gpurun_out/pytest_f.txt 2>&1; tail -3 gpurun_out/pytest_f.txt
for T in 4096 16384 262144; do
  timeout 300 python bench.py --target $T --steps 200 --no-cpu-baseline > gpurun_out/e2e_$T.json 2>/dev/null
  FBB_DEVICE_LOOP=1 timeout 300 python bench.py --target $T --steps 200 --no-cpu-baseline > gpurun_out/e2edl_$T.json 2>/dev/null
done
python scripts/show.py gpurun_out/e2e*.json
