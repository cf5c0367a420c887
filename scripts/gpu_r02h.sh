#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "direct_placement or kernel_variants or device_planned or resolve_traces or solve_traces" > gpurun_out/pytest_h.txt 2>&1; tail -2 gpurun_out/pytest_h.txt
for T in 4096 16384 32768 262144; do
  timeout 300 python bench.py --target $T --steps 200 --no-cpu-baseline --no-e2e > gpurun_out/s_$T.json 2>/dev/null
done
timeout 300 python bench.py --steps 200 --no-cpu-baseline > gpurun_out/s_e2e.json 2>/dev/null
python scripts/show.py gpurun_out/s_*.json
