#!/bin/bash
mkdir -p gpurun_out
FBB_HOST_IN=mapped timeout 900 python -m pytest tests -m gpu -x -q -k pending_host > gpurun_out/pytest_gpu_mapped.txt 2>&1; tail -1 gpurun_out/pytest_gpu_mapped.txt
timeout 300 python scripts/diag_host.py 2>&1 | tail -6 | head -2
FBB_HOST_IN=mapped timeout 300 python scripts/diag_host.py 2>&1 | tail -6 | head -2
for i in 1 2; do
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/q_ta021.json 2> gpurun_out/q_ta021.err; tail -2 gpurun_out/q_ta021.err
FBB_HOST_IN=mapped timeout 600 python bench.py --no-cpu-baseline > gpurun_out/q2_ta021.json 2> gpurun_out/q_ta021.err; tail -2 gpurun_out/q_ta021.err
python scripts/show.py gpurun_out/q_ta021.json gpurun_out/q2_ta021.json
done
