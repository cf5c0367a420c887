#!/bin/bash
# spread_ppc A/B: explorer parity subset + batch sweep
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "traces or device_planned or direct or explorer" > gpurun_out/pytest_s3a.txt 2>&1; tail -2 gpurun_out/pytest_s3a.txt
STEPS=10 timeout 600 python scripts/batch_sweep.py 4096 8192 16384 32768 65536 262144 2>&1 | python scripts/show_sweep.py
