#!/bin/bash
mkdir -p gpurun_out
timeout 600 python scripts/diag.py seq 3000000 > gpurun_out/diag_seq_plain.txt 2>&1; tail -6 gpurun_out/diag_seq_plain.txt
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.txt 2>&1; tail -15 gpurun_out/pytest_gpu.txt
timeout 300 python scripts/diag.py timing > gpurun_out/diag_timing.txt 2>&1; cat gpurun_out/diag_timing.txt
