#!/bin/bash
mkdir -p gpurun_out
FBB_CHECK=1 timeout 900 python scripts/diag.py seq 3000000 > gpurun_out/diag_seq_check.txt 2>&1; tail -12 gpurun_out/diag_seq_check.txt
timeout 300 python scripts/diag.py timing > gpurun_out/diag_timing.txt 2>&1; cat gpurun_out/diag_timing.txt
CUDA_LAUNCH_BLOCKING=1 timeout 1500 compute-sanitizer --tool memcheck --print-limit 10 python scripts/diag.py seq 3000000 > gpurun_out/diag_seq_san.txt 2>&1; tail -40 gpurun_out/diag_seq_san.txt
