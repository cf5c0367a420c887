#!/bin/bash
mkdir -p gpurun_out
timeout 600 python scripts/diag.py seq 3000000 > gpurun_out/diag_seq_plain.txt 2>&1; tail -4 gpurun_out/diag_seq_plain.txt
CUDA_LAUNCH_BLOCKING=1 timeout 900 compute-sanitizer --tool memcheck --print-limit 10 python scripts/diag.py seq 60000 > gpurun_out/diag_seq.txt 2>&1
tail -60 gpurun_out/diag_seq.txt
timeout 300 python scripts/diag.py timing > gpurun_out/diag_timing.txt 2>&1; cat gpurun_out/diag_timing.txt
