#!/bin/bash
mkdir -p gpurun_out
timeout 300 python scripts/diag.py timing > gpurun_out/diag_timing.txt 2>&1
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python scripts/diag.py solve > gpurun_out/diag_solve.txt 2>&1
tail -40 gpurun_out/diag_solve.txt; cat gpurun_out/diag_timing.txt
