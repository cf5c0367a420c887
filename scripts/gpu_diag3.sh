#!/bin/bash
mkdir -p gpurun_out
timeout 1500 compute-sanitizer --tool memcheck --print-limit 10 python scripts/diag.py ta001 > gpurun_out/diag_ta001.txt 2>&1
tail -80 gpurun_out/diag_ta001.txt
