#!/bin/bash
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
timeout 1500 compute-sanitizer --tool racecheck --print-limit 20 python scripts/sanitize.py > gpurun_out/sanitize_racecheck.txt 2>&1; echo "racecheck: $(tail -1 gpurun_out/sanitize_racecheck.txt)"
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python scripts/sanitize.py > gpurun_out/sanitize_memcheck.txt 2>&1; echo "memcheck: $(tail -1 gpurun_out/sanitize_memcheck.txt)"
bash scripts/gpu_k1ab.sh
