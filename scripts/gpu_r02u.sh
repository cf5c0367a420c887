#!/bin/bash
mkdir -p gpurun_out
FBB_LOOP_GRAPH=0 timeout 600 compute-sanitizer --tool racecheck --print-limit 20 python scripts/sanitize.py > gpurun_out/sanitize_racecheck.txt 2>&1
echo "== racecheck: $(grep -c '^ok' gpurun_out/sanitize_racecheck.txt) ok; $(tail -1 gpurun_out/sanitize_racecheck.txt)"
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "traces or device_planned or direct" > gpurun_out/pytest_u.txt 2>&1; tail -2 gpurun_out/pytest_u.txt
timeout 600 python bench.py --steps 200 > gpurun_out/u_bench.json 2> gpurun_out/u_bench.err; python scripts/show.py gpurun_out/u_bench.json
