#!/bin/bash
mkdir -p gpurun_out
timeout 600 compute-sanitizer --tool racecheck --print-limit 20 python scripts/sanitize.py > gpurun_out/sanitize_racecheck.txt 2>&1
echo "== racecheck: $(grep -c '^ok' gpurun_out/sanitize_racecheck.txt) ok; $(tail -1 gpurun_out/sanitize_racecheck.txt)"
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "direct_placement or traces or solve" > gpurun_out/pytest_l.txt 2>&1; tail -2 gpurun_out/pytest_l.txt
for T in 4096 16384 32768; do timeout 300 python bench.py --target $T --steps 200 --no-cpu-baseline --no-e2e > gpurun_out/l_$T.json 2>/dev/null; done
python scripts/show.py gpurun_out/l_*.json
