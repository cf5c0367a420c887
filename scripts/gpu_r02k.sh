#!/bin/bash
mkdir -p gpurun_out
timeout 600 oracle/_ref/dropin_test > gpurun_out/dropin.txt 2>&1; tail -3 gpurun_out/dropin.txt
timeout 900 python -m pytest tests/test_gpu_multirank.py tests/test_gpu_parity.py -q -x -k "group or direct_placement or device_planned or kernel_variants or solve" > gpurun_out/pytest_k.txt 2>&1; tail -3 gpurun_out/pytest_k.txt
for T in 4096 16384; do timeout 300 python bench.py --target $T --steps 200 --no-cpu-baseline --no-e2e > gpurun_out/k_$T.json 2>/dev/null; done
python scripts/show.py gpurun_out/k_*.json
timeout 120 tests/cpp/bin/dropin_bench 262144 20 > gpurun_out/dropin_bench.json 2>&1; cat gpurun_out/dropin_bench.json
for T in memcheck racecheck synccheck; do
  timeout 600 compute-sanitizer --tool $T --print-limit 20 python scripts/sanitize.py > gpurun_out/sanitize_$T.txt 2>&1
  echo "== $T: $(grep -c '^ok' gpurun_out/sanitize_$T.txt) ok; $(tail -1 gpurun_out/sanitize_$T.txt)"
done
