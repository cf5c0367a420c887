#!/bin/bash
# compute-sanitizer over every kernel path (race detection).
mkdir -p gpurun_out
for T in memcheck racecheck synccheck; do
  # racecheck does not follow the conditional-graph device loop (it reports the body's
  # kernels as concurrent and then fails): it checks the same kernels launched without a graph
  G=1; [ $T = racecheck ] && G=0
  FBB_LOOP_GRAPH=$G timeout 900 compute-sanitizer --tool $T --print-limit 20 python scripts/sanitize.py > gpurun_out/sanitize_$T.txt 2>&1
  echo "== $T: $(grep -c '^ok' gpurun_out/sanitize_$T.txt) ok; $(tail -1 gpurun_out/sanitize_$T.txt)"
done
FBB_DEVICE_LOOP=1 timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python scripts/sanitize.py > gpurun_out/sanitize_devloop.txt 2>&1
echo "== memcheck devloop: $(tail -1 gpurun_out/sanitize_devloop.txt)"
