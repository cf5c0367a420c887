#!/bin/bash
# r02: new parity tests (large traces, device loop graph, multi-rank, group), small-pool sweep
# host-planned vs graph device loop, Ta001 solve, reference-API e2e, ncu of K2 v2 / v3 hot lines
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "large_traces or device_planned_loop" > gpurun_out/pytest_new.txt 2>&1; tail -3 gpurun_out/pytest_new.txt
for T in 4096 16384 65536 262144; do
  timeout 300 python bench.py --target $T --steps 200 --no-cpu-baseline --no-e2e > gpurun_out/sweep_$T.json 2>/dev/null
  FBB_DEVICE_LOOP=1 timeout 300 python bench.py --target $T --steps 200 --no-cpu-baseline --no-e2e > gpurun_out/sweepdl_$T.json 2>/dev/null
done
python scripts/show.py gpurun_out/sweep*.json
timeout 120 tests/cpp/bin/dropin_bench 262144 20 > gpurun_out/dropin_bench.json 2>&1; cat gpurun_out/dropin_bench.json
timeout 900 python bench.py --mode solve --instance ta001 --max-seconds 600 --cpu-sample 2000000 > gpurun_out/solve_ta001.json 2> gpurun_out/solve_ta001.err; tail -c 600 gpurun_out/solve_ta001.json
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k2_v3" -s 5 -c 1 \
   -o gpurun_out/prof_k2v3 -f python bench.py --instance ta081 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_k2v3.log 2>&1; tail -1 gpurun_out/ncu_k2v3.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k2_v2" -s 5 -c 1 \
   -o gpurun_out/prof_k2v2 -f python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_k2v2.log 2>&1; tail -1 gpurun_out/ncu_k2v2.log
