#!/bin/bash
# r02 session 3, second confirmation (TMA row staging, place runs): GPU suite + smoke, default
# bench (both arms), Ta001 / Ta051 tuner lines, launch list, K2 ncu, drop-in binary
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu.txt
nproc > gpurun_out/nproc.txt; lscpu | grep -E "Model name|^CPU\(s\)" >> gpurun_out/nproc.txt
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.txt 2>&1; tail -2 gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; tail -1 gpurun_out/smoke.txt
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -1 gpurun_out/bench.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
for I in ta001 ta051 ta081 ta101; do timeout 600 python bench.py --instance $I > gpurun_out/bench_$I.json 2> gpurun_out/bench_$I.err; done
timeout 900 python bench.py --instance ta051 --tuner > gpurun_out/bench_ta051_tuner.json 2> gpurun_out/bench_ta051_tuner.err
python scripts/show.py gpurun_out/bench*.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
   --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
python scripts/summarize_launches.py gpurun_out/launches.csv | tail -8
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k2_|place" -s 12 -c 2 \
   -o gpurun_out/prof_k2_final -f python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_final.log 2>&1; tail -1 gpurun_out/ncu_final.log
timeout 600 oracle/_ref/dropin_test > gpurun_out/dropin.txt 2>&1; tail -1 gpurun_out/dropin.txt
timeout 900 python bench.py --mode exhaust --instance ta021 > gpurun_out/exhaust_ta021.json 2> gpurun_out/exhaust_ta021.err
timeout 900 python bench.py --mode solve --instance ta001 --max-seconds 600 --cpu-sample 2000000 > gpurun_out/solve_ta001.json 2> gpurun_out/solve_ta001.err
python scripts/show.py gpurun_out/solve_ta001.json gpurun_out/exhaust_ta021.json
