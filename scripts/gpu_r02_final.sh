#!/bin/bash
# r02 deliverables: full GPU suite + smoke, default bench (both arms), per-config lines,
# launch list of the default command, ncu --set full of K2 v2 / v3 and K1 v3.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu.txt
nproc > gpurun_out/nproc.txt; lscpu | grep -E "Model name|^CPU\(s\)" >> gpurun_out/nproc.txt
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.txt 2>&1; tail -2 gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; tail -1 gpurun_out/smoke.txt
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -1 gpurun_out/bench.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
for I in ta001 ta051 ta081 ta101; do timeout 600 python bench.py --instance $I > gpurun_out/bench_$I.json 2> gpurun_out/bench_$I.err; done
for I in ta021 ta051 ta101; do timeout 600 python bench.py --mode bound --instance $I --steps 10 > gpurun_out/bench_bound_$I.json 2> gpurun_out/bench_bound_$I.err; done
python scripts/show.py gpurun_out/bench*.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
   --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
python scripts/summarize_launches.py gpurun_out/launches.csv | tail -8
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k2_|place" -s 12 -c 2 \
   -o gpurun_out/prof_k2_final -f python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_final.log 2>&1; tail -1 gpurun_out/ncu_final.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k2_v3" -s 5 -c 1 \
   -o gpurun_out/prof_k2v3_ta081 -f python bench.py --instance ta081 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_v3.log 2>&1; tail -1 gpurun_out/ncu_v3.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k1v3" -s 1 -c 1 \
   -o gpurun_out/prof_k1v3_ta101 -f python bench.py --mode bound --instance ta101 --steps 2 --warmup 1 --pool 1000000 --no-e2e --no-cpu-baseline > gpurun_out/ncu_k1.log 2>&1; tail -1 gpurun_out/ncu_k1.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k1v3" -s 1 -c 1 \
   -o gpurun_out/prof_k1v3_ta021 -f python bench.py --mode bound --instance ta021 --steps 2 --warmup 1 --pool 2000000 --no-e2e --no-cpu-baseline > gpurun_out/ncu_k1b.log 2>&1; tail -1 gpurun_out/ncu_k1b.log
bash scripts/gpu_sweep.sh > gpurun_out/sweep_table.md; cat gpurun_out/sweep_table.md
timeout 600 oracle/_ref/dropin_test > gpurun_out/dropin.txt 2>&1; tail -1 gpurun_out/dropin.txt
timeout 900 python bench.py --mode exhaust --instance ta021 --group 2 > gpurun_out/exhaust_group2.json 2> gpurun_out/exhaust_group2.err; tail -c 400 gpurun_out/exhaust_group2.json
for T in memcheck racecheck synccheck; do G=1; [ $T = racecheck ] && G=0; FBB_LOOP_GRAPH=$G timeout 600 compute-sanitizer --tool $T --print-limit 20 python scripts/sanitize.py > gpurun_out/sanitize_$T.txt 2>&1; echo "== $T: $(grep -c "^ok" gpurun_out/sanitize_$T.txt) ok; $(tail -1 gpurun_out/sanitize_$T.txt)"; done
timeout 900 python bench.py --mode solve --instance ta001 --max-seconds 600 --cpu-sample 2000000 > gpurun_out/solve_ta001.json 2> gpurun_out/solve_ta001.err
timeout 900 python bench.py --mode solve --instance ta001 --group 2 --max-seconds 600 --no-cpu-baseline > gpurun_out/solve_ta001_group2.json 2> gpurun_out/solve_ta001_group2.err
timeout 900 python bench.py --instance ta051 --tuner > gpurun_out/bench_ta051_tuner.json 2> gpurun_out/bench_ta051_tuner.err
timeout 900 python bench.py --mode bound --instance ta101 --pool 0 --steps 3 --warmup 1 > gpurun_out/bench_bound_ta101_max.json 2> gpurun_out/bench_bound_ta101_max.err
python scripts/show.py gpurun_out/solve_*.json gpurun_out/bench_ta051_tuner.json gpurun_out/bench_bound_ta101_max.json
