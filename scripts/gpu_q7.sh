#!/bin/bash
mkdir -p gpurun_out
for I in ta101 ta021; do timeout 600 python bench.py --mode bound --instance $I --steps 10 --no-cpu-baseline > gpurun_out/qb_$I.json 2> gpurun_out/qb_$I.err; tail -2 gpurun_out/qb_$I.err; python -c "
import json; d=json.load(open('gpurun_out/qb_$I.json')); print('$I', round(d['value']/1e6,2), 'M/s', d['ms_per_step'], d['roofline']['frac'], d['roofline']['hbm'], d['e2e']['value'])"; done
timeout 600 ncu --set full --clock-control none -k regex:k1_bound -s 2 -c 1 -o gpurun_out/prof_k1_ta101 -f python bench.py --mode bound --instance ta101 --steps 1 --warmup 1 --pool 1000000 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none -k regex:k1_bound -s 2 -c 1 -o gpurun_out/prof_k1_ta021 -f python bench.py --mode bound --instance ta021 --steps 1 --warmup 1 --pool 4000000 --no-e2e --no-cpu-baseline > /dev/null 2>&1
ls gpurun_out/prof_k1*
