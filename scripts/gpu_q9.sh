#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3
for K in v1 v2; do for I in ta101 ta051 ta021 ta001; do FBB_K1=$K timeout 600 python bench.py --mode bound --instance $I --steps 10 --no-cpu-baseline --no-e2e > gpurun_out/qb_$I.json 2> gpurun_out/qb_$I.err; tail -2 gpurun_out/qb_$I.err; python -c "
import json; d=json.load(open('gpurun_out/qb_$I.json')); print('$K $I', round(d['value']/1e6,2), 'M/s', round(d['ms_per_step'],3), round(d['roofline']['frac'],4))"; done; done
