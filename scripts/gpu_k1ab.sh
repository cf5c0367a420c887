#!/bin/bash
export FBB_NO_CLOCKS=1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "k1" 2>&1 | tail -1
for K in v1 v2; do for I in ta021 ta001 ta051 ta081; do FBB_K1=$K timeout 600 python bench.py --mode bound --instance $I --steps 10 --no-cpu-baseline --no-e2e > gpurun_out/qb.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/qb.json')); print('$K $I', round(d['value']/1e6,2), 'M/s')"; done; done
