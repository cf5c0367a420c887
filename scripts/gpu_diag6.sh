#!/bin/bash
mkdir -p gpurun_out
for i in 1 2 3; do timeout 600 python scripts/diag.py seq 3000000 > gpurun_out/diag_seq_$i.txt 2>&1; grep -c " ok" gpurun_out/diag_seq_$i.txt; grep -E "MISMATCH|Error" gpurun_out/diag_seq_$i.txt | head -3; done
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.txt 2>&1; tail -5 gpurun_out/pytest_gpu.txt
timeout 300 python scripts/diag.py timing > gpurun_out/diag_timing.txt 2>&1; cat gpurun_out/diag_timing.txt
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; python -c "
import json; d=json.load(open('gpurun_out/bench.json')); print(d['value']/1e6, d['wall_value']/1e6, d['ms_per_step'], d['e2e']['value']/1e6, d['e2e']['rounds_match_device_explorer'], d['roofline']['k2_share_of_round'])"
