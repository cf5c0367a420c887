#!/bin/bash
mkdir -p gpurun_out
FBB_LOOP_DEBUG=1 timeout 300 python bench.py --steps 200 --no-cpu-baseline > gpurun_out/t_e2e.json 2> gpurun_out/t_e2e.err
grep -c "grow" gpurun_out/t_e2e.err; grep "\[loop\]" gpurun_out/t_e2e.err | tail -40
python scripts/show.py gpurun_out/t_e2e.json
