#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for V in 2 3; do
export FBB_K2_OCC=$V
for I in ta021 ta051 ta001; do timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 100 --instance $I > gpurun_out/q_$I.json 2>/dev/null; echo -n "occ$V "; python scripts/show.py gpurun_out/q_$I.json | head -1; done
done
