#!/bin/bash
# r02 session 3: confirmation of HEAD (GPU suite, smoke, default bench both arms) + small-pool sweep
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu.txt
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.txt 2>&1; tail -2 gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; tail -1 gpurun_out/smoke.txt
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -1 gpurun_out/bench.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
python scripts/show.py gpurun_out/bench*.json
cat scripts/gpu_sweep.sh > /dev/null
bash scripts/gpu_sweep.sh > gpurun_out/sweep_table.md; cat gpurun_out/sweep_table.md
