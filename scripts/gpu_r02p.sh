#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.txt 2>&1; tail -3 gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; tail -1 gpurun_out/smoke.txt
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
python scripts/show.py gpurun_out/bench.json
timeout 900 python bench.py --mode exhaust --instance ta021 > gpurun_out/exhaust_ta021.json 2> gpurun_out/exhaust_ta021.err; tail -c 500 gpurun_out/exhaust_ta021.json
timeout 900 python bench.py --mode solve --instance ta001 --no-cpu-baseline > gpurun_out/solve_ta001.json 2> gpurun_out/solve_ta001.err; tail -c 300 gpurun_out/solve_ta001.json
