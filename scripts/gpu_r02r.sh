#!/bin/bash
mkdir -p gpurun_out
FBB_SAME_GPU=1 FBB_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 bench.py --mode solve --instance ta001 --gpus 2 > gpurun_out/solve_ta001_2rank.json 2> gpurun_out/solve_ta001_2rank.err; tail -c 600 gpurun_out/solve_ta001_2rank.json; tail -3 gpurun_out/solve_ta001_2rank.err
FBB_SAME_GPU=1 FBB_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29542 bench.py --gpus 2 --steps 100 --no-cpu-baseline > gpurun_out/bench_2rank.json 2> gpurun_out/bench_2rank.err; python scripts/show.py gpurun_out/bench_2rank.json; tail -2 gpurun_out/bench_2rank.err
