#!/bin/bash
# r02: full GPU suite, v3 occupancy, config-3 tuner line, HBM-filling config 5, multi-device
# exhaustion (fbb_group in-process; 2 ranks sharing the GPU over gloo), 2-rank explore overhead
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.txt 2>&1; tail -3 gpurun_out/pytest_gpu.txt
for I in ta081 ta101; do timeout 600 python bench.py --instance $I --no-cpu-baseline > gpurun_out/bench_$I.json 2> gpurun_out/bench_$I.err; done
timeout 900 python bench.py --instance ta051 --tuner > gpurun_out/bench_ta051_tuner.json 2> gpurun_out/bench_ta051_tuner.err
python scripts/show.py gpurun_out/bench_*.json
timeout 900 python bench.py --mode bound --instance ta101 --pool 0 --steps 3 --warmup 1 > gpurun_out/bench_bound_ta101_max.json 2> gpurun_out/bench_bound_ta101_max.err; tail -c 300 gpurun_out/bench_bound_ta101_max.json; tail -2 gpurun_out/bench_bound_ta101_max.err
timeout 900 python bench.py --mode exhaust --instance ta021 --group 2 > gpurun_out/exhaust_group2.json 2> gpurun_out/exhaust_group2.err; tail -c 700 gpurun_out/exhaust_group2.json
FBB_SAME_GPU=1 FBB_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 bench.py --mode exhaust --instance ta021 --gpus 2 > gpurun_out/exhaust_2rank.json 2> gpurun_out/exhaust_2rank.err; tail -c 700 gpurun_out/exhaust_2rank.json
FBB_SAME_GPU=1 FBB_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29532 bench.py --gpus 2 --steps 200 --no-cpu-baseline > gpurun_out/bench_2rank.json 2> gpurun_out/bench_2rank.err; python scripts/show.py gpurun_out/bench_2rank.json
