#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
FBB_SAME_GPU=1 FBB_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29555 bench.py --gpus 2 --steps 40 --no-cpu-baseline > gpurun_out/q_n2.json 2> gpurun_out/q_n2.err; tail -3 gpurun_out/q_n2.err
python scripts/show.py gpurun_out/q_n2.json
for I in ta021 ta081; do timeout 600 python bench.py --instance $I --no-cpu-baseline > gpurun_out/q_$I.json 2>/dev/null; python scripts/show.py gpurun_out/q_$I.json; done
