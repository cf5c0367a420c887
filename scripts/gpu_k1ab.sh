#!/bin/bash
# K1 A/B: parity, then bound-only passes with v3 (default) and v2 on Ta021 / Ta101 pools; ncu of v3.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -k "k1 or range or backendset or synth" > gpurun_out/pytest_k1.txt 2>&1; tail -2 gpurun_out/pytest_k1.txt
for I in ta021 ta101 ta051; do
  for V in v3 v2; do
    FBB_K1=$V timeout 600 python bench.py --mode bound --instance $I --steps 10 --pool ${POOL:-4000000} --no-e2e --no-cpu-baseline > gpurun_out/bound_${I}_$V.json 2> gpurun_out/bound_${I}_$V.err
    python -c "import json;d=json.load(open('gpurun_out/bound_${I}_$V.json'));print('$I $V', round(d['value']/1e6,1),'M/s frac',round(d['roofline']['frac'],3), d['roofline']['kernel'])"
  done
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k1" -s 1 -c 1 \
   -o gpurun_out/prof_k1v3_ta101 -f python bench.py --mode bound --instance ta101 --steps 2 --warmup 1 --pool 500000 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k1" -s 1 -c 1 \
   -o gpurun_out/prof_k1v3_ta021 -f python bench.py --mode bound --instance ta021 --steps 2 --warmup 1 --pool 2000000 --no-e2e --no-cpu-baseline > /dev/null 2>&1
ls gpurun_out
