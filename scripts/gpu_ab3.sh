#!/bin/bash
# device-loop A/B (multi-round calls): working tree vs libflowbb_b200_ab_old.so
mkdir -p gpurun_out
OLD=$PWD/paper_1206_4973_b200/libflowbb_b200_ab_old.so
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "device_planned or direct_placement" > gpurun_out/pytest_ab3.txt 2>&1; tail -2 gpurun_out/pytest_ab3.txt
for rep in 1 2; do
  for v in old new; do
    if [ $v = old ]; then export FBB_LIB=$OLD; else unset FBB_LIB; fi
    for T in 4096 262144; do
      FBB_DEVICE_LOOP=1 timeout 300 python bench.py --target $T --steps 150 --no-cpu-baseline > gpurun_out/ab3_${v}_${T}_$rep.json 2>/dev/null
    done
  done
done
unset FBB_LIB
python - <<'PY'
import json
for T in (4096, 262144):
    for v in ("old", "new"):
        vals = []
        for rep in (1, 2):
            try:
                d = json.load(open(f"gpurun_out/ab3_{v}_{T}_{rep}.json")); vals.append((round(d["value"] / 1e6), round(d["e2e"]["value"] / 1e6)))
            except Exception:
                vals.append("fail")
        print(T, v, vals)
PY
