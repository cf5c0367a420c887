#!/bin/bash
# same-box A/B: the working tree's library vs paper_1206_4973_b200/libflowbb_b200_ab_old.so
mkdir -p gpurun_out
OLD=$PWD/paper_1206_4973_b200/libflowbb_b200_ab_old.so
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "traces or k2 or direct or host_tree" > gpurun_out/pytest_ab.txt 2>&1; tail -2 gpurun_out/pytest_ab.txt
for rep in 1 2; do
  for v in old new; do
    if [ $v = old ]; then export FBB_LIB=$OLD; else unset FBB_LIB; fi
    timeout 300 python bench.py --steps 100 --no-cpu-baseline ${AB_ARGS} > gpurun_out/ab_${v}_$rep.json 2>/dev/null
    timeout 300 python bench.py --instance ta001 --steps 100 --no-cpu-baseline --no-e2e > gpurun_out/ab_${v}_ta001_$rep.json 2>/dev/null
    timeout 300 python bench.py --target 4096 --steps 200 --no-cpu-baseline --no-e2e > gpurun_out/ab_${v}_4k_$rep.json 2>/dev/null
  done
done
unset FBB_LIB
python - <<'PY'
import json
for tag in ["", "_ta001", "_4k"]:
    for v in ["old", "new"]:
        vals = []
        for rep in (1, 2):
            try:
                d = json.load(open(f"gpurun_out/ab_{v}{tag}_{rep}.json"))
                vals.append((round(d["value"] / 1e6), round((d.get("e2e") or {}).get("value", 0) / 1e6)))
            except Exception as e:
                vals.append(("fail", str(e)[:40]))
        print(tag or "_ta021", v, vals)
PY
