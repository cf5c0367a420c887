#!/bin/bash
# same-box A/B over instances: working tree vs libflowbb_b200_ab_old.so (AB_INST="ta101 ta081")
mkdir -p gpurun_out
OLD=$PWD/paper_1206_4973_b200/libflowbb_b200_ab_old.so
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "${AB_TESTS:-large_traces or k2}" > gpurun_out/pytest_ab.txt 2>&1; tail -2 gpurun_out/pytest_ab.txt
for rep in 1 2; do
  for v in old new; do
    if [ $v = old ]; then export FBB_LIB=$OLD; else unset FBB_LIB; fi
    for I in ${AB_INST:-ta101 ta081}; do
      timeout 300 python bench.py --instance $I --steps 100 --no-cpu-baseline --no-e2e > gpurun_out/ab2_${v}_${I}_$rep.json 2>/dev/null
    done
  done
done
unset FBB_LIB
python - <<PY
import json
for I in "${AB_INST:-ta101 ta081}".split():
    for v in ["old", "new"]:
        vals = []
        for rep in (1, 2):
            try:
                d = json.load(open(f"gpurun_out/ab2_{v}_{I}_{rep}.json")); vals.append(round(d["value"] / 1e6))
            except Exception as e:
                vals.append("fail")
        print(I, v, vals)
PY
