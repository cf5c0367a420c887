#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for I in ta081; do timeout 600 python bench.py --instance $I --no-cpu-baseline --steps 100 > gpurun_out/q_$I.json 2>/dev/null; python scripts/show.py gpurun_out/q_$I.json; done
python - <<'PY'
import sys, time
sys.path.insert(0, ".")
import paper_1206_4973_b200 as fbb
for (n, m, seed, ub) in [(200, 20, 2013025619, 11195)]:
    inst = fbb.generate_instance(n, m, seed)
    r = fbb.resolve_workload(inst, [[]], ub, targets=[262144], max_rounds=12)
    print(n, m, [x[2] for x in r.rounds], r.elapsed_seconds)
PY
