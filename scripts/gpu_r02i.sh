#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "solve or leaf or direct_placement or device_planned" > gpurun_out/pytest_i.txt 2>&1; tail -2 gpurun_out/pytest_i.txt
timeout 300 python bench.py --instance ta001 --no-cpu-baseline > gpurun_out/i_ta001.json 2>/dev/null
FBB_DIRECT=0 timeout 300 python bench.py --instance ta001 --no-cpu-baseline > gpurun_out/i_ta001_nodirect.json 2>/dev/null
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/i_ta021.json 2>/dev/null
python scripts/show.py gpurun_out/i_*.json
python - <<'PY'
import json
for f in ["i_ta001", "i_ta021"]:
    d = json.load(open(f"gpurun_out/{f}.json")); print(f, d["e2e"].get("per_round_ms"), d.get("e2e_reference_api"))
PY
