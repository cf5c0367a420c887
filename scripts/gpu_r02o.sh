#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "device_planned or direct_placement or large_traces" > gpurun_out/pytest_o.txt 2>&1; tail -4 gpurun_out/pytest_o.txt
for T in 4096 16384 262144; do
  timeout 300 python bench.py --target $T --steps 200 --no-cpu-baseline > gpurun_out/o_host_$T.json 2>/dev/null
  FBB_DEVICE_LOOP=1 timeout 300 python bench.py --target $T --steps 200 --no-cpu-baseline > gpurun_out/o_dl_$T.json 2>/dev/null
done
python - <<'PY'
import json
for f in ["o_host_4096", "o_dl_4096", "o_host_16384", "o_dl_16384", "o_host_262144", "o_dl_262144"]:
    try:
        d = json.load(open(f"gpurun_out/{f}.json"))
        print(f, round(d["value"] / 1e6), round(d["e2e"]["value"] / 1e6), {k: round(v, 4) for k, v in d["e2e"]["per_round_ms"].items()}, d["e2e"]["rounds_match_device_explorer"])
    except Exception as e:
        print(f, "fail", e)
PY
