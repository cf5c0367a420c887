#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multirank.py -q -x -k "traces or device_planned or direct_placement or group or solve" > gpurun_out/pytest_q.txt 2>&1; tail -4 gpurun_out/pytest_q.txt
for T in 4096 16384 262144; do
  FBB_DEVICE_LOOP=1 timeout 300 python bench.py --target $T --steps 200 --no-cpu-baseline > gpurun_out/q_dl_$T.json 2>/dev/null
done
python - <<'PY'
import json
for f in ["q_dl_4096", "q_dl_16384", "q_dl_262144"]:
    try:
        d = json.load(open(f"gpurun_out/{f}.json"))
        print(f, round(d["value"] / 1e6), round(d["e2e"]["value"] / 1e6), {k: round(v, 4) for k, v in d["e2e"]["per_round_ms"].items()}, d["e2e"]["rounds_match_device_explorer"])
    except Exception as e:
        print(f, "fail", e)
PY
timeout 900 python bench.py --mode exhaust --instance ta021 > gpurun_out/exhaust_ta021.json 2> gpurun_out/exhaust_ta021.err; tail -c 300 gpurun_out/exhaust_ta021.json
