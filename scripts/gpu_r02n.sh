#!/bin/bash
mkdir -p gpurun_out
for T in 4096 262144; do
  timeout 300 python bench.py --target $T --steps 200 --no-cpu-baseline > gpurun_out/n_host_$T.json 2>/dev/null
  FBB_DEVICE_LOOP=1 timeout 300 python bench.py --target $T --steps 200 --no-cpu-baseline > gpurun_out/n_dl_$T.json 2>/dev/null
  FBB_DEVICE_LOOP=1 FBB_HOST_ROWS=full timeout 300 python bench.py --target $T --steps 200 --no-cpu-baseline > gpurun_out/n_dlfull_$T.json 2>/dev/null
done
python - <<'PY'
import json
for f in ["n_host_4096", "n_dl_4096", "n_dlfull_4096", "n_host_262144", "n_dl_262144", "n_dlfull_262144"]:
    try:
        d = json.load(open(f"gpurun_out/{f}.json"))
        print(f, round(d["value"] / 1e6), round(d["e2e"]["value"] / 1e6), {k: round(v, 4) for k, v in d["e2e"]["per_round_ms"].items()}, d["e2e"]["rounds_match_device_explorer"])
    except Exception as e:
        print(f, "fail", e)
PY
