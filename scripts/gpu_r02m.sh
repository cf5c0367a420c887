#!/bin/bash
# e2e (host-resident tree) A/B of the transfer switches
mkdir -p gpurun_out
timeout 300 python bench.py --steps 100 --no-cpu-baseline > gpurun_out/m_default.json 2>/dev/null
FBB_HOST_OUT=staged timeout 300 python bench.py --steps 100 --no-cpu-baseline > gpurun_out/m_out_staged.json 2>/dev/null
FBB_HOST_IN=copy timeout 300 python bench.py --steps 100 --no-cpu-baseline > gpurun_out/m_in_copy.json 2>/dev/null
FBB_HOST_IN=copy FBB_HOST_OUT=staged timeout 300 python bench.py --steps 100 --no-cpu-baseline > gpurun_out/m_both.json 2>/dev/null
FBB_PINNED_WC=1 timeout 300 python bench.py --steps 100 --no-cpu-baseline > gpurun_out/m_wc.json 2>/dev/null
timeout 300 python bench.py --steps 100 --no-cpu-baseline > gpurun_out/m_default2.json 2>/dev/null
python - <<'PY'
import json
for f in ["m_default", "m_out_staged", "m_in_copy", "m_both", "m_wc", "m_default2"]:
    try:
        d = json.load(open(f"gpurun_out/{f}.json"))
        print(f, round(d["value"] / 1e6), round(d["e2e"]["value"] / 1e6), d["e2e"]["per_round_ms"], d["e2e"]["rounds_match_device_explorer"])
    except Exception as e:
        print(f, "fail", e)
PY
