#!/bin/bash
# BASELINE configs[1]: Ta021 pool-size sweep 4K..256K (+ beyond) on one B200, device and e2e.
mkdir -p gpurun_out
for T in 4096 8192 16384 32768 65536 131072 262144 524288 1048576; do
  timeout 600 python bench.py --target $T --steps 100 --no-cpu-baseline > gpurun_out/sweep_$T.json 2>/dev/null
done
python - <<'PY'
import json
print("| pool target | device bounded/s | ms/round | K2 share | e2e bounded/s |")
print("|---|---|---|---|---|")
for T in [4096, 8192, 16384, 32768, 65536, 131072, 262144, 524288, 1048576]:
    try:
        d = json.load(open(f"gpurun_out/sweep_{T}.json"))
    except Exception:
        continue
    print(f"| {T} | {d['value']/1e6:.1f} M | {d['ms_per_step']:.4f} | {d['roofline']['k2_share_of_round']:.3f} | {d['e2e']['value']/1e6:.1f} M |")
PY
