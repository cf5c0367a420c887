#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 600 oracle/_ref/dropin_test 2>&1 | tail -1
for V in 0 1; do
export FBB_DEVICE_LOOP=$V
timeout 600 python bench.py --no-cpu-baseline --steps 100 > gpurun_out/q_hl$V.json 2>/dev/null; echo -n "devloop=$V "; python scripts/show.py gpurun_out/q_hl$V.json | head -1
done
unset FBB_DEVICE_LOOP
timeout 300 python bench.py --mode exhaust --instance ta021 --max-seconds 100 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('exhaust', d['explore_seconds'], d['bounded'], d['proof'])"
FBB_DEVICE_LOOP=1 timeout 300 python bench.py --mode exhaust --instance ta021 --max-seconds 100 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('exhaust devloop', d['explore_seconds'], d['bounded'], d['proof'])"
