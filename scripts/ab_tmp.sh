for i in 1 2; do
  for C in 112 128 144 160 176 192; do
    FBB_K2_CMAX=$C python bench.py --instance ta001 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('ta001 cmax $C', round(d['value']/1e6,1), round(d['ms_per_step']*1e3,2), round(d['roofline']['k2_share_of_round'],3))"
  done
done
for C in 128 160; do
FBB_K2_CMAX=$C python bench.py --instance ta051 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('ta051 cmax $C', round(d['value']/1e6,1), round(d['ms_per_step']*1e3,2))"
done
