for i in 1 2; do
  for C in 128 160 192; do
    FBB_K2_CMAX=$C python bench.py --instance ta081 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('ta081 cmax $C', round(d['value']/1e6,1), round(d['ms_per_step']*1e3,2))"
  done
  for C in 224 256; do
    FBB_K2_CMAX=$C python bench.py --instance ta101 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('ta101 cmax $C', round(d['value']/1e6,1), round(d['ms_per_step']*1e3,2))"
  done
done
