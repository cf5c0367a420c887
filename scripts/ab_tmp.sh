for i in 1 2 3; do
  (cd _ab_old && python bench.py --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('old', round(d['value']/1e6,1), d['ms_per_step'])")
  python bench.py --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('new', round(d['value']/1e6,1), d['ms_per_step'])"
done
for I in ta081 ta001; do
  (cd _ab_old && python bench.py --instance $I --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('old $I', round(d['value']/1e6,1), d['ms_per_step'])")
  python bench.py --instance $I --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('new $I', round(d['value']/1e6,1), d['ms_per_step'])"
done
python scripts/diag_e2e.py ta021
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
