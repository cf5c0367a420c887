for i in 1 2 3; do
  for V in old new; do
    if [ $V = old ]; then export FBB_SUMMARY=copy; else unset FBB_SUMMARY; fi
    for I in ta021 ta001; do
    python bench.py --instance $I --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$V $I', round(d['value']/1e6,1), round(d['ms_per_step']*1e3,2))"
    done
  done
done
unset FBB_SUMMARY
python scripts/diag_e2e.py ta021
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
