for T in 4096 16384 65536 131072 262144; do
  for V in old new; do
    if [ $V = old ]; then export FBB_NO_ROUND_PPC=1; else unset FBB_NO_ROUND_PPC; fi
    python bench.py --target $T --steps 100 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$V $T', round(d['value']/1e6,1), round(d['ms_per_step']*1e3,1), 'us', round(d['roofline']['k2_share_of_round'],3))"
  done
done
unset FBB_NO_ROUND_PPC
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
