for sp in 0,4 2,4 3,4 4,4 2,5 3,5 4,6 1,4; do
  r=$(ETUNE_ROWSEL_IDS=$sp python bench.py --no-cpu-baseline --no-e2e --no-search --no-reproduce --no-sweep --steps 400 2>/dev/null | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1e3,2), round(d['eager_ms_per_step']*1e3,2))")
  echo "$sp $r"
done
