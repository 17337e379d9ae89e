# where the step kernel computes the candidate ids (ETUNE_ROWSEL_IDS=a,b,c: j < a in phase A, [a, b) inside barrier 1,
# [b, c) inside barrier 2, j >= c in phase D's round trip): graph and eager us per step, C2 2^20
for sp in 0,4,7 0,4,6 0,4,5 0,5,6 0,5,7 0,4,4 0,3,6; do
  r=$(ETUNE_ROWSEL_IDS=$sp python bench.py --no-cpu-baseline --no-e2e --no-search --no-reproduce --no-sweep --steps 400 2>/dev/null | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1e3,2), round(d['eager_ms_per_step']*1e3,2))")
  echo "$sp $r"
done
