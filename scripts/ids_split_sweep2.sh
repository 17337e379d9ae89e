# where the step kernel computes the candidate ids, after the L2-only gathers (ETUNE_ROWSEL_IDS=a,b,c;
# a < 0: ids of j < -a between issuing and consuming the row gathers): graph and eager us per step, C2 2^20
O=gpurun_out/ids_split2.log
: > $O
for rep in 1 2; do
for sp in 0,4,8 -1,4,8 -2,4,8 -4,4,8 1,4,8 2,4,8 0,4,7 0,5,8 -2,5,8 -4,5,8 -7,7,8; do
  r=$(ETUNE_ROWSEL_IDS=$sp python bench.py --no-cpu-baseline --no-e2e --no-search --no-reproduce --no-sweep --steps 400 2>/dev/null | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1e3,2), round(d['eager_ms_per_step']*1e3,2))")
  echo "$sp $r" >> $O
done; done
ETUNE_ROWSEL_IDS=-2,4,8 timeout 600 python -m pytest tests/test_gpu_rows.py -x -q 2>&1 | tail -1 >> $O
