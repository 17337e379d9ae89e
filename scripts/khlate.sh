# step kernel: per-key FNV states' bulk copy issued at the start (gmode 1) or after the row gathers (gmode 17)
O=gpurun_out/khlate.log
: > $O
run() {
  r=$(env "$@" python bench.py --no-cpu-baseline --no-e2e --no-search --no-reproduce --no-sweep --steps 400 2>/dev/null | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1e3,2), round(d['eager_ms_per_step']*1e3,2))")
  echo "$*: $r" >> $O
}
for rep in 1 2 3; do run ETUNE_ROWSEL_GMODE=1; run ETUNE_ROWSEL_GMODE=17; done
ETUNE_ROWSEL_GMODE=17 timeout 600 python -m pytest tests/test_gpu_rows.py -x -q 2>&1 | tail -1 >> $O
