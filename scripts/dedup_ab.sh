# step kernel: in-thread row dedup of the gathers (ETUNE_ROWSEL_GMODE=1) vs every candidate gathered (17)
O=gpurun_out/dedup_ab.log
: > $O
run() {
  r=$(env "$@" python bench.py --no-cpu-baseline --no-e2e --no-search --no-reproduce --no-sweep --steps 400 2>/dev/null | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1e3,2), round(d['eager_ms_per_step']*1e3,2))")
  echo "$*: $r" >> $O
}
for rep in 1 2 3; do run ETUNE_ROWSEL_GMODE=1; run ETUNE_ROWSEL_GMODE=17; done
ETUNE_ROWSEL_TRACE=100 python scripts/step_enqueue.py --iters 100 2>&1 | grep "A done\|A1 issued \|sync1\|ranked\|prologue" | head -6 >> $O
timeout 900 python -m pytest tests/test_gpu_rows.py tests/test_gpu_select.py -x -q 2>&1 | tail -1 >> $O
