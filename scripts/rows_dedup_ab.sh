# score_rows_kernel (etune_cu_score, bench score_only): genome dedup within a thread's pass vs none
O=gpurun_out/rows_dedup_ab.log
: > $O
run() {
  r=$(env "$@" python bench.py --no-cpu-baseline --no-e2e --no-search --no-reproduce --no-sweep --steps 400 2>/dev/null | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['score_only']['ms_per_step']*1e3,2), round(d['ms_per_step']*1e3,2))")
  echo "$*: score_only us, step us: $r" >> $O
}
for rep in 1 2 3; do run ETUNE_ROWS_NODEDUP=0; run ETUNE_ROWS_NODEDUP=1; done
timeout 900 python -m pytest tests/test_gpu_rows.py tests/test_gpu_parity.py -x -q 2>&1 | tail -1 >> $O
