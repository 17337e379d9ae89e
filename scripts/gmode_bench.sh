# bench step + score_only with the L1-allocating (gmode 0) and L2-only (gmode 1) row gathers; row/select tests
TAG=${1:-gb}
O=gpurun_out/${TAG}_gmode_bench.log
: > $O
for m in 0 1 0 1; do
  r=$(ETUNE_ROWSEL_GMODE=$m python bench.py --no-cpu-baseline --no-e2e --no-search --no-reproduce --no-sweep --steps 400 2>/dev/null | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1e3,2), round(d['eager_ms_per_step']*1e3,2), round(d['score_only']['ms_per_step']*1e3,2), round(d['feature_mode']['ms_per_step']*1e3,2))")
  echo "gmode $m: step graph/eager us, score_only us, feature us: $r" >> $O
done
timeout 600 python -m pytest tests/test_gpu_rows.py tests/test_gpu_select.py -x -q > gpurun_out/${TAG}_tests.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_tests.log
