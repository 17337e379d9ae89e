for m in 0 1 0 1; do
  r=$(ETUNE_ROWSEL_KHK=$m python bench.py --no-cpu-baseline --no-e2e --no-search --no-reproduce --no-sweep --steps 400 2>/dev/null | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1e3,2), round(d['eager_ms_per_step']*1e3,2))")
  echo "khk=$m $r"
done
ETUNE_ROWSEL_KHK=1 timeout 600 python -m pytest tests/test_gpu_rows.py -q -x -k "bench or edges"
