# e2e after the fused output copy-out and the quarter final chunk: host split per call + host-path tests
O=gpurun_out/e2e_ab.log
: > $O
for rep in 1 2; do
  ETUNE_E2E_TRACE=1 python scripts/e2e_trace.py 2>&1 | grep -v Warn | tail -4 >> $O
done
python bench.py --no-cpu-baseline --no-search --no-reproduce --no-sweep --steps 200 2>/dev/null | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); e=d['e2e']; print('bench e2e', e['value']/1e9, e['ms_per_step'], 'pinned', e['pinned']['value']/1e9, e['pinned']['ms_per_step'], e['h2d_bytes_per_step'], e['pinned']['h2d_bytes_per_step'])" >> $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_rows.py tests/test_gpu_select.py -x -q 2>&1 | tail -2 >> $O
