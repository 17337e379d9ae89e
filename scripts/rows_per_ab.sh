# score_rows_kernel: candidates per thread per pass 4 vs 8 (lib/ab/k4.so vs k8.so), score_only us
O=gpurun_out/rows_per_ab.log
: > $O
L=paper_2411_18873_b200/lib
cp $L/libetune_cuda.so $L/ab/cur.so
for rep in 1 2 3; do for v in k4 k8; do
  cp $L/ab/$v.so $L/libetune_cuda.so
  r=$(python bench.py --no-cpu-baseline --no-e2e --no-search --no-reproduce --no-sweep --steps 400 2>/dev/null | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['score_only']['ms_per_step']*1e3,2))")
  echo "$v: score_only $r us" >> $O
done; done
cp $L/ab/cur.so $L/libetune_cuda.so
timeout 900 python -m pytest tests/test_gpu_rows.py tests/test_gpu_parity.py -x -q 2>&1 | tail -1 >> $O
