# same-box A/B of two step-kernel builds (lib/ab/old.so vs lib/ab/new.so): graph / eager us per step
O=gpurun_out/lib_ab_step.log
: > $O
L=paper_2411_18873_b200/lib
cp $L/libetune_cuda.so $L/ab/cur.so
for rep in 1 2 3; do for v in old new; do
  cp $L/ab/$v.so $L/libetune_cuda.so
  r=$(python bench.py --no-cpu-baseline --no-e2e --no-search --no-reproduce --no-sweep --steps 400 2>/dev/null | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1e3,3), round(d['eager_ms_per_step']*1e3,2))")
  echo "$v: $r" >> $O
done; done
cp $L/ab/cur.so $L/libetune_cuda.so
timeout 900 python -m pytest tests/test_gpu_rows.py tests/test_gpu_select.py -x -q 2>&1 | tail -1 >> $O
