# same-box A/B of the e2e host pipeline: lib/ab/old.so vs lib/ab/new.so, pageable and pinned rows
O=gpurun_out/e2e_ab2.log
: > $O
L=paper_2411_18873_b200/lib
cp $L/libetune_cuda.so $L/ab/cur.so
for rep in 1 2 3; do for v in old new; do
  cp $L/ab/$v.so $L/libetune_cuda.so
  a=$(ETUNE_E2E_TRACE=1 python scripts/e2e_trace.py 2>&1 | grep "^call" | tail -6 | awk '{s+=$3} END {printf "%.3f", s/NR}')
  b=$(E2E_PINNED=1 ETUNE_E2E_TRACE=1 python scripts/e2e_trace.py 2>&1 | grep "^call" | tail -6 | awk '{s+=$3} END {printf "%.3f", s/NR}')
  echo "$v: pageable $a ms, pinned $b ms (mean of the last 6 calls)" >> $O
done; done
cp $L/ab/cur.so $L/libetune_cuda.so
