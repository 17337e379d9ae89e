for n in 1048576 524288 262144 65536 4096; do
  echo "n=$n"; ETUNE_ROWSEL_ONLY_A=1 python scripts/rows_timing.py --forms rows --iters 30 --no-fresh --n $n 2>&1 | grep -v "^\[" | cut -c1-120
  python scripts/rows_timing.py --forms rows --iters 30 --no-fresh --n $n 2>&1 | grep -v "^\[" | cut -c1-120
done > gpurun_out/r02o_scaling.log 2>&1
