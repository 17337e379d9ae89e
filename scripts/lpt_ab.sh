# exact reproduce at 2^20: last wave longest first (default) vs plain item order (ETUNE_BREED_PAR_LPT=0)
O=gpurun_out/lpt_ab.log
: > $O
for rep in 1 2 3; do for v in 1 0; do
  r=$(ETUNE_BREED_PAR_LPT=$v python scripts/breed_once.py 1048576 1024 2>&1 | grep "^reproduce")
  echo "LPT=$v: $r" >> $O
done; done
python scripts/breed_par_timing.py 2>&1 | grep -v Warn >> $O
timeout 900 python -m pytest tests/test_gpu_reproduce.py -x -q 2>&1 | tail -1 >> $O
