# row-record gather cache policy of the step kernel (ETUNE_ROWSEL_GMODE 0..3): device time per step and trace
TAG=${1:-gm}
O=gpurun_out/${TAG}_gmode.log
: > $O
for m in 0 1 2 3 0; do
  echo "== gmode $m" >> $O
  ETUNE_ROWSEL_GMODE=$m python scripts/step_enqueue.py 2>&1 | grep -v Warn >> $O
  ETUNE_ROWSEL_GMODE=$m ETUNE_ROWSEL_TRACE=100 python scripts/step_enqueue.py --iters 100 2>&1 | head -20 | grep "A done\|A1 issued \|x0 last\|sync1\|ranked" >> $O
done
