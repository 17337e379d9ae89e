# phase A of the step kernel: cold (16 population buffers cycled) vs L2-hot (one buffer) inputs,
# whole step vs phase A alone; per-CTA trace with per-SM-bucket means
TAG=${1:-pa}
O=gpurun_out/${TAG}_phase_a.log
: > $O
for b in 16 1; do
  echo "== bufs $b trace" >> $O
  ETUNE_ROWSEL_TRACE=100 python scripts/step_enqueue.py --iters 100 --bufs $b 2>&1 | head -24 >> $O
  echo "== bufs $b phase A only trace (results invalid)" >> $O
  ETUNE_ROWSEL_ONLY_A=1 ETUNE_ROWSEL_TRACE=100 python scripts/step_enqueue.py --iters 100 --bufs $b 2>&1 | head -24 >> $O
  echo "== bufs $b timing" >> $O
  python scripts/step_enqueue.py --bufs $b >> $O 2>&1
done
