for ks in 1 0; do for pad in 0 16; do
  r=$(ETUNE_ROWSEL_KHASH_SMEM=$ks ETUNE_ROWSEL_PAD_KB=$pad python bench.py --no-cpu-baseline --no-e2e --no-search --no-reproduce --no-sweep --steps 400 2>/dev/null | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1e3,2), round(d['eager_ms_per_step']*1e3,2))")
  echo "khash_smem ${ks} pad ${pad} KB: $r"
done; done
