# step kernel: cooperative vs plain launch (graph / eager us per step), C2 2^20
O=gpurun_out/coop_ab.log
: > $O
run() {
  r=$(env "$@" python bench.py --no-cpu-baseline --no-e2e --no-search --no-reproduce --no-sweep --steps 400 2>/dev/null | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1e3,2), round(d['eager_ms_per_step']*1e3,2))")
  echo "$*: $r" >> $O
}
for rep in 1 2 3; do run ETUNE_ROWSEL_REGULAR=0; run ETUNE_ROWSEL_REGULAR=1; done
