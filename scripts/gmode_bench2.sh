# mixed gather policies and genome-load policies of the step kernel (graph/eager us per step)
TAG=${1:-gd}
O=gpurun_out/${TAG}_gmode_bench2.log
: > $O
run() {
  r=$(env "$@" python bench.py --no-cpu-baseline --no-e2e --no-search --no-reproduce --no-sweep --steps 400 2>/dev/null | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1e3,2), round(d['eager_ms_per_step']*1e3,2))")
  echo "$*: $r" >> $O
}
for rep in 1 2; do
for m in 0 1 4 5 6; do run ETUNE_ROWSEL_GMODE=$m; done
for x in 1 2; do run ETUNE_ROWSEL_GMODE=1 ETUNE_ROWSEL_XMODE=$x; done
done
