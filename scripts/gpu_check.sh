# one GPU round trip: parity tests, smoke, bench, launch list, full profile of the step kernel
set -x
TAG=${1:-r}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1
timeout 900 python bench.py --steps 200 --warmup 5 --cpu-seconds 8 > gpurun_out/bench_$TAG.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"score|rowtab|rs_|sel_|key_hash" -c 60 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-search --no-sweep --bufs 2 > gpurun_out/ncu_bench_$TAG.log 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:score_select_rows -s 4 -c 1 -o gpurun_out/prof_step_$TAG python bench.py --steps 2 --warmup 2 --no-cpu-baseline --no-e2e --no-search --no-sweep --bufs 2 > gpurun_out/ncu_full_$TAG.log 2>&1
ls gpurun_out | tail -5
