set -x
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02zb_gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02zb_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02zb_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/r02zb_bench.json 2> gpurun_out/r02zb_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r02zb_bench_ref.json 2> gpurun_out/r02zb_bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r02zb_launches.csv python bench.py --steps 3 --warmup 3 > gpurun_out/r02zb_ncu.log 2>&1
echo done
