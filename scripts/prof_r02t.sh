set -x
python -m pytest tests/test_gpu_rows.py -q -x -k "host" 2>&1 | tail -3 > gpurun_out/r02t_tests.log
python bench.py --steps 100 --warmup 5 --cpu-seconds 8 --no-search --no-sweep > gpurun_out/r02t_bench.log 2>&1
