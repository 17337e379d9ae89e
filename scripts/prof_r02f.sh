set -x
ETUNE_ROWSEL_TRACE=1 python scripts/rows_timing.py --forms rows --iters 3 --no-fresh > gpurun_out/r02f_trace.log 2>&1
python scripts/rows_timing.py --forms rows > gpurun_out/r02f_timing.log 2>&1
python -m pytest tests/test_gpu_rows.py -x -q 2>&1 | tail -5 > gpurun_out/r02f_rows.log
