set -x
ETUNE_ROWSEL_TRACE=1 python scripts/rows_timing.py --forms rows --iters 3 --no-fresh > gpurun_out/r02g_trace.log 2>&1
python scripts/rows_timing.py --forms rows > gpurun_out/r02g_timing.log 2>&1
python -m pytest tests/test_gpu_rows.py tests/test_gpu_sharded.py -x -q 2>&1 | tail -25 > gpurun_out/r02g_rows.log
ncu --set full --clock-control none --import-source on -k regex:"score_select_rows" -c 2 -o gpurun_out/r02g_rows python scripts/rows_timing.py --forms rows --iters 2 --no-fresh > gpurun_out/r02g_ncu_full.log 2>&1
