set -x
python -m pytest tests/test_gpu_rows.py -x -q 2>&1 | tail -5 > gpurun_out/r02b_rows.log
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02b_launches.csv python scripts/rows_timing.py --forms rows --iters 5 --no-fresh > gpurun_out/r02b_ncu_stdout.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"score_rows_kernel|rowtab_build_kernel|rowtab_classes_kernel|sel_" -c 8 -o gpurun_out/r02b_rows python scripts/rows_timing.py --forms rows --iters 2 --no-fresh > gpurun_out/r02b_ncu_full.log 2>&1
