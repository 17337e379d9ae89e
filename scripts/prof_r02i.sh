set -x
ETUNE_ROWSEL_ONLY_A=1 python scripts/rows_timing.py --forms rows --iters 20 --no-fresh > gpurun_out/r02i_onlya.log 2>&1
ETUNE_ROWSEL_ONLY_A=1 ncu --set full --clock-control none --cache-control none --import-source on -k regex:"score_select_rows" -s 5 -c 1 -o gpurun_out/r02i_a python scripts/rows_timing.py --forms rows --iters 8 --no-fresh > gpurun_out/r02i_ncu.log 2>&1
