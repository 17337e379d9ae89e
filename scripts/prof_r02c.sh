set -x
python -m pytest tests/test_gpu_rows.py -x -q 2>&1 | tail -15 > gpurun_out/r02c_rows.log
python scripts/rows_timing.py --forms rows,keyed > gpurun_out/r02c_timing.log 2>&1
python scripts/rows_timing.py --forms rows --op mm:1,512,3072,768 --model c3_bert_ffn >> gpurun_out/r02c_timing.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02c_launches.csv python scripts/rows_timing.py --forms rows --iters 5 --no-fresh > gpurun_out/r02c_ncu_stdout.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"score_select_rows|rowtab_build_kernel|lsd_" -c 6 -o gpurun_out/r02c_rows python scripts/rows_timing.py --forms rows --iters 2 --no-fresh > gpurun_out/r02c_ncu_full.log 2>&1
python -m pytest tests/test_gpu_select.py tests/test_gpu_parity.py tests/test_gpu_search.py -x -q 2>&1 | tail -15 > gpurun_out/r02c_sel.log
