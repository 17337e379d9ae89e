set -x
ETUNE_ROWSEL_TRACE=1 python scripts/rows_timing.py --forms rows --iters 3 --no-fresh > gpurun_out/r02v_trace.log 2>&1
python scripts/rows_timing.py --forms rows > gpurun_out/r02v_timing.log 2>&1
python scripts/rows_timing.py --forms rows --op mm:1,512,3072,768 --model c3_bert_ffn >> gpurun_out/r02v_timing.log 2>&1
python -m pytest tests/test_gpu_rows.py tests/test_gpu_sharded.py tests/test_gpu_reproduce.py tests/test_gpu_binding.py -x -q -s 2>&1 | tail -30 > gpurun_out/r02v_tests.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02v_smoke.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:merge --csv --log-file gpurun_out/r02v_merge.csv python scripts/merge_timing.py 8 1024 > gpurun_out/r02v_merge.log 2>&1
python scripts/merge_timing.py 8 1024 >> gpurun_out/r02v_merge.log 2>&1
