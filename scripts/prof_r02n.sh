set -x
ETUNE_ROWSEL_ONLY_A=1 python scripts/rows_timing.py --forms rows --iters 20 --no-fresh > gpurun_out/r02n_onlya.log 2>&1
ETUNE_ROWSEL_TRACE=1 python scripts/rows_timing.py --forms rows --iters 3 --no-fresh > gpurun_out/r02n_trace.log 2>&1
python scripts/rows_timing.py --forms rows > gpurun_out/r02n_timing.log 2>&1
python scripts/rows_timing.py --forms rows --op mm:1,512,3072,768 --model c3_bert_ffn >> gpurun_out/r02n_timing.log 2>&1
python -m pytest tests/test_gpu_rows.py tests/test_gpu_sharded.py tests/test_gpu_reproduce.py -x -q 2>&1 | tail -25 > gpurun_out/r02n_tests.log
