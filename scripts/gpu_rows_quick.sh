# quick GPU loop for the step kernel: per-CTA phase trace, timing, row/select parity tests
TAG=${1:-q}
ETUNE_ROWSEL_TRACE=100 python scripts/step_enqueue.py --iters 100 > gpurun_out/${TAG}_trace.log 2>&1
python scripts/step_enqueue.py >> gpurun_out/${TAG}_trace.log 2>&1
timeout 600 python -m pytest tests/test_gpu_rows.py tests/test_gpu_select.py tests/test_gpu_sharded.py -x -q > gpurun_out/${TAG}_tests.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_tests.log
