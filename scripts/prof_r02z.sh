set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
ETUNE_ROWSEL_TRACE=1 python scripts/rows_timing.py --forms rows --iters 5 --no-fresh > gpurun_out/r02z_trace.log 2>&1
ETUNE_ROWSEL_ONLY_A=1 python scripts/rows_timing.py --forms rows --no-fresh > gpurun_out/r02z_onlya.log 2>&1
python scripts/rows_timing.py --forms rows --no-fresh > gpurun_out/r02z_timing.log 2>&1
