set -x
timeout 300 python scripts/breed_par_timing.py > gpurun_out/bp_timing.log 2>&1
timeout 900 python -m pytest tests/test_gpu_reproduce.py -x -q > gpurun_out/bp_tests.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:breed --csv --log-file gpurun_out/bp_launches.csv python scripts/breed_par_timing.py > /dev/null 2>&1
