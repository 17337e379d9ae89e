python scripts/breed_par_diag.py 1048576 5 4.5 > gpurun_out/bd.log 2>&1
ETUNE_BREED_PAR_PROF=1 python scripts/breed_par_diag.py 1048576 5 > gpurun_out/bd_prof.log 2>&1
timeout 900 python -m pytest tests/test_gpu_reproduce.py -x -q > gpurun_out/bp_tests.log 2>&1
