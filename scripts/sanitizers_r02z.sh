# compute-sanitizer passes over the round-2 kernels (fused select with exact crossing placement,
# feature mode, block-parallel reproduce with epochs, shard merge, Gaussian sim sampler)
TAG=${1:-r02z}
CS=/usr/local/cuda/bin/compute-sanitizer
O=gpurun_out/sanitizers_$TAG.log
: > $O
run() { echo "\$ $*" >> $O; timeout 1500 "$@" > gpurun_out/san_tmp.log 2>&1; echo "rc=$?" >> gpurun_out/san_tmp.log;
        grep -E "passed|failed|ERROR SUMMARY|rc=" gpurun_out/san_tmp.log | tail -4 >> $O; }
run $CS --tool memcheck python -m pytest tests/test_gpu_rows.py tests/test_gpu_reproduce.py tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "not 2097152"
run $CS --tool racecheck python -m pytest tests/test_gpu_rows.py -x -q -p no:cacheprovider -k "golden or fresh or edges"
run $CS --tool synccheck python -m pytest tests/test_gpu_rows.py -x -q -p no:cacheprovider -k "golden or fresh or edges"
run $CS --tool racecheck python -m pytest tests/test_gpu_reproduce.py -x -q -p no:cacheprovider -k "not counter_mode_speed"
run $CS --tool memcheck python scripts/merge_timing.py 8 1024
run $CS --tool racecheck python scripts/merge_timing.py 8 1024
run $CS --tool memcheck python -m pytest tests/test_gpu_search.py -x -q -p no:cacheprovider
cat $O
