# compute-sanitizer passes over the GPU tests and the training kernels; logs in gpurun_out/
TAG=${1:-r}
CS=/usr/local/cuda/bin/compute-sanitizer
O=gpurun_out/sanitizers_$TAG.log
: > $O
run() { echo "\$ $*" >> $O; timeout 1500 "$@" > gpurun_out/san_tmp.log 2>&1; echo "rc=$?" >> gpurun_out/san_tmp.log;
        grep -E "passed|failed|SUMMARY|rc=" gpurun_out/san_tmp.log | tail -4 >> $O; }
run $CS --tool memcheck python -m pytest tests -m gpu -x -q -p no:cacheprovider
run $CS --tool racecheck python scripts/train_once.py 4096 2
run env ETUNE_TRAIN_MEGA=1 $CS --tool racecheck python scripts/train_once.py 4096 2
run $CS --tool racecheck python -m pytest tests/test_gpu_select.py -q -p no:cacheprovider -k "bred_population or heavy_ties"
run $CS --tool synccheck python -m pytest tests/test_gpu_select.py tests/test_gpu_train.py -q -p no:cacheprovider
run env ETUNE_TRAIN_MEGA=1 $CS --tool synccheck python scripts/train_once.py 4096 2
