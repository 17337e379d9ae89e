# feature mode: per-key records vs table-lookup kernel timing, parity tests, bench feature_mode line
python scripts/features_timing.py > gpurun_out/feat2.log 2>&1
ETUNE_FEATURES_TABLE=0 python scripts/features_timing.py >> gpurun_out/feat2.log 2>&1
python scripts/features_timing.py --op mm:1,512,3072,768 >> gpurun_out/feat2.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x >> gpurun_out/feat2.log 2>&1; echo "rc=$?" >> gpurun_out/feat2.log
