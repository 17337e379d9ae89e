set -x
B="python bench.py --steps 2 --warmup 2 --no-cpu-baseline --no-e2e --no-search --no-sweep --no-reproduce --bufs 2"
timeout 400 ncu --set full --clock-control none --import-source on -k regex:score_select_rows -s 4 -c 1 -o gpurun_out/r02z_step $B > gpurun_out/r02z_ncu_full.log 2>&1
ETUNE_ROWSEL_ONLY_A=1 timeout 400 ncu --set full --clock-control none --import-source on -k regex:score_select_rows -s 4 -c 1 -o gpurun_out/r02z_stepA $B > gpurun_out/r02z_ncu_fullA.log 2>&1
