B="python bench.py --steps 2 --warmup 2 --no-cpu-baseline --no-e2e --no-search --no-sweep --no-reproduce --bufs 2"
timeout 400 ncu --set full --cache-control none --clock-control none --import-source on --warp-sampling-interval 0 --warp-sampling-buffer-size 536870912 -k regex:score_select_rows -s 4 -c 1 -o gpurun_out/${1}_step $B > gpurun_out/${1}_ncu.log 2>&1
