# rowtab_build_kernel: lanes per row of the compact walk (ETUNE_BUILD_LANES), fresh-model step profile
O=gpurun_out/build_lanes.txt
: > $O
for L in 1 2 4 8; do
  echo "== lanes $L" >> $O
  ETUNE_BUILD_LANES=$L python scripts/fresh_profile.py 2>&1 | grep -v Warn | grep "host wall\|rowtab_build\|sum of" >> $O
done
