cd $GRAFT_REPO_ROOT
python tools/seg_phases.py 1 > gpurun_out/seg_phases1.log 2>&1
python tools/seg_phases.py 3 > gpurun_out/seg_phases3.log 2>&1
for k in k_velocity_direct k_gather_fast k_bin_fix k_scan_lookback; do
  ncu --set full --clock-control none --import-source on -k regex:"^$k" --launch-skip 1 -c 1 -o gpurun_out/c1f_$k -f python tools/profile_step.py 1 fast > gpurun_out/ncu_c1f_$k.log 2>&1
  ncu -i gpurun_out/c1f_$k.ncu-rep --page raw --csv > gpurun_out/raw_c1f_$k.csv 2>/dev/null
done
python tools/fast_check.py 1 2
cat gpurun_out/seg_phases1.log gpurun_out/seg_phases3.log
