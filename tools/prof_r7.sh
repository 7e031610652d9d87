# Round-7 captures (under gpurun): ncu --set full of the new bin fix-up and
# the exact / fast velocity kernels, CSV exports only (the .ncu-rep files are
# removed: gpurun_out is capped at 64 MiB).
cd $GRAFT_REPO_ROOT
cap() {  # cfg numerics kernel skip tag
  ncu --set full --clock-control none --import-source on -k regex:"$3" --launch-skip $4 -c 1 -o gpurun_out/r7_$5 -f python tools/profile_step.py $1 $2 50 > gpurun_out/ncu_$5.log 2>&1
  ncu -i gpurun_out/r7_$5.ncu-rep --page raw --csv > gpurun_out/raw_r7_$5.csv 2>/dev/null
  ncu -i gpurun_out/r7_$5.ncu-rep --page details --csv > gpurun_out/details_r7_$5.csv 2>/dev/null
  rm -f gpurun_out/r7_$5.ncu-rep
}
cap 3 fast k_bin_fix_g 2 c3_binfix
cap 1 fast k_bin_fix_g 2 c1_binfix
cap 3 fast k_velocity_compact 1 c3_velc
cap 1 exact k_velocity_exact 1 c1_vexact
cap 3 fast k_scan_lookback 2 c3_scan
python tools/ncu_summary.py gpurun_out/r7_ncu_summary.json gpurun_out/raw_r7_*.csv
du -sh gpurun_out
