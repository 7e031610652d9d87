# Round-6 profile capture (run under gpurun): bench launch list, then one
# ncu --set full launch of each hot fast-numerics kernel (voxel-sorted storage).
cd $GRAFT_REPO_ROOT
python bench.py --steps 2 --warmup 1 --cpu-seconds 1 --no-extras > gpurun_out/b_small.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/r6_launches.csv python bench.py --steps 2 --warmup 1 --cpu-seconds 1 --no-extras > gpurun_out/ncu_launch.log 2>&1
cap() {  # cfg kernel skip tag
  ncu --set full --clock-control none --import-source on -k regex:"^$2" --launch-skip $3 -c 1 -o gpurun_out/r6_$4 -f python tools/profile_step.py $1 fast 50 > gpurun_out/ncu_$4.log 2>&1
  ncu -i gpurun_out/r6_$4.ncu-rep --page raw --csv > gpurun_out/raw_r6_$4.csv 2>/dev/null
  ncu -i gpurun_out/r6_$4.ncu-rep --page details --csv > gpurun_out/details_r6_$4.csv 2>/dev/null
  rm -f gpurun_out/r6_$4.ncu-rep   # (gpurun copies back <= 64 MiB)
}
cap 1 k_plane_seg 12 c1_plane
cap 1 k_zcols_seg 12 c1_z
cap 1 k_velocity_direct 1 c1_vel
cap 1 k_bin_fix 2 c1_binfix
cap 1 k_scan_lookback 2 c1_scan
cap 1 k_integrate_count 1 c1_integrate
cap 3 k_plane_seg 12 c3_plane
cap 3 k_zcols_segw 12 c3_z
cap 3 k_bin_fix 2 c3_binfix
cap 3 k_velocity_direct 1 c3_vel
cap 2 k_velocity_quad 1 c2_vel
python tools/ncu_summary.py gpurun_out/r6_ncu_full_summary.json gpurun_out/raw_r6_*.csv
du -sh gpurun_out; ls gpurun_out | wc -l
