# Round-6 second capture (under gpurun): the bench launch list with the
# final kernels and ncu --set full of config 4's fast streaming kernels.
cd $GRAFT_REPO_ROOT
ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/r6b_launches.csv python bench.py --steps 2 --warmup 1 --cpu-seconds 1 --no-extras > gpurun_out/ncu_launch.log 2>&1
cap() {  # cfg kernel skip tag
  ncu --set full --clock-control none --import-source on -k regex:"$2" --launch-skip $3 -c 1 -o gpurun_out/r6_$4 -f python tools/profile_step.py $1 fast 50 > gpurun_out/ncu_$4.log 2>&1
  ncu -i gpurun_out/r6_$4.ncu-rep --page raw --csv > gpurun_out/raw_r6_$4.csv 2>/dev/null
  ncu -i gpurun_out/r6_$4.ncu-rep --page details --csv > gpurun_out/details_r6_$4.csv 2>/dev/null
  rm -f gpurun_out/r6_$4.ncu-rep
}
cap 4 k_xrows_seg 12 c4_xrows
cap 4 k_ycols_segw 12 c4_ycols
cap 4 k_zcols_nz 12 c4_z
cap 1 k_velocity_compact 1 c1_velc
cap 1 k_bin_fix 2 c1_binfix2
python tools/ncu_summary.py gpurun_out/r6b_ncu_summary.json gpurun_out/raw_r6_c4_*.csv gpurun_out/raw_r6_c1_velc.csv gpurun_out/raw_r6_c1_binfix2.csv
du -sh gpurun_out
