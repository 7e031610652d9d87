set -x
# Round profile capture (run under gpurun): the bench launch list plus one
# ncu --set full per hot kernel (tools/profile_step.py driver); KERNELS / SKIP
# select kernels and how many launches of each to skip.
python bench.py --steps 2 --warmup 1 --cpu-seconds 1 > gpurun_out/b_small.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r3_launches.csv python bench.py --steps 2 --warmup 1 --cpu-seconds 1 > gpurun_out/ncu_launch.log 2>&1
python tools/profile_step.py || exit 1
for k in ${KERNELS:-k_plane_xy_reg k_zcols_reg k_exchange_rec k_cand_lists k_velocity_cells k_bin_fix k_scan_lookback}; do
  ncu --set full --clock-control none --import-source on -k regex:"^$k" --launch-skip ${SKIP:-1} -c 1 -o gpurun_out/full_$k -f python tools/profile_step.py > gpurun_out/ncu_$k.log 2>&1
  ncu -i gpurun_out/full_$k.ncu-rep --page raw --csv > gpurun_out/raw_$k.csv 2>/dev/null
done
ls -la gpurun_out/
