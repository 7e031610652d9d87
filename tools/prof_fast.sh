cd $GRAFT_REPO_ROOT
python tools/profile_step.py 1 fast || exit 1
for k in k_plane_seg k_zcols_seg k_velocity_direct k_exchange_affine k_gather_fast; do
  ncu --set full --clock-control none --import-source on -k regex:"^$k" --launch-skip 2 -c 1 -o gpurun_out/c1f_$k -f python tools/profile_step.py 1 fast > gpurun_out/ncu_c1f_$k.log 2>&1
  ncu -i gpurun_out/c1f_$k.ncu-rep --page raw --csv > gpurun_out/raw_c1f_$k.csv 2>/dev/null
done
for k in k_plane_seg k_zcols_seg; do
  ncu --set full --clock-control none --import-source on -k regex:"^$k" --launch-skip 2 -c 1 -o gpurun_out/c3f_$k -f python tools/profile_step.py 3 fast > gpurun_out/ncu_c3f_$k.log 2>&1
  ncu -i gpurun_out/c3f_$k.ncu-rep --page raw --csv > gpurun_out/raw_c3f_$k.csv 2>/dev/null
done
python tools/ncu_summary.py gpurun_out/fast_summary.json gpurun_out/raw_c1f_*.csv gpurun_out/raw_c3f_*.csv
cat gpurun_out/fast_summary.json | head -150
