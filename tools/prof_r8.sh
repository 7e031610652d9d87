# Round-8 capture (run under gpurun): GPU tests, smoke, the bench line and the
# reference arm, the bench's ncu launch list, and one ncu --set full launch of
# each hot fast-numerics kernel (voxel-sorted storage), CSV exports only.
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r8_gputest.log 2>&1; echo tests=$?
tail -1 gpurun_out/r8_gputest.log
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r8_smoke.log 2>&1; echo smoke=$?
timeout 600 python bench.py > gpurun_out/r8_bench.log 2>&1; echo bench=$?
tail -1 gpurun_out/r8_bench.log > gpurun_out/r8_bench.json
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r8_ref.log 2>&1; echo ref=$?
tail -1 gpurun_out/r8_ref.log > gpurun_out/r8_bench_reference.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/r8_launches.csv python bench.py --steps 2 --warmup 1 --cpu-seconds 1 --no-extras > gpurun_out/r8_ncu_launch.log 2>&1; echo launches=$?
python tools/launch_table.py gpurun_out/r8_launches.csv > gpurun_out/r8_launches_summary.txt 2>&1
cap() {  # cfg kernel skip tag
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:"^$2" --launch-skip $3 -c 1 -o gpurun_out/r8_$4 -f python tools/profile_step.py $1 fast 50 > gpurun_out/ncu_$4.log 2>&1
  ncu -i gpurun_out/r8_$4.ncu-rep --page raw --csv > gpurun_out/raw_r8_$4.csv 2>/dev/null
  rm -f gpurun_out/r8_$4.ncu-rep
}
cap 1 k_plane_seg 12 c1_plane
cap 1 k_zcols_seg 12 c1_z
cap 1 k_velocity_compact 1 c1_vel
cap 3 k_plane_seg 12 c3_plane
cap 3 k_zcols_segw 12 c3_z
cap 2 k_velocity_quad 1 c2_vel
cap 4 k_xrows_seg 12 c4_xrows
cap 4 k_ycols_segw 12 c4_ycols
python tools/ncu_summary.py gpurun_out/r8_ncu_full_summary.json gpurun_out/raw_r8_*.csv
du -sh gpurun_out
