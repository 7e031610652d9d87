# Round-8 final capture (run under gpurun): GPU suite, smoke, bench line,
# reference arm, kernel timelines, and --set full of the pipelined plane kernel.
cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r8b_gputest.log 2>&1; echo tests=$?
tail -1 gpurun_out/r8b_gputest.log
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r8b_smoke.log 2>&1; echo smoke=$?
timeout 600 python bench.py > gpurun_out/r8b_bench.log 2>&1; echo bench=$?
tail -1 gpurun_out/r8b_bench.log > gpurun_out/r8b_bench.json
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r8b_ref.log 2>&1; echo ref=$?
tail -1 gpurun_out/r8b_ref.log > gpurun_out/r8b_bench_reference.json
for c in 1 3; do timeout 200 python tools/timeline.py $c fast 2>&1 | grep -v "Warn\|_warn_once\|profiler.py" > gpurun_out/r8b_timeline_c$c.txt; done
rm -f gpurun_out/timeline_c*.json
cap() {  # cfg kernel skip tag
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:"^$2" --launch-skip $3 -c 1 -o gpurun_out/r8b_$4 -f python tools/profile_step.py $1 fast 50 > gpurun_out/ncu_$4.log 2>&1
  ncu -i gpurun_out/r8b_$4.ncu-rep --page raw --csv > gpurun_out/raw_r8b_$4.csv 2>/dev/null
  rm -f gpurun_out/r8b_$4.ncu-rep
}
cap 1 k_plane_seg 12 c1_plane
cap 3 k_plane_seg 12 c3_plane
python tools/ncu_summary.py gpurun_out/r8b_ncu_full_summary.json gpurun_out/raw_r8b_*.csv
du -sh gpurun_out
