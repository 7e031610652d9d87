# Round-8 final capture (run under gpurun): GPU suite, smoke, bench line
# (deterministic resort amortisation), reference arm, bench launch list.
cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r8d_gputest.log 2>&1; echo tests=$?
tail -1 gpurun_out/r8d_gputest.log
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r8d_smoke.log 2>&1; echo smoke=$?
timeout 600 python bench.py > gpurun_out/r8d_bench.log 2>&1; echo bench=$?
tail -1 gpurun_out/r8d_bench.log > gpurun_out/r8d_bench.json
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r8d_ref.log 2>&1; echo ref=$?
tail -1 gpurun_out/r8d_ref.log > gpurun_out/r8d_bench_reference.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r8d_launches.csv python bench.py --steps 2 --warmup 1 --cpu-seconds 1 --no-extras > gpurun_out/r8d_ncu_launch.log 2>&1; echo launches=$?
python tools/launch_table.py gpurun_out/r8d_launches.csv > gpurun_out/r8d_launches_summary.txt 2>&1
du -sh gpurun_out
