# round-2 final evidence: suite, smoke, bench (both arms), bench launch list, config sweep
cd $GRAFT_REPO_ROOT
bash tools/gpu/full2.sh r02f
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02f_bench_ref.json 2> gpurun_out/r02f_bench_ref.err; echo "rc=$?" >> gpurun_out/r02f_bench_ref.err
O=gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file /tmp/launches_bench.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $O/r02f_launches_bench.log 2>&1
python tools/launch_sum.py /tmp/launches_bench.csv > $O/r02f_launches_bench_summary.txt
timeout 1800 python tools/config_sweep.py 1 2 3 4 5 > $O/r02f_config_sweep.jsonl 2> $O/r02f_config_sweep.err; echo "rc=$?" >> $O/r02f_config_sweep.err
