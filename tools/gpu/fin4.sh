# round-2 final evidence (after the last cfg-4 / CU changes)
cd $GRAFT_REPO_ROOT
bash tools/gpu/full2.sh r02g
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02g_bench_ref.json 2> gpurun_out/r02g_bench_ref.err; echo "rc=$?" >> gpurun_out/r02g_bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file /tmp/l4.csv python tools/build_probe.py sf1 1.0 4 > /dev/null 2>&1
python tools/launch_sum.py /tmp/l4.csv > gpurun_out/r02g_launches_cfg4.txt
timeout 900 python tools/config_sweep.py 2 4 > gpurun_out/r02g_config_sweep_24.jsonl 2> gpurun_out/r02g_config_sweep_24.err
