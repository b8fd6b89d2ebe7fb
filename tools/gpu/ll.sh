mkdir -p gpurun_out
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/ll_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cm > gpurun_out/ll_bench.log 2>&1; echo "rc=$?" >> gpurun_out/ll_bench.log
python tools/launch_sum.py gpurun_out/ll_launches.csv > gpurun_out/ll_launches_summary.txt
rm -f gpurun_out/ll_launches.csv
