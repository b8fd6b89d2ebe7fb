mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/c4_launches_cfg4.csv python tools/one_build.py sf1rec 1.0 1 > gpurun_out/c4.log 2>&1
python tools/launch_sum.py gpurun_out/c4_launches_cfg4.csv > gpurun_out/c4_launches_cfg4_summary.txt
