mkdir -p gpurun_out
timeout 900 ncu --kernel-name regex:blk_bucket_k --launch-skip 170 --launch-count 1 --set full --warp-sampling-interval 0 --import-source on --clock-control none -o gpurun_out/blk_ncu -f python tools/blk_probe.py > gpurun_out/blk_ncu.log 2>&1; echo "rc=$?" >> gpurun_out/blk_ncu.log
ncu -i gpurun_out/blk_ncu.ncu-rep --page source --csv --print-source sass > gpurun_out/blk_src.csv 2>/dev/null
ncu -i gpurun_out/blk_ncu.ncu-rep --page raw --csv > gpurun_out/blk_raw.csv 2>/dev/null
