mkdir -p gpurun_out
timeout 300 python tools/query_bench.py 1000000000 1.0 4 > gpurun_out/qn_bench.log 2>&1
timeout 900 ncu --kernel-name regex:min_query_cw --launch-skip 2 --launch-count 1 --set full --import-source on --clock-control none -o gpurun_out/qn_cw -f python tools/query_bench.py 1000000000 1.0 4 > gpurun_out/qn_ncu.log 2>&1; echo "rc=$?" >> gpurun_out/qn_ncu.log
python tools/ncu_summary.py gpurun_out/qn_cw.ncu-rep > gpurun_out/qn_cw_summary.txt 2>&1
rm -f gpurun_out/qn_cw.ncu-rep
