mkdir -p gpurun_out
lib=paper_1701_04148_b200/_lib/kpl8nbk4/libsfsketch_cuda.so
SFK_LIB_PATH=$lib timeout 600 ncu --set full --import-source on --clock-control none -k regex:min_query_cw -c 1 -f -o gpurun_out/ncu_cw_kpl8nbk4 python tools/query_bench.py 200000000 1.0 4 > gpurun_out/q2_ncu.log 2>&1
echo rc=$? >> gpurun_out/q2_ncu.log
