mkdir -p gpurun_out
for v in r8nb4 r16nb4; do
lib=paper_1701_04148_b200/_lib/$v/libsfsketch_cuda.so
SFK_LIB_PATH=$lib timeout 600 ncu --set full --import-source on --clock-control none -k regex:min_query_cw -c 1 -f -o /tmp/ncu_cw_$v python tools/query_bench.py 200000000 1.0 4 > gpurun_out/q4_ncu_$v.log 2>&1
python tools/ncu_summary.py /tmp/ncu_cw_$v.ncu-rep > gpurun_out/q4_sum_$v.txt
ncu -i /tmp/ncu_cw_$v.ncu-rep --page source --csv --print-source sass > gpurun_out/q4_src_$v.csv 2>/dev/null
done
