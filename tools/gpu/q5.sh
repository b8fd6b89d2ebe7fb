mkdir -p gpurun_out
for v in r8nb4 n24nb4 n24nb2 n20nb4 n32nb2; do
  lib=paper_1701_04148_b200/_lib/$v/libsfsketch_cuda.so
  echo "== $v" >> gpurun_out/q5_bench.log
  SFK_LIB_PATH=$lib timeout 300 python tools/query_bench.py 1000000000 0.0,1.0 4 >> gpurun_out/q5_bench.log 2>&1
done
