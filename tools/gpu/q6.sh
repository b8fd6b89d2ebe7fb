mkdir -p gpurun_out
for v in r8nb4 e1 e2 e3; do
  lib=paper_1701_04148_b200/_lib/$v/libsfsketch_cuda.so
  echo "== $v" >> gpurun_out/q6_bench.log
  SFK_LIB_PATH=$lib timeout 300 python tools/query_bench.py 1000000000 1.0 4 >> gpurun_out/q6_bench.log 2>&1
done
