mkdir -p gpurun_out
for v in kpl8nbk4 r16nb2 r16nb4 r8nb4 r16nw12; do
  lib=paper_1701_04148_b200/_lib/$v/libsfsketch_cuda.so
  echo "== $v" >> gpurun_out/q3_bench.log
  SFK_LIB_PATH=$lib timeout 300 python tools/query_bench.py 1000000000 0.0,1.0,3.0 4 >> gpurun_out/q3_bench.log 2>&1
done
