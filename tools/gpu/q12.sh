mkdir -p gpurun_out
for rep in 1 2; do
for v in main nb4 nw12 kpl8; do
  if [ $v = main ]; then lib=paper_1701_04148_b200/_lib/libsfsketch_cuda.so; else lib=paper_1701_04148_b200/_lib/$v/libsfsketch_cuda.so; fi
  echo "== $v" >> gpurun_out/q12_bench.log
  SFK_LIB_PATH=$lib timeout 300 python tools/query_bench.py 1000000000 0.0,1.0 4 >> gpurun_out/q12_bench.log 2>&1
done
done
