mkdir -p gpurun_out
for v in main nost; do
  if [ $v = main ]; then lib=paper_1701_04148_b200/_lib/libsfsketch_cuda.so; else lib=paper_1701_04148_b200/_lib/$v/libsfsketch_cuda.so; fi
  SFK_LIB_PATH=$lib timeout 300 python tools/api_overhead.py | sed "s/^/$v /" >> gpurun_out/w3.log 2>&1
done
