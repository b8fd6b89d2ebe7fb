mkdir -p gpurun_out
for v in main ch1 ch2; do
  if [ $v = main ]; then lib=paper_1701_04148_b200/_lib/libsfsketch_cuda.so; else lib=paper_1701_04148_b200/_lib/$v/libsfsketch_cuda.so; fi
  for a in 1.0 1.5; do
    SFK_LIB_PATH=$lib timeout 120 python tools/build_probe.py sff $a | sed "s/^/$v /" >> gpurun_out/c2_probe.log 2>&1
  done
done
SFK_NO_CHAIN=1 timeout 120 python tools/build_probe.py sff 1.0 | sed "s/^/nochain /" >> gpurun_out/c2_probe.log 2>&1
