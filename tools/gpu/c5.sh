mkdir -p gpurun_out
for rep in 1 2; do
for v in main su0; do
  if [ $v = main ]; then lib=paper_1701_04148_b200/_lib/libsfsketch_cuda.so; else lib=paper_1701_04148_b200/_lib/$v/libsfsketch_cuda.so; fi
  for args in "sff 1.0" "sff 0.5" "sf1 1.0 4" "sf1 1.0 1" "sf4 1.0"; do
    SFK_LIB_PATH=$lib timeout 300 python tools/build_probe.py $args | sed "s/^/$v /" >> gpurun_out/c5_probe.log 2>&1
  done
done
done
