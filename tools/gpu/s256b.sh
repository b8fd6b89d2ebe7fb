mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_configs_full.py tests/test_gpu_baselines.py -x -q > gpurun_out/s256_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s256_pytest.log
rm -f gpurun_out/s256_probe.log
for rep in 1 2; do
for v in main old; do
  if [ $v = main ]; then lib=paper_1701_04148_b200/_lib/libsfsketch_cuda.so; else lib=paper_1701_04148_b200/_lib/$v/libsfsketch_cuda.so; fi
  for args in "sff 1.0" "sff 0.5" "sf1 1.2 4" "cu 1.0"; do
    SFK_LIB_PATH=$lib timeout 600 python tools/build_probe.py $args | sed "s/^/$v /" >> gpurun_out/s256_probe.log 2>&1
  done
done
done
