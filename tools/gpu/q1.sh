set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/q1_smi.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_query_paths.py -x -q > gpurun_out/q1_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/q1_pytest.log
for v in main nw8nbk4 kpl8 kpl8nbk4; do
  if [ $v = main ]; then lib=paper_1701_04148_b200/_lib/libsfsketch_cuda.so; else lib=paper_1701_04148_b200/_lib/$v/libsfsketch_cuda.so; fi
  echo "== $v" >> gpurun_out/q1_bench.log
  SFK_LIB_PATH=$lib timeout 300 python tools/query_bench.py 1000000000 0.0,1.0 3,4 >> gpurun_out/q1_bench.log 2>&1
done
