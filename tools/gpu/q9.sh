mkdir -p gpurun_out
SFK_LIB_PATH=paper_1701_04148_b200/_lib/d16/libsfsketch_cuda.so timeout 600 python -m pytest tests/test_gpu_query_paths.py -x -q > gpurun_out/q9_pytest.log 2>&1
for v in d16 d16nb2 d16w12 d8; do
  lib=paper_1701_04148_b200/_lib/$v/libsfsketch_cuda.so
  echo "== $v" >> gpurun_out/q9_bench.log
  SFK_LIB_PATH=$lib timeout 300 python tools/query_bench.py 1000000000 0.0,1.0,3.0 4 >> gpurun_out/q9_bench.log 2>&1
done
