mkdir -p gpurun_out
SFK_LIB_PATH=paper_1701_04148_b200/_lib/xb8/libsfsketch_cuda.so timeout 600 python -m pytest tests/test_gpu_query_paths.py -x -q -k "CW or 4-" > gpurun_out/q7_pytest.log 2>&1
for v in r8nb4 xb8 xb8n2 xb16; do
  lib=paper_1701_04148_b200/_lib/$v/libsfsketch_cuda.so
  echo "== $v" >> gpurun_out/q7_bench.log
  SFK_LIB_PATH=$lib timeout 300 python tools/query_bench.py 1000000000 0.0,1.0 4 >> gpurun_out/q7_bench.log 2>&1
done
