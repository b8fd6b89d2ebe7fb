mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_query_paths.py -x -q > gpurun_out/q11_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/q11_pytest.log
timeout 300 python tools/query_bench.py 1000000000 0.0,1.0 3,4 u64 > gpurun_out/q11_bench.log 2>&1
timeout 300 python tools/query_bench.py 1000000000 1.0 4 >> gpurun_out/q11_bench.log 2>&1
