mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_host_query.py -q > gpurun_out/hq_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/hq_pytest.log
timeout 1500 python tools/host_query_bench.py 1000000000 3:24:0:4:p 3:24:0:4:p:4 3:24:0:4:p:8 3:24:0:4:p:12 3:24:4:4:p:8 3:24:4:4:p:12 3:22:0:8:p:8 3:22:0:8:p 3:26:0:3:p:8 3:24:0:4:g:0:1 3:24:0:4:k:0:1 3:24:0:4:g:8:1 > gpurun_out/hq_bench.jsonl 2> gpurun_out/hq_bench.err; echo "rc=$?" >> gpurun_out/hq_bench.err
