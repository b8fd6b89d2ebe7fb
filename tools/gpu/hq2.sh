mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_host_query.py -q > gpurun_out/hq_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/hq_pytest.log
timeout 1500 python tools/host_query_bench.py 1000000000 3:24:0:4:p 3:24:0:4:p:12 3:24:0:4:p:10 3:24:0:4:p:14 3:24:4:4:p 3:24:4:4:p:8 3:24:3:4:p:10 3:23:0:4:p 3:23:4:6:p 2:24:0:4:p > gpurun_out/hq_bench2.jsonl 2> gpurun_out/hq_bench2.err; echo "rc=$?" >> gpurun_out/hq_bench2.err
timeout 900 python bench.py > gpurun_out/hq_benchline.json 2> gpurun_out/hq_benchline.err; echo "rc=$?" >> gpurun_out/hq_benchline.err
