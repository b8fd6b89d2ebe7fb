mkdir -p gpurun_out
timeout 1500 python -m pytest tests/ -q -m gpu -x > gpurun_out/w4_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/w4_pytest.log
timeout 300 python tools/api_overhead.py > gpurun_out/w4_overhead.jsonl 2>&1
timeout 600 python tools/small_batch_curve.py 1,8,64,128,192,256,1024,4096,16384 > gpurun_out/w4_curve.jsonl 2> gpurun_out/w4_curve.err
