mkdir -p gpurun_out
timeout 300 python tools/api_micro.py > gpurun_out/api_micro.json 2>&1
timeout 1800 python -m pytest tests/test_gpu_api.py tests/test_gpu_baselines.py tests/test_gpu_parity.py -x -q > gpurun_out/api_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/api_pytest.log
timeout 900 python tools/small_batch_curve.py 1,8,64,256,1024,2048 > gpurun_out/api_curve.jsonl 2>&1
