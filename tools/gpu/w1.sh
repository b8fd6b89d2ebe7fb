mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_api.py -x -q -k "warp or tiny or bad_op" > gpurun_out/w1_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/w1_pytest.log
timeout 600 python tools/small_batch_curve.py > gpurun_out/w1_curve.jsonl 2> gpurun_out/w1_curve.err
