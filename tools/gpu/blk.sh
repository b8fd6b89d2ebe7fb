mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_api.py -x -q -k "block or engine or tiny" > gpurun_out/blk_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/blk_pytest.log
timeout 900 python tools/small_batch_curve.py > gpurun_out/blk_curve.jsonl 2> gpurun_out/blk_curve.err; echo "rc=$?" >> gpurun_out/blk_curve.err
