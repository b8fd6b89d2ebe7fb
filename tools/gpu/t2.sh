mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_configs_full.py tests/test_gpu_distributed.py -x -q --durations=12 > gpurun_out/t2_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/t2_pytest.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/t2_bench.json 2> gpurun_out/t2_bench.err; echo "rc=$?" >> gpurun_out/t2_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/t2_ref.json 2> gpurun_out/t2_ref.err; echo "rc=$?" >> gpurun_out/t2_ref.err
