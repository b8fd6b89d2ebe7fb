mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_configs_full.py tests/test_gpu_baselines.py tests/test_gpu_api.py -x -q -k "sf1 or cu or cfg1 or cfg2 or cfg4 or fixture or prefix or dropped" > gpurun_out/c7_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/c7_pytest.log
for args in "sf1 1.0 4" "sf1 1.0 1" "cu 1.0"; do
  timeout 300 python tools/build_probe.py $args >> gpurun_out/c7_probe.log 2>&1
done
