mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_configs_full.py -x -q -k "sf1 or sf2 or cfg1 or cfg4 or fixture or prefix or saturation" > gpurun_out/c3_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/c3_pytest.log
timeout 300 python tools/build_probe.py sf1 1.0 4 > gpurun_out/c3_probe.log 2>&1
timeout 300 python tools/build_probe.py sf2 1.0 >> gpurun_out/c3_probe.log 2>&1
timeout 300 python tools/build_probe.py sf1 1.0 1 >> gpurun_out/c3_probe.log 2>&1
