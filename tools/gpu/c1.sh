mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -x -q -k "sff or sf3 or sf4 or cfg3 or long_runs or sum_trigger or fixture" > gpurun_out/c1_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/c1_pytest.log
for a in 1.0 0.5 1.5; do
  for v in sff sf4 sf3; do
    timeout 120 python tools/build_probe.py $v $a >> gpurun_out/c1_probe.log 2>&1
    SFK_NO_CHAIN=1 timeout 120 python tools/build_probe.py $v $a | sed 's/^/nochain /' >> gpurun_out/c1_probe.log 2>&1
  done
done
