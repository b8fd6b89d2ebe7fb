mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_configs_full.py -x -q -k "sff or cfg3 or fuzz or fixture" > gpurun_out/ch_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/ch_pytest.log
rm -f gpurun_out/ch_probe.log
for rep in 1 2; do
for cfg in "0 4" "128 4" "32 4" "128 1" "512 8" "128 16"; do
  set -- $cfg
  for a in 1.0 0.5 1.5; do
    SFK_CHAIN_MIN_A=$1 SFK_CHAIN_LEN=$2 timeout 300 python tools/build_probe.py sff $a | sed "s/^/minA=$1 len=$2 /" >> gpurun_out/ch_probe.log 2>&1
  done
done
done
