mkdir -p gpurun_out
timeout 300 ./tools/hop_latency > gpurun_out/hop_latency.json 2>&1
