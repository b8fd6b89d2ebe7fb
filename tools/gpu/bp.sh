mkdir -p gpurun_out
timeout 600 python tools/blk_probe.py > gpurun_out/blk_probe.jsonl 2> gpurun_out/blk_probe.err; echo "rc=$?" >> gpurun_out/blk_probe.err
