mkdir -p gpurun_out
(nproc; lscpu | head -30; free -g; numactl -H 2>/dev/null | head; nvidia-smi topo -m 2>/dev/null | head -5) > gpurun_out/io_host.txt 2>&1
timeout 600 tools/host_io_probe 1000000000 > gpurun_out/io_probe.jsonl 2> gpurun_out/io_probe.err; echo "rc=$?" >> gpurun_out/io_probe.err
