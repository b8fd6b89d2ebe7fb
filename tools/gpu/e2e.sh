mkdir -p gpurun_out
timeout 900 python bench.py --steps 10 --warmup 3 --no-cm > gpurun_out/e2e_bench.json 2> gpurun_out/e2e_bench.err
timeout 1200 python tools/host_query_bench.py 1000000000 3:24:0:4:p 3:24:0:4:p:8 3:24:0:4:p:10 3:24:4:4:p:8 3:24:0:4:p:16 3:25:0:3:p:12 > gpurun_out/e2e_hq.jsonl 2>&1
