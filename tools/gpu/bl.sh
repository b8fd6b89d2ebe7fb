mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/hq_benchline.json 2> gpurun_out/hq_benchline.err; echo "rc=$?" >> gpurun_out/hq_benchline.err
