mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_query_paths.py -q -x -k "CW or 4-" > gpurun_out/san_memcheck_query.log 2>&1; echo "rc=$?" >> gpurun_out/san_memcheck_query.log
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_api.py -q -x -k "warp or bad_op" > gpurun_out/san_memcheck_warp.log 2>&1; echo "rc=$?" >> gpurun_out/san_memcheck_warp.log
timeout 1500 compute-sanitizer --tool synccheck --print-limit 20 python -m pytest tests/test_gpu_query_paths.py -q -x -k "CW and 65536" > gpurun_out/san_synccheck_query.log 2>&1; echo "rc=$?" >> gpurun_out/san_synccheck_query.log
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -x -k "sf1 and fixture" > gpurun_out/san_memcheck_bmin.log 2>&1; echo "rc=$?" >> gpurun_out/san_memcheck_bmin.log
