cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_sf1_keys.py -x -q > gpurun_out/pytest_ab14_keys.log 2>&1; echo rc=$? >> gpurun_out/pytest_ab14_keys.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_ab14.log 2>&1; echo rc=$? >> gpurun_out/pytest_ab14.log
for rep in 1 2; do for v in base main; do
  if [ $v = main ]; then lib=paper_1701_04148_b200/_lib/libsfsketch_cuda.so; else lib=paper_1701_04148_b200/_lib/$v/libsfsketch_cuda.so; fi
  echo -n "$v "; SFK_LIB_PATH=$lib timeout 300 python tools/build_probe.py sf1 1.0 4
  echo -n "$v "; SFK_LIB_PATH=$lib timeout 120 python tools/build_probe.py cu 1.0 2
  echo -n "$v "; SFK_LIB_PATH=$lib timeout 120 python tools/build_probe.py sf1 1.0 1
done; done > gpurun_out/ab14.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file /tmp/l4.csv python tools/build_probe.py sf1 1.0 4 > /dev/null 2>&1
python tools/launch_sum.py /tmp/l4.csv > gpurun_out/launches_cfg4_j3.txt
