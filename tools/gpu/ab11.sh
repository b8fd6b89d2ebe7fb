cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_sf1_keys.py -x -q > gpurun_out/pytest_ab11_keys.log 2>&1; echo rc=$? >> gpurun_out/pytest_ab11_keys.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_ab11.log 2>&1; echo rc=$? >> gpurun_out/pytest_ab11.log
for rep in 1 2; do for v in sort excl; do
  if [ $v = sort ]; then export SFK_SF1_FAT=sort; else unset SFK_SF1_FAT; fi
  echo -n "$v "; timeout 300 python tools/build_probe.py sf1 1.0 4
done; done > gpurun_out/ab11.log 2>&1
unset SFK_SF1_FAT
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file /tmp/l4.csv python tools/build_probe.py sf1 1.0 4 > /dev/null 2>&1
python tools/launch_sum.py /tmp/l4.csv > gpurun_out/launches_cfg4_excl.txt
