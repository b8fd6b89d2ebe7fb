cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_ab2.log 2>&1; echo rc=$? >> gpurun_out/pytest_ab2.log
for rep in 1 2; do for v in tile op; do
  if [ $v = tile ]; then export SFK_SF1_DROP=tile; else unset SFK_SF1_DROP; fi
  echo -n "$v "; timeout 300 python tools/build_probe.py sf1 1.0 4
  echo -n "$v "; timeout 120 python tools/build_probe.py cu 1.0 2
  echo -n "$v "; timeout 120 python tools/build_probe.py sf1 1.0 1
done; done > gpurun_out/ab2.log 2>&1
unset SFK_SF1_DROP
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg4.csv python tools/build_probe.py sf1 1.0 4 > gpurun_out/ncu_cfg4.log 2>&1
