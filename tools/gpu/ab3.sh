cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_distributed.py -x -q > gpurun_out/pytest_dist.log 2>&1; echo rc=$? >> gpurun_out/pytest_dist.log
for rep in 1 2; do for v in sort slot; do
  if [ $v = sort ]; then export SFK_KEY_GROUP=sort; else unset SFK_KEY_GROUP; fi
  echo -n "$v "; timeout 300 python tools/build_probe.py sf1 1.0 4
  echo -n "$v "; timeout 120 python tools/build_probe.py cu 1.0 2
done; done > gpurun_out/ab3.log 2>&1
unset SFK_KEY_GROUP
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_ab3.log 2>&1; echo rc=$? >> gpurun_out/pytest_ab3.log
