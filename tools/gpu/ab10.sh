cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_ab10.log 2>&1; echo rc=$? >> gpurun_out/pytest_ab10.log
for rep in 1 2 3; do for v in base main; do
  if [ $v = main ]; then lib=paper_1701_04148_b200/_lib/libsfsketch_cuda.so; else lib=paper_1701_04148_b200/_lib/$v/libsfsketch_cuda.so; fi
  echo -n "$v "; SFK_LIB_PATH=$lib timeout 120 python tools/build_probe.py cu 1.0 2
done; done > gpurun_out/ab10.log 2>&1
