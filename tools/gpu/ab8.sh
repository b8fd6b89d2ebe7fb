cd $GRAFT_REPO_ROOT
for rep in 1 2; do for v in def 32 64; do
  if [ $v = def ]; then unset SFK_L2_FETCH; else export SFK_L2_FETCH=$v; fi
  echo -n "$v "; timeout 300 python tools/build_probe.py sf1 1.0 4 2>>gpurun_out/ab8.err
  echo -n "$v "; timeout 120 python tools/build_probe.py cu 1.0 2 2>>gpurun_out/ab8.err
  echo -n "$v "; timeout 120 python tools/build_probe.py sff 1.0 3 2>>gpurun_out/ab8.err
done; done > gpurun_out/ab8.log 2>&1
unset SFK_L2_FETCH
