cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q -k "sf1 or SF1 or flat or cfg1 or cfg4 or cu or CU or config or fuzz" > gpurun_out/pytest_ab7.log 2>&1; echo rc=$? >> gpurun_out/pytest_ab7.log
for rep in 1 2; do for v in base main; do
  if [ $v = main ]; then lib=paper_1701_04148_b200/_lib/libsfsketch_cuda.so; else lib=paper_1701_04148_b200/_lib/$v/libsfsketch_cuda.so; fi
  echo -n "$v "; SFK_LIB_PATH=$lib timeout 300 python tools/build_probe.py sf1 1.0 4
  echo -n "$v "; SFK_LIB_PATH=$lib timeout 120 python tools/build_probe.py cu 1.0 2
done; done > gpurun_out/ab7.log 2>&1
mkdir -p /tmp/ncu
for k in sf1_ignore_k key_meta_k runs_mark_k segscan_apply_k; do
timeout 900 ncu --kernel-name regex:$k --launch-count 1 --set full --import-source on --clock-control none -o /tmp/ncu/$k -f python tools/build_probe.py sf1 1.0 4 > gpurun_out/ncu_cfg4_$k.log 2>&1
python tools/ncu_summary.py /tmp/ncu/$k.ncu-rep > gpurun_out/ncu_cfg4_${k}_summary.txt 2>&1
done
