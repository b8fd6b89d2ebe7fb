for b in 256 1024 4096 16384 65536; do
  echo "budget=$b"; SFK_ENGINE_BUDGET=$b SFK_ENGINE_TRACE=1 timeout 300 python tools/trace_engine.py 1.0 2>&1 | sed -n 1,3p
done
for bp in 2 4; do
  echo "blocks_per_sm=$bp"; SFK_ENGINE_BLOCKS_PER_SM=$bp SFK_ENGINE_TRACE=1 timeout 300 python tools/trace_engine.py 1.0 2>&1 | sed -n 1,3p
done
