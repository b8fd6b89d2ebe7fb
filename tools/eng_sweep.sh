# engine tuning sweep (diagnostics): critical-path trace per knob value
for v in 0 2 8 32; do
  echo "nap=$v"; SFK_ENGINE_NAP=$v SFK_ENGINE_TRACE=1 timeout 300 python tools/trace_engine.py 1.0 2>&1 | sed -n 1,2p
done
SFK_ENGINE_NAP=8 SFK_ENGINE_TRACE=1 timeout 300 python tools/trace_engine.py 0.5 2>&1 | sed -n 1,2p
