#!/bin/bash
# A/B of the polling and dataflow engines on one box (timing + parity subset).
cd "$(dirname "$0")/.."
for a in 1.0 0.5; do
  timeout 120 python tools/build_probe.py sff $a
  SFK_ENGINE=flow timeout 120 python tools/build_probe.py sff $a
done
SFK_ENGINE=flow timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "fixture or cfg3 or cfg1 or cfg2 or chunked or prefix or long_runs or sf1_dropped" 2>&1 | tail -3
