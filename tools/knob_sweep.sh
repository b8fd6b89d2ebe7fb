#!/bin/bash
# Engine knob A/B on one box: cfg-3 SFF build at alpha 1.0 per knob value.
cd "$(dirname "$0")/.."
python tools/build_probe.py sff 1.0
for b in 64 256 4096; do SFK_ENGINE_BUDGET=$b python tools/build_probe.py sff 1.0; done
for k in 2 3; do SFK_ENGINE_BLOCKS_PER_SM=$k python tools/build_probe.py sff 1.0; done
python tools/build_probe.py sff 1.0
