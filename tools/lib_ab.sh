#!/bin/bash
# A/B of library builds on one box: tools/lib_ab.sh variant-dir... (each a dir
# under paper_1701_04148_b200/_lib holding libsfsketch_cuda.so; "main" = the
# default build). cfg-3 SFF build at alpha 1.0 / 0.5 / 1.5, interleaved twice.
cd "$(dirname "$0")/.."
for rep in 1 2; do
  for v in "$@"; do
    for a in 1.0 0.5 1.5; do
      if [ "$v" = main ]; then lib=paper_1701_04148_b200/_lib/libsfsketch_cuda.so; else lib=paper_1701_04148_b200/_lib/$v/libsfsketch_cuda.so; fi
      echo -n "$v "; SFK_LIB_PATH=$lib timeout 120 python tools/build_probe.py sff $a
    done
  done
done
