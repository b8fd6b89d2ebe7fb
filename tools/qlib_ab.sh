#!/bin/bash
# A/B of library builds on the cfg-5 query (1B keys, cluster path): tools/qlib_ab.sh variant-dir...
cd "$(dirname "$0")/.."
for rep in 1 2; do
  for v in "$@"; do
    if [ "$v" = main ]; then lib=paper_1701_04148_b200/_lib/libsfsketch_cuda.so; else lib=paper_1701_04148_b200/_lib/$v/libsfsketch_cuda.so; fi
    echo -n "$v "; SFK_LIB_PATH=$lib timeout 300 python tools/query_bench.py 1000000000 0.0,1.0 3 2>&1 | tail -2 | tr '\n' ' '; echo
  done
done
