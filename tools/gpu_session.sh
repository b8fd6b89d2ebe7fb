#!/bin/bash
# One GPU session: parity tests, bench line, launch list, ncu --set full of the
# dominant kernels. Usage (from the repo root, under gpurun):
#   bash tools/gpu_session.sh [tag] [what...]   what in {tests,bench,launches,ncu_engine,ncu_query,ncu_scan}
tag=${1:-r01}; shift
what=${@:-tests bench launches ncu_engine ncu_query}
out=gpurun_out/$tag; mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $out/gpu.txt 2>&1
for w in $what; do
  case $w in
  tests) timeout 1800 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.log 2>&1; echo "tests rc=$?" ;;
  smoke) timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke rc=$?" ;;
  bench) timeout 900 python bench.py --steps 10 --warmup 3 > $out/bench.json 2> $out/bench.err; echo "bench rc=$?"; tail -c 3000 $out/bench.json ;;
  launches) timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
      --log-file $out/launches_bench.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-cm \
      > $out/ncu_launch.log 2>&1; echo "launches rc=$?"; python tools/launches.py $out/launches_bench.csv > $out/launches_bench_summary.txt 2>&1 ;;
  ncu_engine) timeout 900 ncu --set full --clock-control none --import-source on -k regex:poll_engine -c 1 \
      -o $out/ncu_engine -f python tools/one_build.py sff 1.0 1 > $out/ncu_engine.log 2>&1; echo "ncu_engine rc=$?" ;;
  ncu_scan) timeout 900 ncu --set full --clock-control none --import-source on -k regex:segscan_apply -c 1 \
      -o $out/ncu_scan -f python tools/one_build.py sff 1.0 1 > $out/ncu_scan.log 2>&1; echo "ncu_scan rc=$?" ;;
  ncu_query) timeout 900 ncu --set full --clock-control none --import-source on -k regex:min_query -c 1 \
      -o $out/ncu_query -f python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-cm \
      > $out/ncu_query.log 2>&1; echo "ncu_query rc=$?" ;;
  esac
done
