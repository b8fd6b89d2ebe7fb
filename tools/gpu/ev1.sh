# evidence session: launch list of the bench, ncu --set full of the dominant kernels, batch curve
mkdir -p gpurun_out/ev1
O=gpurun_out/ev1
timeout 600 python tools/batch_curve.py > $O/batch_curve.jsonl 2> $O/batch_curve.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/launches_bench.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $O/launches_bench.log 2>&1
python tools/launch_sum.py $O/launches_bench.csv > $O/launches_bench_summary.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg4.csv python tools/one_build.py sf1rec 1.0 1 > $O/launches_cfg4.log 2>&1
python tools/launch_sum.py $O/launches_cfg4.csv > $O/launches_cfg4_summary.txt
run_full() {  # name, kernel regex, count, command...
  name=$1; k=$2; cnt=$3; shift 3
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:"$k" -c $cnt -f -o /tmp/$name "$@" > $O/ncu_$name.log 2>&1
  python tools/ncu_summary.py /tmp/$name.ncu-rep > $O/ncu_${name}_summary.txt 2>&1
}
run_full query_cw min_query_cw 1 python tools/query_bench.py 1000000000 1.0 4
ncu -i /tmp/query_cw.ncu-rep --page source --csv --print-source sass > $O/ncu_query_cw_source.csv 2>/dev/null
run_full cm_atomic cm_atomic_k 1 python tools/one_build.py cm 1.0 1
run_full sff_segscan segscan_apply_k 1 python tools/one_build.py sff 1.0 1
run_full sff_sort DeviceRadixSortOnesweep 2 python tools/one_build.py sff 1.0 1
run_full cu_engine poll_engine_k 1 python tools/one_build.py cu 1.0 1
run_full sff_engine poll_engine_k 1 python tools/one_build.py sff 1.0 1
