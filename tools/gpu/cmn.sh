mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none -k regex:"cm_atomic_k|stats_" -c 6 -f -o /tmp/cmn python tools/cm_probe.py > gpurun_out/cmn.log 2>&1
ncu -i /tmp/cmn.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,lts__t_sectors.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,smsp__pcsamp_warps_issue_stalled_long_scoreboard,smsp__pcsamp_warps_issue_stalled_lg_throttle,smsp__inst_executed.sum > gpurun_out/cmn_raw.csv 2>&1
