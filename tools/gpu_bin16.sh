set -x
python __graft_entry__.py build > gpurun_out/build_bin16.log 2>&1; tail -1 gpurun_out/build_bin16.log
timeout 600 python tools/binned_perf.py > gpurun_out/binned_perf16.jsonl 2> gpurun_out/binned_perf16.err; head -2 gpurun_out/binned_perf16.jsonl; tail -3 gpurun_out/binned_perf16.err
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,launch__occupancy_limit_shared_mem,launch__occupancy_limit_registers,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"k_bin" --csv --log-file gpurun_out/launches_bin16.csv python tools/bin_c2_once.py > /dev/null 2>&1
