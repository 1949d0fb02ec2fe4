set -x
python __graft_entry__.py build > gpurun_out/build_bin5.log 2>&1; tail -1 gpurun_out/build_bin5.log
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "binned and not c2_full" > gpurun_out/pytest_bin5.log 2>&1; tail -3 gpurun_out/pytest_bin5.log
CBAA_BIN_STAGED=1 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "binned and not c2_full" > gpurun_out/pytest_bin5s.log 2>&1; tail -3 gpurun_out/pytest_bin5s.log
timeout 600 python tools/binned_perf.py > gpurun_out/binned_perf5.jsonl 2> gpurun_out/binned_perf5.err; cat gpurun_out/binned_perf5.jsonl; tail -3 gpurun_out/binned_perf5.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none -k regex:"k_bin" --csv --log-file gpurun_out/launches_bin5.csv python tools/bin_c2_once.py > /dev/null 2>&1
