set -x
python __graft_entry__.py build > gpurun_out/build_bin15.log 2>&1; tail -1 gpurun_out/build_bin15.log
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "binned and not c2_full" > gpurun_out/pytest_bin15.log 2>&1; tail -3 gpurun_out/pytest_bin15.log
timeout 600 python tools/binned_perf.py > gpurun_out/binned_perf11.jsonl 2> gpurun_out/binned_perf11.err; cat gpurun_out/binned_perf11.jsonl; tail -3 gpurun_out/binned_perf11.err
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:"k_bin" --csv --log-file gpurun_out/launches_bin15.csv python tools/bin_c2_once.py > /dev/null 2>&1
