set -x
python __graft_entry__.py build > gpurun_out/build_bin1.log 2>&1; tail -1 gpurun_out/build_bin1.log
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "binned and not c2_full" > gpurun_out/pytest_bin1.log 2>&1; tail -15 gpurun_out/pytest_bin1.log
timeout 600 python tools/binned_perf.py > gpurun_out/binned_perf1.jsonl 2> gpurun_out/binned_perf1.err; cat gpurun_out/binned_perf1.jsonl; tail -3 gpurun_out/binned_perf1.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_(bin|update)" --csv --log-file gpurun_out/launches_bin1.csv python tools/binned_perf.py > /dev/null 2>&1
