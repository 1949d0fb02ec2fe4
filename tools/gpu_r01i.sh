set -x
python __graft_entry__.py build > gpurun_out/build_r01i.log 2>&1; tail -1 gpurun_out/build_r01i.log
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_r01i.log 2>&1; tail -3 gpurun_out/pytest_r01i.log
timeout 600 python tools/binned_perf.py > gpurun_out/binned_perf_i.jsonl 2> gpurun_out/binned_perf_i.err; head -2 gpurun_out/binned_perf_i.jsonl
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:"k_bin" --csv --log-file gpurun_out/launches_r01i.csv python tools/bin_c2_once.py > /dev/null 2>&1
python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_r01i.json 2> gpurun_out/bench_r01i.err; python -c "import json;d=json.load(open('gpurun_out/bench_r01i.json'));print({k:d[k] for k in ('value','ms_per_step','ms_per_step_serial','update_ms','detect_ms')})"
timeout 1500 python -m tests.sweep_c5 > gpurun_out/sweep_c5_i.jsonl 2> gpurun_out/sweep_c5_i.err; tail -2 gpurun_out/sweep_c5_i.err
timeout 1500 python -m tests.full_c4 > gpurun_out/full_c4_i.jsonl 2> gpurun_out/full_c4_i.err; tail -2 gpurun_out/full_c4_i.jsonl
