set -x
python __graft_entry__.py build > gpurun_out/build_bin10.log 2>&1; tail -1 gpurun_out/build_bin10.log
python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --update-mode binned > gpurun_out/bench_bin10.json 2> gpurun_out/bench_bin10.err; python -c "import json;d=json.load(open('gpurun_out/bench_bin10.json'));print({k:d[k] for k in ('value','ms_per_step','ms_per_step_serial','update_ms','detect_ms','post_update_ms')})"
python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --update-mode binned --no-pipeline > gpurun_out/bench_bin10s.json 2>> gpurun_out/bench_bin10.err; python -c "import json;d=json.load(open('gpurun_out/bench_bin10s.json'));print({k:d[k] for k in ('value','ms_per_step','ms_per_step_serial','update_ms','detect_ms','post_update_ms')})"
python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_bin10t.json 2>> gpurun_out/bench_bin10.err; python -c "import json;d=json.load(open('gpurun_out/bench_bin10t.json'));print({k:d[k] for k in ('value','ms_per_step','ms_per_step_serial','update_ms','detect_ms','post_update_ms')})"
tail -3 gpurun_out/bench_bin10.err
