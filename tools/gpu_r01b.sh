# round-1 iteration: parity of both update modes, then the bench of each mode
set -x
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu_b.log 2>&1; tail -5 gpurun_out/pytest_gpu_b.log
python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/bench_r01b_ts.json 2>&1; tail -c 1500 gpurun_out/bench_r01b_ts.json
for p in 1 3; do python bench.py --steps 20 --warmup 5 --passes $p --no-cpu-baseline --no-e2e > gpurun_out/bench_r01b_ts_p$p.json 2>&1; done
python bench.py --steps 20 --warmup 5 --update-mode red --no-cpu-baseline --no-e2e > gpurun_out/bench_r01b_red.json 2>&1
grep -ho '"update_ms": [0-9.]*' gpurun_out/bench_r01b_*.json
