set -x
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu_e.log 2>&1; tail -5 gpurun_out/pytest_gpu_e.log
python __graft_entry__.py smoke > gpurun_out/smoke_e.log 2>&1; tail -2 gpurun_out/smoke_e.log
python bench.py --steps 50 --warmup 5 > gpurun_out/bench_r01e.json 2>&1; tail -c 3000 gpurun_out/bench_r01e.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_(update|zero|zero_hot|tuples|or_merge)" --csv --log-file gpurun_out/launches_r01e.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch_e.log 2>&1
