# round-1: parity, bench, launch list and full ncu capture of the current kernels
set -x
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu_c.log 2>&1; tail -5 gpurun_out/pytest_gpu_c.log
python __graft_entry__.py smoke > gpurun_out/smoke_c.log 2>&1; tail -2 gpurun_out/smoke_c.log
python bench.py --steps 50 --warmup 5 > gpurun_out/bench_r01c.json 2> gpurun_out/bench_r01c.err; tail -c 3000 gpurun_out/bench_r01c.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_(update|zero|zero_hot|tuples|or_merge)" --csv --log-file gpurun_out/launches_r01c.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch_c.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_(update|zero_hot|tuples)" -s 6 -c 4 -o gpurun_out/prof_r01c python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full_c.log 2>&1
tail -3 gpurun_out/ncu_full_c.log
