set -x
python bench.py --steps 50 --warmup 5 > gpurun_out/bench_r01a.json 2> gpurun_out/bench_r01a.err
tail -3 gpurun_out/bench_r01a.err
cat gpurun_out/bench_r01a.json
python bench.py --steps 20 --warmup 5 --passes 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_r01a_p1.json 2>&1
python bench.py --steps 20 --warmup 5 --passes 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_r01a_p3.json 2>&1
tail -c 600 gpurun_out/bench_r01a_p1.json; tail -c 600 gpurun_out/bench_r01a_p3.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_(update|zero|zero_hot|tuples|or_merge)" --csv --log-file gpurun_out/launches_r01a.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_update|k_zero_hot|k_tuples" -s 6 -c 4 -o gpurun_out/prof_r01a python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out
