set -x
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_(update|zero|zero_counts|hot|tuples|join3|union|or_merge)" --csv --log-file gpurun_out/launches_r01g.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch_g.log 2>&1
CBAA_FORCE_CARTESIAN=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_(zero_counts|hot|tuples|join3|union)" --csv --log-file gpurun_out/launches_r01g_cart.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch_g2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_(zero_counts|hot|join3|union)" -s 4 -c 4 -o gpurun_out/prof_r01g python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full_g.log 2>&1
CBAA_FORCE_CARTESIAN=1 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_r01g_cart.json 2>&1
python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_r01g_join.json 2>&1
grep -o '"detect_ms": [0-9.]*\|"post_update_ms": [0-9.]*' gpurun_out/bench_r01g_*.json
