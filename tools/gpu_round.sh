# Round evidence in one call: build, GPU tests, smoke, bench (N=1), ncu launch list, ncu --set full of the
# update and detect kernels, compute-sanitizer (4 tools).  Outputs under gpurun_out/ (tag = $1).
set -x
T=${1:-rXX}
python __graft_entry__.py build > gpurun_out/build_$T.log 2>&1; tail -1 gpurun_out/build_$T.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_$T.log 2>&1; tail -3 gpurun_out/pytest_gpu_$T.log
python __graft_entry__.py smoke > gpurun_out/smoke_$T.log 2>&1; tail -1 gpurun_out/smoke_$T.log
python bench.py --steps 50 --warmup 5 > gpurun_out/bench_$T.json 2> gpurun_out/bench_$T.err; tail -c 600 gpurun_out/bench_$T.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_(bin_|update|zero|zero_counts|hot|tuples|join3|union|or_merge)" --csv --log-file gpurun_out/launches_$T.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch_$T.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_(bin_count|bin_sample|bin_scatter|bin_wc|bin_apply|zero_counts|hot|join3|union)" -s 14 -c 8 -o gpurun_out/prof_$T python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full_$T.log 2>&1
python tools/ncu_binned.py gpurun_out/prof_$T.ncu-rep > gpurun_out/ncu_binned_$T.json 2>/dev/null
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 python tools/sanitize.py > gpurun_out/sanitize_${tool}_$T.log 2>&1; echo "$tool rc=$?"
done
