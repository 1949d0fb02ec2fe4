set -x
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu_d.log 2>&1; tail -5 gpurun_out/pytest_gpu_d.log
python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench_r01d.json 2>&1; tail -c 2500 gpurun_out/bench_r01d.json
