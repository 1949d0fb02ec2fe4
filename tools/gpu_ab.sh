set -x
for i in 1 2; do
python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ab_pipe_$i.json 2>&1
python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e --no-pipeline > gpurun_out/ab_serial_$i.json 2>&1
done
grep -ho '"ms_per_step": [0-9.]*\|"ms_per_step_serial": [0-9.]*\|"detect_ms": [0-9.]*\|"update_ms": [0-9.]*' gpurun_out/ab_*.json
