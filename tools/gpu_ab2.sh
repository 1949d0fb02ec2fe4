for i in 1 2 3; do python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ab2_$i.json 2>&1; done
grep -ho '"ms_per_step": [0-9.]*\|"ms_per_step_serial": [0-9.]*\|"update_ms": [0-9.]*' gpurun_out/ab2_*.json
CBAA_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29582 bench.py --gpus 2 --steps 5 --warmup 3 --no-e2e > gpurun_out/bench_n2_func.json 2> gpurun_out/bench_n2_func.err; echo rc=$?
grep -o '"n_super_hosts": [0-9]*' gpurun_out/bench_n2_func.json
