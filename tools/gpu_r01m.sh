set -x
for N in 2 4; do
CBAA_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2957$N bench.py --gpus $N --steps 5 --warmup 3 --no-e2e > gpurun_out/bench_n${N}_func.json 2> gpurun_out/bench_n${N}_func.err; echo rc=$?
grep -o '"n_gpus": [0-9]*\|"n_super_hosts": [0-9]*\|"exchange": "[a-z]*"\|"global_pairs": [0-9]*' gpurun_out/bench_n${N}_func.json | tr '\n' ' '; echo
done
