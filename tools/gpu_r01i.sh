set -x
# functional N=2 run of the bench's multi-router path on a 1-GPU box (both ranks share GPU 0; the
# timing is meaningless, the point is the ipc exchange + owned-range detect + gather + max-over-ranks)
CBAA_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29561 bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/bench_n2_func.json 2> gpurun_out/bench_n2_func.err; echo rc=$?
tail -c 1500 gpurun_out/bench_n2_func.json; tail -5 gpurun_out/bench_n2_func.err
