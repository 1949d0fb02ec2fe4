set -x
python __graft_entry__.py build > gpurun_out/build_f.log 2>&1; tail -1 gpurun_out/build_f.log
timeout 600 python -m pytest tests/test_gpu_c_api.py -m gpu -q -p no:cacheprovider 2>&1 | tail -3
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_torchrun1.json 2> gpurun_out/bench_torchrun1.err; tail -c 400 gpurun_out/bench_torchrun1.json; tail -3 gpurun_out/bench_torchrun1.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2>&1; tail -c 600 gpurun_out/bench_ref.json
