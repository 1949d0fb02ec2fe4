# round evidence with the binned update: full round, C5 sweep, workload shapes, full-size C4
set -x
bash tools/gpu_round.sh r01h
timeout 1500 python -m tests.sweep_c5 > gpurun_out/sweep_c5_h.jsonl 2> gpurun_out/sweep_c5_h.err; tail -2 gpurun_out/sweep_c5_h.err
timeout 900 python tools/workload_perf.py > gpurun_out/workload_perf_h.jsonl 2> gpurun_out/workload_perf_h.err; tail -2 gpurun_out/workload_perf_h.err
timeout 1500 python -m tests.full_c4 > gpurun_out/full_c4_h.jsonl 2> gpurun_out/full_c4_h.err; tail -2 gpurun_out/full_c4_h.err
