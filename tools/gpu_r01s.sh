# C5 sweep and config 4 at full size with the sampled-region binned update (the default).
set -x
timeout 2400 python -m tests.sweep_c5 > gpurun_out/sweep_c5_s.jsonl 2> gpurun_out/sweep_c5_s.err; tail -2 gpurun_out/sweep_c5_s.err
timeout 2400 python -m tests.full_c4 > gpurun_out/full_c4_s.jsonl 2> gpurun_out/full_c4_s.err; tail -3 gpurun_out/full_c4_s.jsonl
timeout 900 python tools/workload_perf.py > gpurun_out/workload_perf_s.jsonl 2> gpurun_out/workload_perf_s.err; cat gpurun_out/workload_perf_s.jsonl
