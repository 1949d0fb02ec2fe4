# Final round evidence (code as committed): round script, reference arm, C5 sweep, config 4 full size, workload shapes.
set -x
bash tools/gpu_round.sh r01w
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_r01w.json 2> gpurun_out/bench_ref_r01w.err; tail -c 300 gpurun_out/bench_ref_r01w.json
timeout 2400 python -m tests.sweep_c5 > gpurun_out/sweep_c5_w.jsonl 2> gpurun_out/sweep_c5_w.err; tail -2 gpurun_out/sweep_c5_w.err
timeout 2400 python -m tests.full_c4 > gpurun_out/full_c4_w.jsonl 2> gpurun_out/full_c4_w.err; tail -2 gpurun_out/full_c4_w.jsonl
timeout 900 python tools/workload_perf.py > gpurun_out/workload_perf_w.jsonl 2> gpurun_out/workload_perf_w.err; cat gpurun_out/workload_perf_w.jsonl
