# Round evidence with 8-pair-unit sampling: round script, reference arm, config 4 full size, workload shapes.
set -x
bash tools/gpu_round.sh r01t
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_r01t.json 2> gpurun_out/bench_ref_r01t.err; tail -c 300 gpurun_out/bench_ref_r01t.json
timeout 2400 python -m tests.full_c4 > gpurun_out/full_c4_t.jsonl 2> gpurun_out/full_c4_t.err; tail -2 gpurun_out/full_c4_t.jsonl
timeout 900 python tools/workload_perf.py > gpurun_out/workload_perf_t.jsonl 2> gpurun_out/workload_perf_t.err; cat gpurun_out/workload_perf_t.jsonl
