# Final round evidence: round script (tests, smoke, bench, ncu, sanitizers) + reference arm.
set -x
bash tools/gpu_round.sh r01v
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_r01v.json 2> gpurun_out/bench_ref_r01v.err; tail -c 300 gpurun_out/bench_ref_r01v.json
