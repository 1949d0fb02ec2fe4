# Final round evidence: round script (tests, smoke, bench, ncu, sanitizers) + reference arm.
set -x
bash tools/gpu_round.sh r01u
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_r01u.json 2> gpurun_out/bench_ref_r01u.err; tail -c 300 gpurun_out/bench_ref_r01u.json
