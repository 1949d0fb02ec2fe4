# Round evidence with sampled bin regions: full round script + reference arm.
set -x
bash tools/gpu_round.sh r01r
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_r01r.json 2> gpurun_out/bench_ref_r01r.err; tail -c 300 gpurun_out/bench_ref_r01r.json
