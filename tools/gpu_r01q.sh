# Round evidence on HEAD after the container restore: full round script + reference arm.
set -x
bash tools/gpu_round.sh r01q
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_r01q.json 2> gpurun_out/bench_ref_r01q.err; tail -c 400 gpurun_out/bench_ref_r01q.json
