# final round-1 evidence with the measured pass table: full round + C5 sweep
set -x
bash tools/gpu_round.sh r01f
timeout 1500 python -m tests.sweep_c5 > gpurun_out/sweep_c5_f.jsonl 2> gpurun_out/sweep_c5_f.err; tail -3 gpurun_out/sweep_c5_f.err
