set -x
./tools/atoms_bench > gpurun_out/atoms_bench.jsonl 2>&1; cat gpurun_out/atoms_bench.jsonl
timeout 900 python tools/wc_ab.py > gpurun_out/wc_ab_b.jsonl 2> gpurun_out/wc_ab_b.err; cat gpurun_out/wc_ab_b.jsonl; tail -3 gpurun_out/wc_ab_b.err
