set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "binned" > gpurun_out/pytest_ab3.log 2>&1; tail -3 gpurun_out/pytest_ab3.log
timeout 900 python tools/wc_ab.py > gpurun_out/wc_ab_c.jsonl 2> gpurun_out/wc_ab_c.err; cat gpurun_out/wc_ab_c.jsonl; tail -3 gpurun_out/wc_ab_c.err
