set -x
timeout 600 python tools/wc_ab.py C2 "C2 bursty" 2>&1 | grep tile > gpurun_out/ab5.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "binned" > gpurun_out/pytest_ab5.log 2>&1; tail -1 gpurun_out/pytest_ab5.log
