set -x
for so in paper_1901_06207_b200/libcbaa.so tools/ab/t512.so tools/ab/t384.so; do
  echo "== $so"
  CBAA_LIB=$PWD/$so timeout 600 python tools/wc_ab.py C2 2>&1 | grep tile
done > gpurun_out/ab4.txt
CBAA_LIB=$PWD/tools/ab/t512.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "binned" > gpurun_out/pytest_ab4.log 2>&1; tail -1 gpurun_out/pytest_ab4.log
