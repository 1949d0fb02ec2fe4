set -x
python __graft_entry__.py build > gpurun_out/build_bin14.log 2>&1; tail -1 gpurun_out/build_bin14.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_bin_(scatter)" -c 1 -o gpurun_out/prof_bin14 python tools/bin_c2_once.py > gpurun_out/ncu_bin14.log 2>&1; tail -3 gpurun_out/ncu_bin14.log
