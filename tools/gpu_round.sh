# One parameterised GPU call (run through gpurun from the repo root):
#   bash tools/gpu_round.sh TAG STAGE [STAGE ...]
# Stages (outputs under gpurun_out/, named *_TAG.*):
#   build     __graft_entry__.build()
#   test      pytest -m gpu (and the smoke)
#   bench     bench.py N=1 (C2, default); bench_c3 / bench_c4: the other workloads; ref: --impl reference
#   launches  ncu launch list (gpu__time_duration, clock-control none) of a short bench run
#   ncu       ncu --set full of one binned update + one detect → ncu_binned_TAG.json
#   sanitize  compute-sanitizer memcheck/racecheck/synccheck/initcheck of tools/sanitize.py (closed on the
#             GPU pool since run r02j: the tool refuses to run there)
#   sweep     tests/sweep_c5.py (C5 accuracy/throughput sweep)
#   c4full    tests/full_c4.py (config 4 at full size)
#   func2     functional N = 2 runs on ONE GPU (gloo process group, IPC exchange with device barriers):
#             C2 pipelined, C3, C4 — their times are meaningless (two ranks share the GPU)
set -x
T=$1; shift
for S in "$@"; do
  case $S in
    build) python __graft_entry__.py build > gpurun_out/build_$T.log 2>&1; tail -1 gpurun_out/build_$T.log ;;
    test)
      timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_$T.log 2>&1; tail -3 gpurun_out/pytest_gpu_$T.log
      python __graft_entry__.py smoke > gpurun_out/smoke_$T.log 2>&1; tail -1 gpurun_out/smoke_$T.log ;;
    bench) python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$T.json 2> gpurun_out/bench_$T.err; tail -c 1500 gpurun_out/bench_$T.json ;;
    bench_c3) python bench.py --workload C3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3_$T.json 2> gpurun_out/bench_c3_$T.err; tail -c 600 gpurun_out/bench_c3_$T.json ;;
    bench_c4) python bench.py --workload C4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4_$T.json 2> gpurun_out/bench_c4_$T.err; tail -c 600 gpurun_out/bench_c4_$T.json ;;
    ref) python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_$T.json 2> gpurun_out/bench_ref_$T.err; tail -c 600 gpurun_out/bench_ref_$T.json ;;
    launches) timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" --csv --log-file gpurun_out/launches_$T.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --detect-samples 3 > gpurun_out/ncu_launch_$T.log 2>&1 ;;
    ncu)
      timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_(bin_|zero_counts|hot|join3|union)" -s 10 -c 9 -o gpurun_out/prof_$T python tools/bin_c2_once.py > gpurun_out/ncu_full_$T.log 2>&1
      python tools/ncu_binned.py gpurun_out/prof_$T.ncu-rep "ncu --set full --clock-control none, the third C2 update + one detect (tools/bin_c2_once.py)" > gpurun_out/ncu_binned_$T.json 2> gpurun_out/ncu_binned_$T.err
      python tools/ncu_summary.py gpurun_out/prof_$T.ncu-rep > gpurun_out/ncu_counters_$T.json 2>/dev/null ;;
    sanitize)
      for tool in memcheck racecheck synccheck initcheck; do
        timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 python tools/sanitize.py > gpurun_out/sanitize_${tool}_$T.log 2>&1; echo "$tool rc=$?"
      done ;;
    sweep) timeout 2400 python -m tests.sweep_c5 > gpurun_out/sweep_c5_$T.jsonl 2> gpurun_out/sweep_c5_$T.err; tail -2 gpurun_out/sweep_c5_$T.err ;;
    c4full) timeout 2400 python -m tests.full_c4 > gpurun_out/full_c4_$T.jsonl 2> gpurun_out/full_c4_$T.err; tail -2 gpurun_out/full_c4_$T.jsonl ;;
    func2)
      for W in C2 C3 C4; do
        CBAA_BENCH_BACKEND=gloo timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --workload $W --steps 3 --warmup 3 --no-e2e --detect-samples 5 > gpurun_out/bench_n2func_${W}_$T.json 2> gpurun_out/bench_n2func_${W}_$T.err; echo "func2 $W rc=$?"; tail -c 400 gpurun_out/bench_n2func_${W}_$T.json
      done ;;
    *) echo "unknown stage $S" ;;
  esac
done
