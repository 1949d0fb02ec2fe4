for r in 1 2; do
CBAA_BIN_WIDE=0 python tools/ab_update.py "" | sed "s/\"default\"/\"narrow-branch1 r$r\"/"
CBAA_BIN_WIDE=0 CBAA_LIB=build/ab/lib_prev.so python tools/ab_update.py "" | sed "s/\"default\"/\"narrow-prev r$r\"/"
done > gpurun_out/ab_narrow_branch1.jsonl 2>&1
python -c "
import json
for l in open('gpurun_out/ab_narrow_branch1.jsonl'):
    try: d=json.loads(l)
    except Exception: print(l[:300]); continue
    print(d['variant'], round(d['update_ms_median'],4), {k:round(v,4) for k,v in d['phase_ms'].items()})
"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -q -x -p no:cacheprovider 2>&1 | tail -2
