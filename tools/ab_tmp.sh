for r in 1 2; do
CBAA_LIB=build/ab/lib_prev.so python tools/ab_update.py "" | sed "s/\"default\"/\"prev r$r\"/"
python tools/ab_update.py "" | sed "s/\"default\"/\"batch r$r\"/"
done > gpurun_out/ab_batch.jsonl 2>&1
python -c "
import json
for l in open('gpurun_out/ab_batch.jsonl'):
    try: d=json.loads(l)
    except Exception: print(l[:300]); continue
    print(d['variant'], round(d['update_ms_median'],4), {k:round(v,4) for k,v in d['phase_ms'].items()})
"
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "binned or c2 or sampled or prefix" -p no:cacheprovider 2>&1 | tail -2
