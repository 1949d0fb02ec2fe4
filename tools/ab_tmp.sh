for r in 1 2; do
python tools/ab_update.py "" | sed "s/\"default\"/\"dedup r$r\"/"
CBAA_LIB=build/ab/lib_nodedup.so python tools/ab_update.py "" | sed "s/\"default\"/\"nodedup r$r\"/"
done > gpurun_out/ab_dedup.jsonl 2>&1
python -c "
import json
for l in open('gpurun_out/ab_dedup.jsonl'):
    try: d=json.loads(l)
    except Exception: print(l[:300]); continue
    print(d['variant'], round(d['update_ms_median'],4), {k:round(v,4) for k,v in d['phase_ms'].items()})
"
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "c2 or binned or sampled" 2>&1 | tail -2
