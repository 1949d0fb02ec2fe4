for r in 1 2; do
python tools/ab_update.py "" "CBAA_WAPPLY_GRID=148" | sed "s/\"default\"/\"zeroflush r$r\"/; s/\"CBAA_WAPPLY_GRID=148\"/\"persist148 r$r\"/"
CBAA_LIB=build/ab/lib_prev.so python tools/ab_update.py "" | sed "s/\"default\"/\"prev r$r\"/"
done > gpurun_out/ab_persist.jsonl 2>&1
python -c "
import json
for l in open('gpurun_out/ab_persist.jsonl'):
    try: d=json.loads(l)
    except Exception: print(l[:300]); continue
    print(d['variant'], round(d['update_ms_median'],4), {k:round(v,4) for k,v in d['phase_ms'].items()})
"
