for r in 1 2; do
python tools/ab_update.py "" | sed "s/\"default\"/\"red64 r$r\"/"
for v in prev; do CBAA_LIB=build/ab/lib_$v.so python tools/ab_update.py "" | sed "s/\"default\"/\"$v r$r\"/"; done
done > gpurun_out/ab_red64.jsonl 2>&1
python -c "
import json
for l in open('gpurun_out/ab_red64.jsonl'):
    try: d=json.loads(l)
    except Exception: print(l[:300]); continue
    print(d['variant'], round(d['update_ms_median'],4), {k:round(v,4) for k,v in d['phase_ms'].items()})
"
