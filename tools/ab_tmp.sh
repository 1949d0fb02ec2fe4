for r in 1 2; do
python tools/ab_update.py "" | sed "s/\"default\"/\"base r$r\"/"
for v in T512 T384 T1024P16; do CBAA_LIB=build/ab/lib_$v.so python tools/ab_update.py "" | sed "s/\"default\"/\"$v r$r\"/"; done
done > gpurun_out/ab_wtile.jsonl 2>&1
python -c "
import json
for l in open('gpurun_out/ab_wtile.jsonl'):
    try: d=json.loads(l)
    except Exception: print(l[:300]); continue
    print(d['variant'], round(d['update_ms_median'],4), {k:round(v,4) for k,v in d['phase_ms'].items()})
"
