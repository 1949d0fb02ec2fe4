for r in 1 2; do
python tools/ab_update.py "" "CBAA_BIN_SAMPLE=10" "CBAA_BIN_SAMPLE=11" | sed "s/\"default\"/\"L9 r$r\"/; s/\"CBAA_BIN_SAMPLE=10\"/\"L10 r$r\"/; s/\"CBAA_BIN_SAMPLE=11\"/\"L11 r$r\"/"
done > gpurun_out/ab_sample.jsonl 2>&1
python -c "
import json
for l in open('gpurun_out/ab_sample.jsonl'):
    try: d=json.loads(l)
    except Exception: print(l[:300]); continue
    print(d['variant'], round(d['update_ms_median'],4), {k:round(v,4) for k,v in d['phase_ms'].items()})
"
