# C2 binned update with each A/B build of libcbaa.so (tools/ab/*.so) and the in-tree one
for so in paper_1901_06207_b200/libcbaa.so tools/ab/*.so; do
  CBAA_LIB=$PWD/$so python - <<'PY'
import os, sys, json
import numpy as np, torch
sys.path.insert(0, ".")
from oracle import oracle as O
from paper_1901_06207_b200 import workload as W
from paper_1901_06207_b200.cbaa import Cbaa, config_from_dict
w = W.generate(W.C2, 1, with_raw=False)
s = torch.from_numpy(w.src.view(np.int32)).cuda(); d = torch.from_numpy(w.dst.view(np.int32)).cuda()
cb = Cbaa(config_from_dict(dict(O.default_params(), update_mode=2)), 0)
ts = []
cb.set_phase_timing(True)
for i in range(12):
    cb.reset(); a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); cb.update(s, d); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    if i == 1: cb.update_phase_ms()
ph, calls = cb.update_phase_ms()
print(json.dumps({"lib": os.environ["CBAA_LIB"].split("/")[-1], "ms_median": round(float(np.median(ts[2:])), 4),
                  "phases_ms": [round(x / calls, 4) for x in ph]}), flush=True)
PY
done
