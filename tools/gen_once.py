"""Three binned updates of the C2 window on a C5 geometry (r g cbn as arguments), for ncu captures of the
generic wide kernels: -k regex:k_bin_ -s 10 -c 5 = the third update's sample, starts, scatter, apply, log."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import oracle as O  # noqa: E402
from paper_1901_06207_b200 import workload as W  # noqa: E402
from paper_1901_06207_b200.cbaa import Cbaa, config_from_dict  # noqa: E402

r, g, cbn = (int(x) for x in sys.argv[1:4])
geo = next(x for x in W.c5_geometries() if x["r"] == r and x["g"] == g and x["cbn"][0] == cbn)
w = W.generate(W.C2, 1, with_raw=False)
s = torch.from_numpy(w.src.view(np.int32)).cuda()
d = torch.from_numpy(w.dst.view(np.int32)).cuda()
cb = Cbaa(config_from_dict(dict(O.default_params(), **geo)), 0)
print(cb.update_plan(len(w.src)))
for _ in range(3):
    cb.reset()
    cb.update(s, d)
torch.cuda.synchronize()
