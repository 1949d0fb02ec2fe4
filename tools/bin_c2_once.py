"""One binned C2 update (for ncu captures)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import oracle as O  # noqa: E402
from paper_1901_06207_b200 import workload as W  # noqa: E402
from paper_1901_06207_b200.cbaa import Cbaa, config_from_dict  # noqa: E402

w = W.generate(W.C2, 1, with_raw=False)
s = torch.from_numpy(w.src.view(np.int32)).cuda()
d = torch.from_numpy(w.dst.view(np.int32)).cuda()
cb = Cbaa(config_from_dict(dict(O.default_params(), update_mode=int(sys.argv[1]) if len(sys.argv) > 1 else 2)), 0)
for _ in range(2):
    cb.reset()
    cb.update(s, d)
torch.cuda.synchronize()
if len(sys.argv) > 2:   # occupancy report of the binned kernels
    import ctypes
    print("max active scatter CTAs/SM reported via ncu launch__occupancy_limit_shared_mem")
