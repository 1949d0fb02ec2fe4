"""Three binned C2 updates then one detect, for ncu captures (tools/gpu_round.sh ncu: -k k_bin_*|detect
kernels -s 10 -c 9 = the third update's 5 kernels + the detect's 4)."""
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
for _ in range(3):
    cb.reset()
    cb.update(s, d)
hosts, _, _ = cb.detect(1024)
torch.cuda.synchronize()
print(len(hosts), "hosts")
