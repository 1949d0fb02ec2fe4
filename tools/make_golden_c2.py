"""Writes tests/golden/c2_seed1_theta1024_hosts.txt: the oracle's super-host list of bench.py's default
window (BASELINE config 2, seed 1, paper geometry, θ = 1024).  Calls only oracle/ and the seeded input
generator; bench.py compares its last timed window with this file.

  python tools/make_golden_c2.py          # ~30 s: generation + oracle update of 100M pairs + detect
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import oracle as O                       # noqa: E402
from paper_1901_06207_b200 import workload as W      # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "c2_seed1_theta1024_hosts.txt")


def main():
    t0 = time.time()
    p = O.default_params()
    w = W.generate(W.C2, 1, with_raw=False)
    cube, _ = O.update(p, w.src, w.dst)
    st, hosts, stats = O.detect(p, cube, 1024)
    assert st == 0
    with open(OUT, "w") as f:
        f.write("# Oracle super-host list of BASELINE config 2 (workload.C2, seed 1, 100M pairs), paper geometry\n")
        f.write("# (P:437, Q3/Q4/Q8 seeds), theta = 1024, Alg. 2/3 output (P:263-316) in the S:418 order.\n")
        f.write("# Written by tools/make_golden_c2.py (oracle/ only).  Columns: ip cs lp z estimate (repr; inf = Z 0).\n")
        f.write(f"# hosts {len(hosts)}\n")
        for h in hosts:
            f.write(f"0x{int(h['ip']):08X} {int(h['cs'])} {int(h['lp'])} {int(h['z'])} {float(h['estimate'])!r}\n")
    print(f"{len(hosts)} hosts -> {OUT} ({time.time() - t0:.1f} s)")


if __name__ == "__main__":
    main()
