"""Per-SASS-instruction view of one kernel in an ncu report: address, instruction, stall samples and
executed warp instructions, plus totals per region (split at the given SASS address offsets).
Usage: python tools/ncu_sass.py REPORT KERNEL_REGEX [top N]"""
import csv
import io
import subprocess
import sys


def rows(path, kernel):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass", "-k", kernel],
                         capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    hdr = r[1]
    res = []
    for x in r[2:]:
        d = dict(zip(hdr, x))
        try:
            res.append((int(d["Address"], 16), d["Source"].strip(), int(d["Warp Stall Sampling (All Samples)"] or 0),
                        int(d["Instructions Executed"] or 0)))
        except (KeyError, ValueError):
            pass
    seen, uniq = set(), []
    for x in res:   # the CSV can list an instruction more than once
        if x[0] not in seen:
            seen.add(x[0])
            uniq.append(x)
    return uniq


if __name__ == "__main__":
    rs = rows(sys.argv[1], sys.argv[2])
    base = rs[0][0]
    tot_s = sum(r[2] for r in rs)
    tot_i = sum(r[3] for r in rs)
    print(f"instructions {len(rs)}, samples {tot_s}, warp instructions executed {tot_i}")
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 0
    if top:
        for a, s, n, i in sorted(rs, key=lambda r: -r[2])[:top]:
            print(f"{a - base:06x} {n:8d} {100.0 * n / tot_s:5.1f}% {i:10d}  {s}")
    else:
        for a, s, n, i in rs:
            print(f"{a - base:06x} {n:8d} {i:10d}  {s}")
