"""DRAM bytes per launch of the binned-update kernels (k_bin_*) from an ncu --set full report, as the
JSON bench.py reads for roofline.traffic (profiles/r01_ncu_binned.json).
Usage: python tools/ncu_binned.py gpurun_out/prof_X.ncu-rep > profiles/r01_ncu_binned.json"""
import json
import subprocess
import sys

sys.path.insert(0, "tools")
from ncu_summary import main as _summary  # noqa: E402


def main(path):
    import contextlib
    import io
    buf = io.StringIO()
    with contextlib.redirect_stdout(buf):
        _summary(path)
    launches = json.loads(buf.getvalue())["launches"]
    out = {"source": path}
    for e in launches:
        k = e["kernel"].replace("void ", "").split("<")[0].strip()
        if not k.startswith("k_bin"):
            continue
        d = out.setdefault(k, {"launches": 0, "dram_read": 0.0, "dram_write": 0.0, "duration_us": 0.0})
        d["launches"] += 1
        d["dram_read"] += e.get("dram_read_bytes", 0.0)
        d["dram_write"] += e.get("dram_write_bytes", 0.0)
        d["duration_us"] += e.get("duration_us", 0.0)
    for k, d in out.items():
        if k == "source":
            continue
        n = d["launches"]
        d["dram_bytes_per_launch"] = (d["dram_read"] + d["dram_write"]) / n
        d["dram_read_per_launch"] = d.pop("dram_read") / n
        d["dram_write_per_launch"] = d.pop("dram_write") / n
        d["duration_us_per_launch_cold"] = d.pop("duration_us") / n
    json.dump(out, sys.stdout, indent=1)


if __name__ == "__main__":
    main(sys.argv[1])
