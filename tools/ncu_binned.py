"""Per-launch DRAM bytes and issued L2 REDs of the binned-update kernels (k_bin_*) from an ncu --set full
report of ONE update call, plus their sum per update: the JSON bench.py reads for roofline.traffic and
roofline.update.dram / l2_red (profiles/r02_ncu_binned.json).
Usage: python tools/ncu_binned.py gpurun_out/prof_X.ncu-rep "how it was captured" > profiles/r02_ncu_binned.json"""
import json
import sys

sys.path.insert(0, "tools")
from ncu_summary import main as _summary  # noqa: E402

FIELDS = ("dram_read_bytes", "dram_write_bytes", "duration_us", "red_requests_to_l2", "red_sectors_to_l2",
          "atom_requests_to_l2", "smem_wavefronts", "smem_bank_conflicts", "warps_active_pct",
          "l1tex_throughput_pct", "registers", "l2_hit_pct", "lts_throughput_avg_pct", "dram_throughput_pct")


def main(path, how=""):
    import contextlib
    import io
    buf = io.StringIO()
    with contextlib.redirect_stdout(buf):
        _summary(path)
    launches = json.loads(buf.getvalue())["launches"]
    out = {"source": path, "captured": how}
    for e in launches:
        k = e["kernel"].replace("void ", "").split("<")[0].strip()
        if not k.startswith("k_bin"):
            continue
        d = out.setdefault(k, {"launches": 0, **{f: 0.0 for f in FIELDS}})
        d["launches"] += 1
        for f in FIELDS:
            d[f] += e.get(f, 0.0)
    upd = {"dram_bytes": 0.0, "l2_red_requests": 0.0, "l2_red_sectors": 0.0, "duration_us_cold": 0.0}
    for k, d in list(out.items()):
        if not k.startswith("k_bin"):
            continue
        n = d["launches"]
        for f in FIELDS:
            d[f] /= n
        d["dram_bytes_per_launch"] = d["dram_read_bytes"] + d["dram_write_bytes"]
        upd["dram_bytes"] += d["dram_bytes_per_launch"]
        upd["l2_red_requests"] += d["red_requests_to_l2"]
        upd["l2_red_sectors"] += d["red_sectors_to_l2"]
        upd["duration_us_cold"] += d["duration_us"]
    out["update"] = upd
    json.dump(out, sys.stdout, indent=1)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "")
