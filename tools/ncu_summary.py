"""Key counters of an ncu --set full report, per launch, as JSON (profiles/<round>_ncu_counters.json).
Usage: python tools/ncu_summary.py gpurun_out/prof_r01k.ncu-rep > profiles/r01_ncu_counters.json"""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "duration_us": ("gpu__time_duration.sum", 1.0),
    "dram_read_bytes": ("dram__bytes_read.sum", None),
    "dram_write_bytes": ("dram__bytes_write.sum", None),
    "dram_throughput_pct": ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1.0),
    "lts_throughput_avg_pct": ("lts__throughput.avg.pct_of_peak_sustained_elapsed", 1.0),
    "lts_throughput_max_pct": ("lts__throughput.max.pct_of_peak_sustained_elapsed", 1.0),
    "l1tex_throughput_pct": ("l1tex__throughput.avg.pct_of_peak_sustained_active", 1.0),
    "l2_hit_pct": ("lts__t_sector_hit_rate.pct", 1.0),
    "l1_hit_pct": ("l1tex__t_sector_hit_rate.pct", 1.0),
    "red_sectors_to_l2": ("lts__t_sectors_srcunit_tex_op_red.sum", 1.0),
    "red_requests_to_l2": ("lts__t_requests_srcunit_tex_op_red.sum", 1.0),
    "atom_requests_to_l2": ("lts__t_requests_srcunit_tex_op_atom.sum", 1.0),
    "smem_wavefronts": ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", 1.0),
    "smem_bank_conflicts": ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", 1.0),
    "global_load_sectors": ("l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", 1.0),
    "warps_active_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", 1.0),
    "sm_throughput_pct": ("sm__throughput.avg.pct_of_peak_sustained_elapsed", 1.0),
    "ipc_per_sm": ("sm__inst_executed.avg.per_cycle_active", 1.0),
    "warp_instructions": ("smsp__inst_executed.sum", 1.0),
    "registers": ("launch__registers_per_thread", 1.0),
    "grid": ("launch__grid_size", 1.0),
    "block": ("launch__block_size", 1.0),
}
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1, "msecond": 1e3, "nsecond": 1e-3}


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        e = {"kernel": d["Kernel Name"].split("(")[0]}
        for k, (m, _) in KEYS.items():
            if m not in d or d[m] in ("", "n/a"):
                continue
            v = float(d[m].replace(",", ""))
            u = units[hdr.index(m)]
            if k.endswith("_bytes"):
                v *= UNIT.get(u, 1)
            if k == "duration_us":
                v *= UNIT.get(u, 1)
            e[k] = v
        # stall reasons: warps stalled per issued instruction, by reason (largest first)
        st = {}
        for m, v in d.items():
            if m.startswith("smsp__average_warps_issue_stalled_") and m.endswith("_per_issue_active.ratio") and v not in ("", "n/a"):
                st[m[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = float(v.replace(",", ""))
        if st:
            e["stalls_per_issue"] = dict(sorted(((k, round(x, 3)) for k, x in st.items() if x >= 0.01), key=lambda kv: -kv[1]))
        res.append(e)
    json.dump({"source": path, "launches": res}, sys.stdout, indent=1)


if __name__ == "__main__":
    main(sys.argv[1])
