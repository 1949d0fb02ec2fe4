#!/usr/bin/env python
"""CBAA window benchmark (BASELINE.json metric: packet pairs/s per window update + window-end detect ms).

One step = one window of the hot path: reset (a7) → update of the window's pairs (a0-a6) →
[OR-merge over NVLink, a8, N > 1] → detect (a9-a14, host list filled).  Workload: BASELINE config 2
(100M core-network-shaped pairs per GPU, Zipf hosts, ~0.1% super hosts, paper geometry, θ = 1024),
synthetic and seeded.  Inputs (800 MB per GPU) exceed the 126 MB L2, so no extra flush.

  python bench.py [--gpus N --steps K --warmup W]           # our CUDA path, one JSON line on rank 0
  python bench.py --impl reference [...]                    # the CPU oracle as it stands (reference arm)
Multi-GPU: torchrun --nproc-per-node N bench.py --gpus N ...; each rank is one edge router with its own
100M-pair shard of one global window (weak scaling); max-over-ranks device time.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "packet pairs/sec per window update (1/2/4/8 B200) + window-end detect ms"
THETA = 1024


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=["C2", "C1"], default="C2")
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--passes", type=int, default=0, help="update passes (0 = library auto)")
    ap.add_argument("--update-mode", choices=["test_set", "red", "binned"], default="binned",
                    help="binned (default): count/scatter/apply through shared memory; test_set / red: the "
                         "direct random-access kernel (DESIGN.md §6)")
    ap.add_argument("--no-pipeline", action="store_true",
                    help="N=1: run windows strictly one after another (default: window k's detect overlaps "
                         "window k+1's reset+update on a second cube and a high-priority stream)")
    ap.add_argument("--exchange", choices=["nccl", "p2p", "ipc"], default="ipc",
                    help="N>1 window-end exchange: NCCL all_to_all + OR kernel, or the NVLink pull-OR over "
                         "symmetric memory (p2p) / CUDA IPC mappings (ipc)")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def workload(name, seed, rank, world):
    from paper_1901_06207_b200 import workload as W
    spec = W.C2 if name == "C2" else W.C1
    # one global flow set (shared seed); each router sees its own packets of those flows
    pseed = seed if world == 1 else seed * 1000 + rank + 1
    return spec, W.generate(spec, seed, packet_seed=pseed, with_raw=False)


def config_block(name, spec, world):
    return {"workload": f"{name}: {spec.n // 1_000_000}M pairs/GPU, {spec.n_hosts} inner hosts, "
                        f"{spec.n_flows / 1e6:.1f}M Zipf(s={spec.zipf_s}) flows, shuffled",
            "pairs_per_gpu": spec.n, "global_pairs": spec.n * world,
            "geometry": "r=4 |RA|=3 |VA|=1 g=4096 c=4096 (128 MiB cube, P:437)", "theta": THETA,
            "parallelism": f"routers{world}" if world > 1 else "single",
            "l2": "inputs 800 MB/GPU > 126 MB L2 (no extra flush); cube reset each window"}


# --------------------------------------------------------------------------------------- clocks
class ClockSampler:
    """NVML sampling of SM clock and throttle reasons during the timed region."""

    def __init__(self, index):
        self.samples, self.reasons, self.stop_ev = [], set(), threading.Event()
        self.max_mhz = None
        try:
            import pynvml as N
            N.nvmlInit()
            self.N, self.h = N, N.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = N.nvmlDeviceGetMaxClockInfo(self.h, N.NVML_CLOCK_SM)
        except Exception as e:   # no NVML: report it instead of guessing
            self.N, self.err = None, str(e)

    def _run(self):
        N = self.N
        names = {getattr(N, k): k for k in dir(N) if k.startswith("nvmlClocksEventReason") or
                 k.startswith("nvmlClocksThrottleReason")}
        while not self.stop_ev.is_set():
            try:
                self.samples.append(N.nvmlDeviceGetClockInfo(self.h, N.NVML_CLOCK_SM))
                mask = N.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in names.items():
                    if isinstance(bit, int) and bit and (mask & bit) == bit and "None" not in name and "All" not in name:
                        self.reasons.add(name.replace("nvmlClocksEventReason", "").replace("nvmlClocksThrottleReason", ""))
            except Exception:
                pass
            time.sleep(0.01)

    def __enter__(self):
        if self.N:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.N:
            self.stop_ev.set()
            self.t.join()

    def summary(self):
        if not self.N:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "error": self.err}
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def access_peaks():
    """Measured random single-word access rates over an L2-resident 64 MiB buffer (tools/redbench --quick):
    {"red": RED.OR/s, "ldg": 32-bit loads/s}.  The update touches one random word per bit it sets."""
    exe = os.path.join(ROOT, "tools", "redbench")
    peaks = {}
    try:
        out = subprocess.run([exe, "--quick"], capture_output=True, text=True, timeout=120).stdout
        for line in out.splitlines():
            d = json.loads(line)
            if d.get("mode") in ("red", "ldg", "ldg_ca"):
                peaks[d["mode"]] = d["Gops"] * 1e9
    except Exception:
        pass
    return peaks


def measured_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


def ncu_traffic():
    try:
        return json.load(open(os.path.join(ROOT, "profiles", "ncu_update_traffic.json")))
    except Exception:
        return None


def ncu_binned():
    """DRAM bytes per launch of the binned-update kernels from the committed ncu --set full capture."""
    try:
        return json.load(open(os.path.join(ROOT, "profiles", "r01_ncu_binned.json")))
    except Exception:
        return {}


def ncu_update_counters():
    """Per-launch L1/L2 utilisation of k_update from the committed ncu --set full capture."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "r01_ncu_counters.json")))
        ls = [e for e in d["launches"] if "k_update" in e["kernel"]]
        keys = ("lts_throughput_avg_pct", "lts_throughput_max_pct", "l1tex_throughput_pct", "l1_hit_pct", "l2_hit_pct")
        return {k: [round(e[k], 1) for e in ls] for k in keys} | {"source": "profiles/r01_ncu_counters.json"}
    except Exception:
        return None


# --------------------------------------------------------------------------------------- reference arm
def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from oracle import oracle as O
    spec, w = workload(args.workload, args.seed, 0, 1)
    p = O.default_params()
    m = 1_000_000 if spec.n >= 1_000_000 else spec.n
    times = []
    for k in range(args.warmup + args.steps):
        off = (k * m) % max(1, spec.n - m + 1)
        t0 = time.perf_counter()
        cube, _ = O.update(p, w.src[off:off + m], w.dst[off:off + m])
        O.detect(p, cube, THETA)
        t1 = time.perf_counter()
        if k >= args.warmup:
            times.append(t1 - t0)
    tot = sum(times)
    value = m * len(times) / tot
    sample = f"{m} consecutive pairs of the {args.workload} window per step (update + detect, θ={THETA})"
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "pairs/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / len(times),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": config_block(args.workload, spec, 1),
            "cpu_baseline": {"value": value, "unit": "pairs/s", "cores": 1, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": "pairs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def cpu_baseline(w, seconds_budget=20.0):
    """The oracle as it stands, single-threaded, on a bounded sample of the same window."""
    from oracle import oracle as O
    p = O.default_params()
    m = min(w.src.size, 60_000_000)   # ~10-15 s of single-thread oracle work on the box's CPU
    t0 = time.perf_counter()
    cube, _ = O.update(p, w.src[:m], w.dst[:m])
    O.detect(p, cube, THETA)
    t1 = time.perf_counter()
    return {"value": m / (t1 - t0), "unit": "pairs/s", "cores": 1, "kind": "oracle",
            "sample": f"first {m} pairs of the window: oracle update + detect (θ={THETA}), {t1 - t0:.1f} s"}


# --------------------------------------------------------------------------------------- our arm
def _allreduce(v: float, op) -> float:
    """Scalar all-reduce (max over ranks for times) on the process group's own device kind."""
    import torch
    import torch.distributed as dist
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([v], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=op)
    return float(t.item())


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_1901_06207_b200 import distributed as D
    from paper_1901_06207_b200.cbaa import Cbaa, default_config

    rank, world, local = dist_env()
    # one GPU per rank; more ranks than GPUs (functional runs on a 1-GPU box) wrap around and then
    # need CBAA_BENCH_BACKEND=gloo, since NCCL refuses two ranks on one device
    local = local % max(1, torch.cuda.device_count())
    if world > 1:
        backend = os.environ.get("CBAA_BENCH_BACKEND", "nccl")
        dist.init_process_group(backend, device_id=torch.device("cuda", local) if backend == "nccl" else None)
    torch.cuda.set_device(local)
    peaks_acc = access_peaks() if rank == 0 and args.update_mode != "binned" else {}
    spec, w = workload(args.workload, args.seed, rank, world)
    n = spec.n
    src = torch.from_numpy(w.src.view(np.int32)).cuda()
    dst = torch.from_numpy(w.dst.view(np.int32)).cuda()
    cfg = default_config()
    cfg.update_passes = args.passes
    cfg.update_mode = {"test_set": 0, "red": 1, "binned": 2}[args.update_mode]
    from paper_1901_06207_b200.cbaa import cube_bytes
    peer = None
    exchange = args.exchange if world > 1 else "none"
    if exchange == "p2p":
        try:
            peer = D.PeerExchange(cube_bytes(cfg), torch.device("cuda", local))
        except Exception as e:   # no symmetric memory on this box: say so and use NCCL
            print(f"[bench] p2p exchange unavailable ({e}); using nccl", file=sys.stderr)
            exchange = "nccl"
    cb = Cbaa(cfg, local, cube=peer.buf if peer else None)
    if exchange == "ipc":
        # collective fallback: every rank must be able to map every peer cube, else all use NCCL
        err = None
        try:
            peer = D.IpcExchange(cb, rank, world)
        except Exception as e:
            err, peer = e, None
        if not int(_allreduce(0.0 if err else 1.0, dist.ReduceOp.MIN)):
            if peer:
                peer.close()
            peer, exchange = None, "nccl"
            print(f"[bench] ipc exchange unavailable ({err}); using nccl", file=sys.stderr)
    n_cs = cb.n_cs
    cs_bytes = cb.nbytes // n_cs
    stream = torch.cuda.Stream()
    cube_view = cb.cube()

    def merge_slices(peers, lo, hi):
        cb.merge_slice(peers, lo, hi, stream=stream)

    def window(ev=None):
        cb.reset(stream)
        if ev:
            ev[0].record(stream)
        cb.update(src, dst, stream)
        if ev:
            ev[1].record(stream)
        lo, hi = 0, n_cs
        if world > 1:
            with torch.cuda.stream(stream):
                if peer:
                    lo, hi = peer.exchange(cb, rank, world, n_cs, cs_bytes, stream)
                else:
                    lo, hi = D.exchange_owned(cube_view, rank, world, n_cs, cs_bytes, merge_slices)
        hosts, _, rc = cb.detect(THETA, cs_lo=lo, cs_hi=hi, stream=stream, with_stats=False)
        if exchange == "p2p":
            with torch.cuda.stream(stream):
                peer.window_done()
        elif exchange == "ipc":
            peer.window_done(stream)
        if ev:
            ev[2].record(stream)
        return D.gather_hosts(hosts, rank, world)

    with torch.cuda.stream(stream):
        for _ in range(max(args.warmup, 3)):   # at least 3 untimed warm-up windows
            window()
    torch.cuda.synchronize()
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = cb.kernel_launches
    cb.set_phase_timing(True)       # event pair around every update kernel, on its stream
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        t_start.record(stream)
        for k in range(args.steps):
            hosts = window(evs[k])
        t_end.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches = cb.kernel_launches - launches0
    phase_ms, phase_calls = cb.update_phase_ms()
    cb.set_phase_timing(False)
    elapsed_ms = t_start.elapsed_time(t_end)
    upd_ms = [e[0].elapsed_time(e[1]) for e in evs]
    post_ms = [e[1].elapsed_time(e[2]) for e in evs]
    if world > 1:
        elapsed_ms = _allreduce(elapsed_ms, dist.ReduceOp.MAX)
    serial_ms = elapsed_ms

    # Pipelined windows (N = 1): two cubes; window k's reset+update run on the update stream while
    # window k-1's detect runs on a high-priority stream (its 128-thread CTAs fit beside the persistent
    # update CTAs).  Cube k%2 is reset only after the detect of window k-2 has returned (host order).
    # Pipelined windows: two cubes; window k's reset+update run on the update stream while window k-1's
    # [exchange +] detect runs on a high-priority stream (its kernels fit beside the persistent update
    # CTAs).  Cube k%2 is reset only after the detect of window k-2 has returned on every rank (host
    # order; at N > 1 the ipc exchange's window_done barrier).  N > 1 pipelines with the ipc exchange.
    pipelined = not args.no_pipeline and (world == 1 or exchange == "ipc")
    if pipelined:
        cfg.detect_overlap = 1             # window-end kernels without shared memory: they co-run
        cbs = [Cbaa(cfg, local), Cbaa(cfg, local)]
        cb2 = cbs[1]
        peers = [D.IpcExchange(c, rank, world) for c in cbs] if world > 1 else [None, None]
        lo_pri, hi_pri = torch.cuda.Stream.priority_range()
        s_upd, s_det = stream, torch.cuda.Stream(priority=hi_pri)

        # the window reset moves to the detect stream: cube k%2 is cleared right after its detect (and,
        # at N > 1, after every peer has finished reading it), overlapping the other cube's update
        clean = [torch.cuda.Event(), torch.cuda.Event()]
        for i, c in enumerate(cbs):
            c.reset(s_det)
            clean[i].record(s_det)

        def finish(c, pe, px, i):
            s_det.wait_event(pe)
            lo, hi = 0, n_cs
            if px:
                lo, hi = px.exchange(c, rank, world, n_cs, cs_bytes, s_det)
            out, _, _ = c.detect(THETA, cs_lo=lo, cs_hi=hi, stream=s_det, with_stats=False)
            if px:
                px.window_done(s_det)
            c.reset(s_det)
            clean[i].record(s_det)
            return D.gather_hosts(out, rank, world)

        def run_pipelined(n_win, upd_evs=None):
            pending, out = None, None
            for k in range(n_win):
                c = cbs[k % 2]
                s_upd.wait_event(clean[k % 2])
                if upd_evs:
                    upd_evs[k][0].record(s_upd)
                c.update(src, dst, s_upd)
                done = torch.cuda.Event()
                done.record(s_upd)
                if upd_evs:
                    upd_evs[k][1].record(s_upd)
                if pending:
                    out = finish(*pending)
                pending = (c, done, peers[k % 2], k % 2)
            return finish(*pending)

        run_pipelined(max(args.warmup, 3))
        torch.cuda.synchronize()
        launches0 = cbs[0].kernel_launches + cb2.kernel_launches
        for c in cbs:
            c.set_phase_timing(True)
        pevs = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(args.steps)]
        p_start, p_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        with ClockSampler(local) as clk:
            p_start.record(s_upd)
            hosts = run_pipelined(args.steps, pevs)
            p_end.record(s_det)
            torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        launches = cbs[0].kernel_launches + cb2.kernel_launches - launches0
        phase_ms, phase_calls = [0.0] * 4, 0
        for c in cbs:
            ms_c, calls_c = c.update_phase_ms()
            phase_ms = [a + b for a, b in zip(phase_ms, ms_c)]
            phase_calls += calls_c
            c.set_phase_timing(False)
        elapsed_ms = p_start.elapsed_time(p_end)
        if world > 1:
            elapsed_ms = _allreduce(elapsed_ms, dist.ReduceOp.MAX)
        upd_ms = [e[0].elapsed_time(e[1]) for e in pevs]
        for px in peers:
            if px:
                px.close()

    # window-end detect latency alone: update finished, then detect until the host list is filled
    det_ms = []
    with torch.cuda.stream(stream):
        for _ in range(10):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            h, _, _ = cb.detect(THETA, stream=stream, with_stats=False)
            det_ms.append(1e3 * (time.perf_counter() - t0))

    e2e = None
    if not args.no_e2e:
        ps = torch.from_numpy(w.src.view(np.int32)).pin_memory()
        pd = torch.from_numpy(w.dst.view(np.int32)).pin_memory()
        ke = min(args.steps, 5)
        with torch.cuda.stream(stream):
            cb.reset(stream)
            cb.update_host(ps, pd, stream)
            cb.detect(THETA, stream=stream)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            nh = 0
            a.record(stream)
            for _ in range(ke):
                cb.reset(stream)
                cb.update_host(ps, pd, stream)     # pinned host → device inside the timed region
                hh, st, _ = cb.detect(THETA, stream=stream)   # device → host of the result
                nh = len(hh)
            b.record(stream)
            torch.cuda.synchronize()
        e2e_ms = a.elapsed_time(b) / ke
        if world > 1:
            e2e_ms = _allreduce(e2e_ms, dist.ReduceOp.MAX)
        e2e = {"value": n * world / (e2e_ms / 1e3), "unit": "pairs/s", "ms_per_step": e2e_ms,
               "h2d_bytes_per_step": 8 * n, "d2h_bytes_per_step": 24 * nh + 104 * n_cs + 8,
               "path": "cbaa_update_host (pinned, double-buffered chunks) + cbaa_detect"}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    ms_step = elapsed_ms / args.steps
    value = n * world * args.steps / (elapsed_ms / 1e3)
    upd = statistics.median(upd_ms)
    passes = cb.update_passes
    peaks = measured_peaks()
    hbm = peaks.get("hbm_gbs", 6650.0)
    per_call = [t / max(1, phase_calls) for t in phase_ms]
    binned = args.update_mode == "binned"
    if binned:
        # binned update (binned.cuh): algorithmic DRAM bytes of each kernel per launch
        nb = ncu_binned()
        # scatter kernel: tile sort k_bin_scatter unless CBAA_BIN_SCATTER=wc (the library's rule)
        scat = "k_bin_wc" if os.environ.get("CBAA_BIN_SCATTER") == "wc" else "k_bin_scatter"
        # region sizing: a 1/16 sample (k_bin_sample) for chunks of ≥ 2^24 pairs with the tile scatter,
        # else the exact count (k_bin_count) — the library's rule (cbaa.cu update_binned)
        samp = (scat == "k_bin_scatter" and os.environ.get("CBAA_BIN_SAMPLE", "9") != "0"
                and n >= int(os.environ.get("CBAA_BIN_SAMPLE_MIN", str(1 << 24))))
        lg = int(os.environ.get("CBAA_BIN_SAMPLE", "9"))
        cnt = ("k_bin_sample", 8 * 8 * (n >> lg)) if samp else ("k_bin_count", 8 * n)
        algo = {cnt[0]: cnt[1], "k_bin_starts": 3 * 4 * 4096, scat: 12 * n,
                "k_bin_apply": 4 * n + cb.nbytes}
        kernels = {}
        for name, t in zip(algo, per_call):
            kernels[name] = {"ms": t, "share": t / max(1e-9, sum(per_call)), "algorithmic_bytes": algo[name],
                             "gbs": algo[name] / (t / 1e3) / 1e9 if t > 0 else None,
                             "frac_hbm": algo[name] / (t / 1e3) / 1e9 / hbm if t > 0 else None,
                             "ncu_dram_bytes": (nb.get(name) or {}).get("dram_bytes_per_launch")}
        dom = max(kernels, key=lambda k: kernels[k]["ms"])
        kd = kernels[dom]
        roofline = {"kernel": dom, "bound": "hbm", "achieved": kd["gbs"], "peak": hbm, "unit": "GB/s",
                    "frac": kd["frac_hbm"], "traffic": kd["ncu_dram_bytes"],
                    "algorithmic": {cnt[0]: "8 B/pair read" + (f" for 8 of every {1 << lg} pairs" if samp else ""),
                                    scat: "8 B/pair read + 4 B/pair entry written",
                                    "k_bin_apply": "4 B/pair entry read + the cube's words OR-ed once (+ overflow "
                                                   "log, normally empty)"},
                    "per_launch_ms": kd["ms"], "timing": "CUDA event pair around every update kernel on its launch "
                    "stream over the timed region (cbaa_set_phase_timing), averaged per update call",
                    "peak_source": "MEASURED_PEAKS.json hbm_gbs", "kernels": kernels,
                    "update_ms": upd, "update_mode": args.update_mode,
                    "traffic_source": "profiles/r01_ncu_binned.json (ncu --set full, dram__bytes_read+write)",
                    "limiter": "the dominant binned kernel is not DRAM-bound (ncu DRAM traffic = its algorithmic "
                                "bytes): k_bin_scatter is issue/latency-bound (ATOMS rank, per-tile bin scan, "
                                "4 barriers per 8192-pair tile, 16 warps/SM at 119 registers), k_bin_apply is "
                                "shared-memory-bound (4 random LDS tests per entry); see DESIGN.md section 6"}
        roofline_hbm = None
    else:
        algo = 4 * n                       # |RA|+|VA| = 4 bit-sets per pair, one random word each
        achieved = algo / (upd / 1e3)
        peak_acc = max(peaks_acc.values()) if peaks_acc else None
        traffic = ncu_traffic()
        roofline = {"kernel": "k_update (cbaa_update, all passes)", "bound": "lsu_random_word",
                    "achieved": achieved / 1e9, "peak": (peak_acc or float("nan")) / 1e9, "unit": "G word-updates/s",
                    "frac": achieved / peak_acc if peak_acc else None,
                    "traffic": (traffic or {}).get("dram_bytes_per_update"),
                    "algorithmic": f"4 random 32-bit word updates per pair (one per RA/VA bit, Alg. 1) x {n} pairs "
                                   f"per update; {passes} address-range launches",
                    "peak_source": "tools/redbench --quick in this run: best of random 32-bit LDG (L2 / L1-cached) "
                                   "and RED.OR over a 64 MiB L2-resident buffer (not in MEASURED_PEAKS.json)",
                    "peak_ldg": peaks_acc.get("ldg", 0) / 1e9, "peak_ldg_ca": peaks_acc.get("ldg_ca", 0) / 1e9,
                    "peak_red": peaks_acc.get("red", 0) / 1e9,
                    "update_ms": upd, "launch_ms": per_call[0] / max(1, passes), "update_passes": passes,
                    "update_mode": args.update_mode, "ncu_per_pass": ncu_update_counters()}
        roofline_hbm = {"bound": "hbm", "achieved": 8 * n / (upd / 1e3) / 1e9, "peak": hbm, "unit": "GB/s",
                        "frac": 8 * n / (upd / 1e3) / 1e9 / hbm,
                        "note": "input stream, 8 B/pair algorithmic; peak = MEASURED_PEAKS.json hbm_gbs"}
    line = {"metric": METRIC, "value": value, "unit": "pairs/s", "n_gpus": world, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": dict(config_block(args.workload, spec, world), exchange=exchange),
            "detect_ms": statistics.median(det_ms), "update_ms": upd,
            "post_update_ms": statistics.median(post_ms),
            "windows": ("pipelined: [exchange +] detect(k) + reset overlap update(k+1), two cubes" if pipelined
                        else "serial"),
            "ms_per_step_serial": serial_ms / args.steps,
            "update_pairs_per_s": n * world / (upd / 1e3),
            "n_super_hosts": int(len(hosts)) if hosts is not None else None,
            "roofline": roofline, **({"roofline_hbm": roofline_hbm} if roofline_hbm else {}),
            "gpu_launches": int(launches), "clocks": clk.summary(), "e2e": e2e,
            "baseline_note": "paper publishes no pairs/s (BASELINE.md); its restore time is <11 ms on a Titan Xp"}
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(w)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
