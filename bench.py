#!/usr/bin/env python
"""CBAA window benchmark (BASELINE.json metric: packet pairs/s per window update + window-end detect ms).

One step = one window of the hot path: reset (a7) → update of the window's pairs (a0-a6) → [OR-merge
of router cubes, a8] → detect (a9-a14, host list filled).  Synthetic, seeded workloads:

  C2 (default)  BASELINE config 2: 100M core-network-shaped pairs per GPU (Zipf hosts, ~0.1 % super
                hosts), paper geometry, θ = 1024; weak scaling (each rank one edge router with its own
                100M-pair stream of one global flow set); windows pipelined (detect of window k beside the
                update of window k+1, two cubes).  The last window is checked against the oracle's
                host list (tests/golden/c2_seed1_theta1024_hosts.txt) at N = 1.
  C3            config 3: 4 edge routers × 50M pairs of one flow set, per-router cubes OR-merged, global
                detect; the 4 routers are spread over the N ranks (N ∈ {1, 2, 4}).
  C4            config 4: one 2B-pair window (8 shards of 250M, planted scanners and DDoS victims),
                strong scaling: rank p updates shards [8p/N, 8(p+1)/N) into its cube.
  C1            config 1: the 1M-pair tiny window.

  python bench.py [--gpus N --steps K --warmup W --workload C2]   # our CUDA path, one JSON line on rank 0
  python bench.py --impl reference [...]                          # the CPU oracle as it stands
Multi-GPU: torchrun --nproc-per-node N bench.py --gpus N ...; max-over-ranks device time.
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
GOLDEN_C2 = os.path.join(ROOT, "tests", "golden", "c2_seed1_theta1024_hosts.txt")
NCU_BINNED = os.path.join(ROOT, "profiles", "r02_ncu_binned.json")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=["C2", "C1", "C3", "C4"], default="C2")
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--detect-samples", type=int, default=200, help="detects timed for the latency percentiles")
    ap.add_argument("--passes", type=int, default=0, help="direct update: address-range passes (0 = auto)")
    ap.add_argument("--update-mode", choices=["test_set", "red", "binned"], default="binned",
                    help="binned (default): sample/scatter/apply through shared memory; test_set / red: the "
                         "direct random-access kernel (DESIGN.md §6)")
    ap.add_argument("--no-pipeline", action="store_true",
                    help="C1/C2: run windows strictly one after another (default: pipelined, two cubes)")
    ap.add_argument("--exchange", choices=["nccl", "p2p", "ipc"], default="ipc",
                    help="N>1 window-end exchange: NCCL all_to_all + OR kernel, or the NVLink pull-OR over "
                         "symmetric memory (p2p) / CUDA IPC mappings (ipc)")
    return ap.parse_args()


def dist_env():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("LOCAL_RANK", "0"))


# --------------------------------------------------------------------------------------- workloads
class Plan:
    """What one rank processes per window: a list of streams, each fed to its own router cube (C3) or all
    into one cube (C1/C2/C4)."""

    def __init__(self, name, seed, rank, world):
        from paper_1901_06207_b200 import workload as W
        self.name = name
        if name in ("C1", "C2"):
            self.spec = W.C2 if name == "C2" else W.C1
            # one global flow set (shared seed); each router sees its own packets of those flows
            self.units = [("router", seed if world == 1 else seed * 1000 + rank + 1)]
            self.scaling, self.per_router_cube = "weak", False
            self.global_pairs = self.spec.n * world
            self.desc = (f"{name}: {self.spec.n // 1_000_000}M pairs/GPU, {self.spec.n_hosts} inner hosts, "
                         f"{self.spec.n_flows / 1e6:.1f}M Zipf(s={self.spec.zipf_s}) flows, shuffled")
        elif name == "C3":
            if 4 % world:
                raise SystemExit("C3 has 4 edge routers: run it on N ∈ {1, 2, 4} GPUs")
            self.spec = W.C3_ROUTER
            self.units = [("router", k + 1) for k in range(rank * 4 // world, (rank + 1) * 4 // world)]
            self.scaling, self.per_router_cube = "weak", True
            self.global_pairs = 4 * self.spec.n
            self.desc = "C3: 4 edge routers x 50M pairs of one C2-like flow set, router cubes OR-merged (P:249)"
        else:   # C4
            if 8 % world:
                raise SystemExit("C4 has 8 shards: run it on N ∈ {1, 2, 4, 8} GPUs")
            self.spec = W.c4_spec()
            self.units = [("shard", j + 1) for j in range(rank * 8 // world, (rank + 1) * 8 // world)]
            self.scaling, self.per_router_cube = "strong", False
            self.global_pairs = 8 * self.spec.n
            self.desc = ("C4: one 2B-pair window (8 shards x 250M, 16M Zipf flows over 1.2M hosts, 50 scanners, "
                         "20 DDoS victims with 5% of the packets), strong scaling over the ranks")
        self.seed = seed if name != "C4" else 4

    def generate(self, k):
        """Host arrays (src, dst) of unit k of this rank."""
        from paper_1901_06207_b200 import workload as W
        w = W.generate(self.spec, self.seed, packet_seed=self.units[k][1], with_raw=False)
        return w.src, w.dst

    @property
    def rank_pairs(self):
        return self.spec.n * len(self.units)


def config_block(plan, world, exchange):
    return {"workload": plan.desc, "pairs_per_gpu": plan.rank_pairs, "global_pairs": plan.global_pairs,
            "geometry": "r=4 |RA|=3 |VA|=1 g=4096 c=4096 (128 MiB cube, P:437)", "theta": THETA,
            "parallelism": f"routers{world}" if world > 1 else "single", "exchange": exchange,
            "l2": "inputs (>= 400 MB/GPU) exceed the 126 MB L2, no extra flush; cube reset each window"}


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
            time.sleep(0.005)

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


# --------------------------------------------------------------------------------------- peaks / profiles
def access_peaks():
    """Measured random single-word access rates over an L2-resident 64 MiB buffer (tools/redbench --quick,
    run in this process before the timed region): {"red": RED.OR/s, "ldg": loads/s, "ldg_ca": ...}."""
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


def ncu_binned():
    """Per-launch DRAM bytes and issued L2 REDs of the update kernels from the committed ncu capture."""
    try:
        return json.load(open(NCU_BINNED))
    except Exception:
        return {}


def cpu_info():
    info = {"threads": os.cpu_count()}
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            k, _, v = line.partition(":")
            k, v = k.strip(), v.strip()
            if k == "Model name":
                info["model"] = v
            elif k in ("Socket(s)", "Core(s) per socket", "Thread(s) per core"):
                info[k.lower().replace("(s)", "s").replace(" ", "_")] = int(v)
    except Exception:
        pass
    return info


# --------------------------------------------------------------------------------------- the oracle on the host
def oracle_window(blocks, threads):
    """The oracle as it stands over one window: `threads` workers each run oracle update (Alg. 1) on a
    contiguous block into a private cube, the cubes are OR-merged with the oracle's merge (the shard-OR
    invariant), then the oracle's detect.  Returns (update_s, detect_s, pairs, hosts)."""
    from concurrent.futures import ThreadPoolExecutor

    import numpy as np

    from oracle import oracle as O
    p = O.default_params()
    src = np.concatenate([b[0] for b in blocks]) if len(blocks) > 1 else blocks[0][0]
    dst = np.concatenate([b[1] for b in blocks]) if len(blocks) > 1 else blocks[0][1]
    n = src.size
    cuts = [n * t // threads for t in range(threads + 1)]
    t0 = time.perf_counter()
    with ThreadPoolExecutor(threads) as ex:   # ctypes releases the GIL inside the oracle
        cubes = list(ex.map(lambda t: O.update(p, src[cuts[t]:cuts[t + 1]], dst[cuts[t]:cuts[t + 1]])[0],
                            range(threads)))
    for c in cubes[1:]:
        O.merge(cubes[0], c)
    t1 = time.perf_counter()
    _, hosts, _ = O.detect(p, cubes[0], THETA)
    t2 = time.perf_counter()
    return t1 - t0, t2 - t1, n, hosts


def cpu_baseline(blocks):
    """Oracle timings on the host cores (rank 0, N = 1): single-threaded on a 20M-pair sample, and with
    T = nproc threads (private cubes OR-merged) on the whole window; update and detect separately."""
    info = cpu_info()
    T = info["threads"] or 1
    m = min(20_000_000, blocks[0][0].size)
    u1, d1, n1, _ = oracle_window([(blocks[0][0][:m], blocks[0][1][:m])], 1)
    uT, dT, nT, _ = oracle_window(blocks, T)
    return {"value": nT / (uT + dT), "unit": "pairs/s", "cores": T, "kind": "oracle",
            "sample": f"whole window ({nT} pairs): oracle update on {T} threads (private cubes OR-merged) "
                      f"{uT:.2f} s + oracle detect {dT:.2f} s (θ={THETA})",
            "threads_T": {"threads": T, "pairs": nT, "update_s": uT, "detect_s": dT,
                          "update_pairs_per_s": nT / uT},
            "single_thread": {"threads": 1, "pairs": n1, "update_s": u1, "detect_s": d1,
                              "update_pairs_per_s": n1 / u1,
                              "sample": f"first {n1} pairs of the window (update), detect of that cube"},
            "cpu": info}


def run_reference(args):
    """Reference arm: the oracle as it stands on the same workload, T = nproc threads (rank 0 only)."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    plan = Plan(args.workload, args.seed, 0, 1)
    # C4: the whole 2B-pair window would take minutes per step on the host; one 250M shard per step
    nunits = 1 if args.workload == "C4" else len(plan.units)
    blocks = [plan.generate(k) for k in range(nunits)]
    T = os.cpu_count() or 1
    times, ups, dets = [], [], []
    n = 0
    for k in range(args.warmup + args.steps):
        u, d, n, _ = oracle_window(blocks, T)
        if k >= args.warmup:
            times.append(u + d)
            ups.append(u)
            dets.append(d)
    tot = sum(times)
    value = n * len(times) / tot
    sample = (f"{'first shard (250M pairs) of the 2B window' if args.workload == 'C4' else 'the whole window'} "
              f"per step: oracle update on {T} threads (private cubes OR-merged) + oracle detect (θ={THETA})")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "pairs/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / len(times),
            "higher_is_better": True, "scaling": plan.scaling, "vs_baseline": None, "dtype": "u32",
            "data": "synthetic", "config": config_block(plan, 1, "none"),
            "update_ms": 1e3 * statistics.median(ups), "detect_ms": 1e3 * statistics.median(dets),
            "cpu_baseline": {"value": value, "unit": "pairs/s", "cores": T, "kind": "oracle", "sample": sample,
                             "cpu": cpu_info()},
            "e2e": {"value": value, "unit": "pairs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------------------- our arm
def _allreduce(v: float, op) -> float:
    import torch
    import torch.distributed as dist
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([v], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=op)
    return float(t.item())


def pct(xs, q):
    xs = sorted(xs)
    return xs[min(len(xs) - 1, int(round(q / 100.0 * (len(xs) - 1))))]


def golden_check(hosts):
    """Compare a host list with the oracle's list of the same window (tests/golden, tools/make_golden_c2.py):
    (ip, cs, lp, Z) exact and in order, estimates within 1e-12 relative (+inf exact)."""
    import math
    rows = []
    for line in open(GOLDEN_C2):
        if line.startswith("#") or not line.strip():
            continue
        ip, cs, lp, z, est = line.split()
        rows.append((int(ip, 16), int(cs), int(lp), int(z), float(est)))
    got = [(int(h["ip"]), int(h["cs"]), int(h["lp"]), int(h["z"]), float(h["estimate"])) for h in hosts]
    ok = len(got) == len(rows) and all(
        a[:4] == b[:4] and (a[4] == b[4] if math.isinf(b[4]) else abs(a[4] - b[4]) <= 1e-12 * max(1.0, abs(b[4])))
        for a, b in zip(got, rows))
    return {"golden": os.path.relpath(GOLDEN_C2, ROOT), "hosts": len(got), "oracle_hosts": len(rows), "match": ok}


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_1901_06207_b200 import distributed as D
    from paper_1901_06207_b200.cbaa import Cbaa, cube_bytes, default_config
    from paper_1901_06207_b200.pipeline import WindowPipeline

    rank, world, local = dist_env()
    # one GPU per rank; more ranks than GPUs (functional runs on a 1-GPU box) wrap around and then
    # need CBAA_BENCH_BACKEND=gloo, since NCCL refuses two ranks on one device
    local = local % max(1, torch.cuda.device_count())
    if world > 1:
        backend = os.environ.get("CBAA_BENCH_BACKEND", "nccl")
        dist.init_process_group(backend, device_id=torch.device("cuda", local) if backend == "nccl" else None)
    torch.cuda.set_device(local)
    peaks_acc = access_peaks() if rank == 0 else {}
    plan = Plan(args.workload, args.seed, rank, world)
    # inputs: device-resident per unit (host copies kept only where e2e / the CPU baseline need them)
    keep_host = args.workload != "C4"
    host_blocks, dev_blocks = [], []
    for k in range(len(plan.units)):
        s, d = plan.generate(k)
        dev_blocks.append((torch.from_numpy(s.view(np.int32)).cuda(), torch.from_numpy(d.view(np.int32)).cuda()))
        if keep_host or (k == 0 and rank == 0):
            host_blocks.append((s, d))
        del s, d
    n = plan.rank_pairs
    cfg = default_config()
    cfg.update_passes = args.passes
    cfg.update_mode = {"test_set": 0, "red": 1, "binned": 2}[args.update_mode]
    exchange = args.exchange if world > 1 else "none"
    peer = None
    if exchange == "p2p":
        try:
            peer = D.PeerExchange(cube_bytes(cfg), torch.device("cuda", local))
        except Exception as e:   # no symmetric memory on this box: say so and use NCCL
            print(f"[bench] p2p exchange unavailable ({e}); using nccl", file=sys.stderr)
            exchange = "nccl"
    nh = len(plan.units) if plan.per_router_cube else 1
    cbs = [Cbaa(cfg, local, cube=peer.buf if (peer and j == 0) else None) for j in range(nh)]
    cb = cbs[0]
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

    def exchange_and_detect(s):
        lo, hi = 0, n_cs
        if world > 1:
            with torch.cuda.stream(s):
                if peer:
                    lo, hi = peer.exchange(cb, rank, world, n_cs, cs_bytes, s)
                else:
                    lo, hi = D.exchange_owned(cube_view, rank, world, n_cs, cs_bytes,
                                              lambda ps, a, b: cb.merge_slice(ps, a, b, stream=s))
        hosts, _, rc = cb.detect(THETA, cs_lo=lo, cs_hi=hi, stream=s, with_stats=False)
        if exchange == "p2p":
            with torch.cuda.stream(s):
                peer.window_done()
        elif exchange == "ipc":
            peer.window_done(s)
        return hosts

    def window(ev=None):
        """Serial window: reset, update every unit (per-router cubes OR-merged), exchange, detect."""
        for c in cbs:
            c.reset(stream)
        if ev:
            ev[0].record(stream)
        for j, (s, d) in enumerate(dev_blocks):
            cbs[j if plan.per_router_cube else 0].update(s, d, stream)
        if len(cbs) > 1:
            cb.merge(cbs[1:], stream)
        if ev:
            ev[1].record(stream)
        hosts = exchange_and_detect(stream)
        if ev:
            ev[2].record(stream)
        return D.gather_hosts(hosts, rank, world)

    def launches():
        return sum(c.kernel_launches for c in cbs)

    pipelined = not args.no_pipeline and args.update_mode == "binned" and (world == 1 or exchange == "ipc")
    if not pipelined:
        with torch.cuda.stream(stream):
            for _ in range(max(args.warmup, 3)):   # at least 3 untimed warm-up windows
                window()
        torch.cuda.synchronize()
        evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
        t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        launches0 = launches()
        for c in cbs:
            c.set_phase_timing(True)       # event pair around every update kernel, on its stream
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
        nlaunch = launches() - launches0
        phase_ms, phase_calls = [0.0] * 4, 0
        for c in cbs:
            m, k_ = c.update_phase_ms()
            phase_ms = [a + b for a, b in zip(phase_ms, m)]
            phase_calls += k_
            c.set_phase_timing(False)
        elapsed_ms = t_start.elapsed_time(t_end)
        upd_ms = [e[0].elapsed_time(e[1]) for e in evs]
        lat_handle = cb
        schedule = "serial: reset, update, [merge, exchange], detect"
    else:
        # the object tests/test_gpu_measured.py checks against the oracle window by window
        pipe = WindowPipeline(cfg, local, THETA, rank=rank, world=world, update_stream=stream,
                              gather=lambda h: D.gather_hosts(h, rank, world),
                              routers=len(dev_blocks) if plan.per_router_cube else 1)
        if world > 1:
            pipe.set_exchanges([D.IpcExchange(c, rank, world) for c in pipe.cbs])
        for _ in range(max(args.warmup, 3)):
            pipe.submit(dev_blocks)
        pipe.flush()
        torch.cuda.synchronize()
        launches0 = pipe.kernel_launches
        for c in pipe.handles:
            c.set_phase_timing(True)
        pevs = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(args.steps)]
        t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        with ClockSampler(local) as clk:
            t_start.record(pipe.s_upd)
            for k in range(args.steps):
                pipe.submit(dev_blocks, events=pevs[k])
            hosts = pipe.flush()
            t_end.record(pipe.s_det)
            torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        nlaunch = pipe.kernel_launches - launches0
        phase_ms, phase_calls = [0.0] * 4, 0
        for c in pipe.handles:
            m, k_ = c.update_phase_ms()
            phase_ms = [a + b for a, b in zip(phase_ms, m)]
            phase_calls += k_
            c.set_phase_timing(False)
        elapsed_ms = t_start.elapsed_time(t_end)
        upd_ms = [e[0].elapsed_time(e[1]) for e in pevs]
        # the detect-latency samples below run on a window of the measured configuration
        lat_handle = pipe.cbs[0]
        with torch.cuda.stream(stream):
            st0 = pipe.sets[0]
            for j, (s_, d_) in enumerate(dev_blocks):
                st0[j if plan.per_router_cube else 0].update(s_, d_, stream)
            if len(st0) > 1:
                st0[0].merge(st0[1:], stream)
        if world > 1:
            for px in pipe.exchanges:
                px.close()
            with torch.cuda.stream(stream):
                window()                  # N > 1: the latency below includes the exchange on this cube
            lat_handle = cb
        schedule = ("pipelined: [merge of the router cubes,] detect(k) + reset on a high-priority stream beside "
                    "update(k+1), two cube sets")
    if world > 1:
        elapsed_ms = _allreduce(elapsed_ms, dist.ReduceOp.MAX)

    # ---- window-end detect latency: update finished → host list filled (incl. the exchange at N > 1)
    torch.cuda.synchronize()
    det_host, det_dev = [], []
    a_ev, b_ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(args.detect_samples):
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        a_ev.record(stream)
        if world > 1:
            exchange_and_detect(stream)
        else:
            lat_handle.detect(THETA, stream=stream, with_stats=False)
        b_ev.record(stream)
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        det_host.append(1e3 * (t1 - t0))
        det_dev.append(a_ev.elapsed_time(b_ev))
    detect = {"p50_ms": pct(det_host, 50), "p99_ms": pct(det_host, 99), "max_ms": max(det_host),
              "device_p50_ms": pct(det_dev, 50), "device_p99_ms": pct(det_dev, 99), "samples": len(det_host),
              "includes_exchange": world > 1,
              "clock": "host perf_counter around the detect call (it returns with the host list filled); "
                       "device: CUDA events on the detect stream",
              "target_ms": 10.0}
    if world > 1:
        detect["p99_ms_max_over_ranks"] = _allreduce(detect["p99_ms"], dist.ReduceOp.MAX)

    # ---- end to end through the public API from pinned host memory
    e2e = None
    if not args.no_e2e and keep_host:
        pinned = [(torch.from_numpy(s.view(np.int32)).pin_memory(), torch.from_numpy(d.view(np.int32)).pin_memory())
                  for s, d in host_blocks]
        ke = min(args.steps, 5)

        def e2e_window():
            for c in cbs:
                c.reset(stream)
            for j, (ps, pd) in enumerate(pinned):
                cbs[j if plan.per_router_cube else 0].update_host(ps, pd, stream)   # H2D inside
            if len(cbs) > 1:
                cb.merge(cbs[1:], stream)
            return exchange_and_detect(stream)                                     # D2H of the result

        with torch.cuda.stream(stream):
            e2e_window()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            for _ in range(ke):
                hh = e2e_window()
            b.record(stream)
            torch.cuda.synchronize()
        e2e_ms = a.elapsed_time(b) / ke
        if world > 1:
            e2e_ms = _allreduce(e2e_ms, dist.ReduceOp.MAX)
        e2e = {"value": plan.rank_pairs * world / (e2e_ms / 1e3), "unit": "pairs/s", "ms_per_step": e2e_ms,
               "h2d_bytes_per_step": 8 * n, "d2h_bytes_per_step": 24 * len(hh) + 8,
               "path": "cbaa_update_host (pinned, double-buffered chunks) + [cbaa_merge] + cbaa_detect"}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    ms_step = elapsed_ms / args.steps
    global_pairs = plan.rank_pairs * world if plan.scaling == "weak" else plan.global_pairs
    value = global_pairs * args.steps / (elapsed_ms / 1e3)
    upd = statistics.median(upd_ms)
    peaks = measured_peaks()
    hbm = peaks.get("hbm_gbs", 6550.0)
    per_call = [t / max(1, phase_calls) for t in phase_ms]
    per_call_pairs = n / max(1, phase_calls / max(1, args.steps))   # pairs per update call
    red_peak = peaks_acc.get("red")
    algo_in = 8 * n                       # §8(d): 8 B of input per pair
    algo_bits = 4 * n                     # §8(d): |RA|+|VA| = 4 single-bit ORs per pair
    nb = ncu_binned()

    def ncu_per_pair(key):
        u, m = nb.get("update") or {}, nb.get("pairs_per_update")
        return u[key] / m if (key in u and m) else None

    update_block = {
        "update_ms": upd, "pairs": n,
        "input_hbm": {"achieved_gbs": algo_in / (upd / 1e3) / 1e9, "peak_gbs": hbm,
                      "frac": algo_in / (upd / 1e3) / 1e9 / hbm,
                      "note": "8 B/pair input stream over the whole update (all kernels), SURVEY 8(d)"},
        "l2_red": {"algorithmic_bitsets_per_s": algo_bits / (upd / 1e3), "red_peak_per_s": red_peak,
                   "frac": (algo_bits / (upd / 1e3) / red_peak) if red_peak else None,
                   "issued_l2_reds_per_update": (ncu_per_pair("l2_red_requests") or 0) * n or None,
                   "issued_l2_reds_per_pair": ncu_per_pair("l2_red_requests"),
                   "issued_l2_red_sectors_per_update": (ncu_per_pair("l2_red_sectors") or 0) * n or None,
                   "note": "4 bit-sets/pair / update time vs tools/redbench --quick RED.OR peak (random unique "
                           "words, 64 MiB L2-resident) measured in this run; > 1 means the design sets more "
                           "bits per second than one L2 RED each could (binned: ORs done in shared memory)"},
        # ncu bytes/REDs come from one 100M-pair C2 update: scaled per pair to this run's update
        "l2_hit_pct": {k: (nb.get(k) or {}).get("l2_hit_pct") for k in nb if k.startswith("k_bin")},
        "dram": {"bytes_per_update": ncu_per_pair("dram_bytes") * n if ncu_per_pair("dram_bytes") else None,
                 "algorithmic_bytes": algo_in,
                 "ratio": ncu_per_pair("dram_bytes") / 8 if ncu_per_pair("dram_bytes") else None,
                 "source": os.path.relpath(NCU_BINNED, ROOT) + f" ({nb.get('pairs_per_update')} pairs per captured "
                           "update, scaled per pair)"},
    }
    plan_s = lat_handle.update_plan(int(per_call_pairs))
    if plan_s.startswith("binned"):
        # the kernels the library launched per phase (cbaa_update_plan), e.g. "binned-wide k_bin_sample
        # k_bin_starts k_bin_scatter_w k_bin_apply_w+k_bin_log_w entry_bytes=8"
        words = plan_s.split()
        names, ebytes = words[1:5], int(words[5].split("=")[1])
        scat = names[2]
        kernels = {}
        for name, t in zip(names, per_call):
            kernels[name] = {"ms": t, "share": t / max(1e-9, sum(per_call))}
        tsc = per_call[2]
        design = 8 + ebytes
        roofline = {"kernel": scat, "bound": "hbm",
                    "achieved": 8 * per_call_pairs / (tsc / 1e3) / 1e9, "peak": hbm, "unit": "GB/s",
                    "frac": 8 * per_call_pairs / (tsc / 1e3) / 1e9 / hbm,
                    "traffic": ((nb.get(scat) or {}).get("dram_bytes_per_launch", 0) / nb["pairs_per_update"]
                                * per_call_pairs) if (nb.get(scat) and nb.get("pairs_per_update")) else None,
                    "traffic_source": os.path.relpath(NCU_BINNED, ROOT) + " (ncu --set full, dram__bytes_read+write "
                                      "of the captured launch, scaled to this launch's pairs)",
                    "algorithmic": "SURVEY 8(d): 8 B/pair of input read per launch (pairs per launch x 8 B)",
                    "design_bytes_per_pair": design,
                    "design_frac": design * per_call_pairs / (tsc / 1e3) / 1e9 / hbm,
                    "design_note": f"the binned design also writes a {ebytes} B entry per pair (read back by the apply)",
                    "update_plan": plan_s,
                    "per_launch_ms": tsc,
                    "timing": "CUDA event pair around every update kernel on its launch stream over the timed "
                              "region (cbaa_set_phase_timing), averaged per launch",
                    "peak_source": "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks else "fallback 6550 GB/s",
                    "kernels": kernels, "update": update_block}
    else:
        peak_acc = max(peaks_acc.values()) if peaks_acc else None
        achieved = algo_bits / (upd / 1e3)
        roofline = {"kernel": "k_update", "bound": "lsu_random_word", "achieved": achieved / 1e9, "update_plan": plan_s,
                    "peak": (peak_acc or float("nan")) / 1e9, "unit": "G word-updates/s",
                    "frac": achieved / peak_acc if peak_acc else None, "traffic": None,
                    "peak_source": "tools/redbench --quick in this run (best of random LDG / RED.OR)",
                    "update": update_block}
    line = {"metric": METRIC, "value": value, "unit": "pairs/s", "n_gpus": world, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": plan.scaling, "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": config_block(plan, world, exchange), "windows": schedule,
            "update_ms": upd, "update_pairs_per_s": n / (upd / 1e3),
            "detect_ms": detect["p50_ms"], "detect": detect,
            "n_super_hosts": int(len(hosts)) if hosts is not None else None,
            "roofline": roofline, "gpu_launches": int(nlaunch), "clocks": clk.summary(), "e2e": e2e,
            "access_peaks": {k: v / 1e9 for k, v in peaks_acc.items()},
            "baseline_note": "paper publishes no pairs/s (BASELINE.md); its restore time is <11 ms on a Titan Xp"}
    if args.workload == "C2" and args.seed == 1 and world == 1:
        line["parity"] = golden_check(hosts)
    if e2e is None:
        line["e2e_note"] = "C4 keeps no host copy of its 16 GB window" if not keep_host else "disabled (--no-e2e)"
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(host_blocks)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
