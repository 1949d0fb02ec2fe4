"""Back-to-back windows with the window end overlapped: the schedule bench.py times.

Two cube sets alternate (library handles created with ``detect_overlap = 1``).  Window k's update runs
on the update stream while window k−1's [exchange +] detect and the reset of its cubes run on a
high-priority stream; a cube set is handed back to the update stream only after its detect has returned
(and, with an exchange at N > 1, after every peer has finished reading it).  A set holds one cube, or
one per edge router of this rank (config 3): the routers' cubes are OR-merged into the first
on the update stream before the window end.  This module is argument plumbing around the C ABI only
(streams, events, the order of calls); every step runs in libcbaa.so.
"""
from __future__ import annotations


class WindowPipeline:
    """``submit(src, dst)`` — or ``submit([(src, dst), ...])`` for several streams — queues one window's
    update and returns the host list of the previous window (None for the first); ``flush()`` returns
    the last window's host list.

    routers:   cubes per set; with routers > 1 stream j of a window goes to router cube j and the cubes
               are merged, with routers == 1 every stream of the window goes into the one cube.
    exchanges: optional pair of objects with ``exchange(cb, rank, world, n_cs, cs_bytes, stream) -> (lo, hi)``
               and ``window_done(stream)`` (distributed.IpcExchange), one per set, for N > 1 ranks.
    gather:    callable(hosts) -> hosts applied to each detected list (e.g. distributed.gather_hosts)."""

    def __init__(self, cfg, device: int, theta: int, exchanges=None, rank: int = 0, world: int = 1, gather=None,
                 update_stream=None, with_stats: bool = False, routers: int = 1):
        import torch

        from .cbaa import Cbaa

        cfg = type(cfg).from_buffer_copy(cfg)   # the caller's config is left untouched
        cfg.detect_overlap = 1             # window-end kernels without shared memory: they co-run
        self.sets = [[Cbaa(cfg, device) for _ in range(routers)] for _ in range(2)]
        self.cbs = [s[0] for s in self.sets]   # the cube each window is detected on
        self.routers = routers
        self.theta, self.rank, self.world = theta, rank, world
        self.exchanges = exchanges or [None, None]
        self.gather = gather
        self.with_stats = with_stats
        _, hi_pri = torch.cuda.Stream.priority_range()
        self.s_upd = update_stream or torch.cuda.Stream(device=device)
        self.s_det = torch.cuda.Stream(device=device, priority=hi_pri)
        self.n_cs = self.cbs[0].n_cs
        self.cs_bytes = self.cbs[0].nbytes // self.n_cs
        self.clean = [torch.cuda.Event(), torch.cuda.Event()]
        for i, st in enumerate(self.sets):
            for c in st:
                c.reset(self.s_det)
            self.clean[i].record(self.s_det)
        self.k = 0
        self.pending = None
        self.last_stats = None

    def set_exchanges(self, exchanges):
        self.exchanges = exchanges

    def _finish(self, i, done):
        c, px = self.cbs[i], self.exchanges[i]
        self.s_det.wait_event(done)
        lo, hi = 0, self.n_cs
        if px:
            lo, hi = px.exchange(c, self.rank, self.world, self.n_cs, self.cs_bytes, self.s_det)
        out, stats, _ = c.detect(self.theta, cs_lo=lo, cs_hi=hi, stream=self.s_det, with_stats=self.with_stats)
        if px:
            px.window_done(self.s_det)
        for r in self.sets[i]:
            r.reset(self.s_det)
        self.clean[i].record(self.s_det)
        self.last_stats = stats
        return self.gather(out) if self.gather else out

    def submit(self, src, dst=None, events=None):
        """src, dst: one stream of device tensors, or src = a list of (src, dst) pairs and dst = None.
        The update runs asynchronously on the update stream: the caller keeps the tensors alive until the
        window's hosts have been returned (the C ABI's ownership rule).
        events: optional (start, end) CUDA events recorded around the update (and merge) on the update
        stream."""
        import torch

        blocks = [(src, dst)] if dst is not None else list(src)
        i = self.k % 2
        st = self.sets[i]
        self.s_upd.wait_event(self.clean[i])
        if events:
            events[0].record(self.s_upd)
        for j, (s, d) in enumerate(blocks):
            st[j if self.routers > 1 else 0].update(s, d, self.s_upd)
        if self.routers > 1:
            st[0].merge(st[1:], self.s_upd)      # the routers' cubes OR-merged
        done = torch.cuda.Event()
        done.record(self.s_upd)
        if events:
            events[1].record(self.s_upd)
        out = self._finish(*self.pending) if self.pending else None
        self.pending = (i, done)
        self.k += 1
        return out

    def flush(self):
        out = self._finish(*self.pending) if self.pending else None
        self.pending = None
        return out

    @property
    def handles(self):
        return [c for st in self.sets for c in st]

    @property
    def kernel_launches(self) -> int:
        return sum(c.kernel_launches for c in self.handles)

    def close(self):
        for c in self.handles:
            c.close()
