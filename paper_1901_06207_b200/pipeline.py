"""Back-to-back windows with the window end overlapped: the schedule bench.py times.

Two cubes (two library handles created with ``detect_overlap = 1``) alternate.  Window k's update
runs on the update stream while window k−1's [exchange +] detect and the reset of its cube run on a
high-priority stream; a cube is handed back to the update stream only after its detect has returned
(and, with an exchange at N > 1, after every peer has finished reading it).  This module is argument
plumbing around the C ABI only (streams, events, the order of calls); every step runs in libcbaa.so.
"""
from __future__ import annotations


class WindowPipeline:
    """``submit(src, dst)`` queues one window's update and returns the host list of the previous window
    (None for the first); ``flush()`` returns the last window's host list.

    exchanges: optional pair of objects with ``exchange(cb, rank, world, n_cs, cs_bytes, stream) -> (lo, hi)``
    and ``window_done(stream)`` (distributed.IpcExchange), one per cube, for N > 1 routers.
    gather:    callable(hosts) -> hosts applied to each detected list (e.g. distributed.gather_hosts)."""

    def __init__(self, cfg, device: int, theta: int, exchanges=None, rank: int = 0, world: int = 1, gather=None,
                 update_stream=None, with_stats: bool = False):
        import torch

        from .cbaa import Cbaa

        cfg = type(cfg).from_buffer_copy(cfg)   # the caller's config is left untouched
        cfg.detect_overlap = 1             # window-end kernels without shared memory: they co-run
        self.cbs = [Cbaa(cfg, device), Cbaa(cfg, device)]
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
        for i, c in enumerate(self.cbs):
            c.reset(self.s_det)
            self.clean[i].record(self.s_det)
        self.k = 0
        self.pending = None
        self.last_stats = None

    def set_exchanges(self, exchanges):
        self.exchanges = exchanges

    def _finish(self, c, done, px, i):
        self.s_det.wait_event(done)
        lo, hi = 0, self.n_cs
        if px:
            lo, hi = px.exchange(c, self.rank, self.world, self.n_cs, self.cs_bytes, self.s_det)
        out, stats, _ = c.detect(self.theta, cs_lo=lo, cs_hi=hi, stream=self.s_det, with_stats=self.with_stats)
        if px:
            px.window_done(self.s_det)
        c.reset(self.s_det)
        self.clean[i].record(self.s_det)
        self.last_stats = stats
        return self.gather(out) if self.gather else out

    def submit(self, src, dst, events=None):
        """events: optional (start, end) CUDA events recorded around the update on the update stream."""
        import torch

        i = self.k % 2
        c = self.cbs[i]
        self.s_upd.wait_event(self.clean[i])
        if events:
            events[0].record(self.s_upd)
        c.update(src, dst, self.s_upd)
        done = torch.cuda.Event()
        done.record(self.s_upd)
        if events:
            events[1].record(self.s_upd)
        out = self._finish(*self.pending) if self.pending else None
        self.pending = (c, done, self.exchanges[i], i)
        self.k += 1
        return out

    def flush(self):
        out = self._finish(*self.pending) if self.pending else None
        self.pending = None
        return out

    @property
    def kernel_launches(self) -> int:
        return sum(c.kernel_launches for c in self.cbs)

    def close(self):
        for c in self.cbs:
            c.close()
