"""Multi-GPU window: the paper's distributed edge routers on one NVLink domain.

Each rank is one local server: it updates its own packet shard into its own cube (no communication
during the window).  At window end the global CBA is the bitwise OR of the local cubes (Q1).
NCCL has no bitwise OR reduction, so the exchange is reduce-scatter shaped:

  * rank p owns the CS range [lo_p, hi_p) (Alg. 2/3 are independent per CS);
  * ``all_to_all_single`` sends every rank the bytes of its owned CSs from every peer cube;
  * the owner ORs the k−1 received slices into its own slice (``cbaa_merge_slice`` kernel);
  * the owner runs detect on its CSs only; the small host lists are gathered to rank 0.

Per-GPU traffic is (k−1)/k of one cube each way instead of (k−1) cubes for an all-gather.
The orchestration is backend-agnostic so that the gloo CPU tests can drive it with the oracle.
"""
from __future__ import annotations

import numpy as np


def owned_range(rank: int, world: int, n_cs: int):
    """Contiguous CS range of a rank (every CS owned by exactly one rank)."""
    return rank * n_cs // world, (rank + 1) * n_cs // world


def exchange_owned(cube, rank: int, world: int, n_cs: int, cs_bytes: int, merge_slices, group=None):
    """OR-reduce-scatter of per-rank cubes by CS ownership.

    cube:          this rank's cube as a contiguous uint8 torch tensor (device or CPU per backend)
    merge_slices:  callable(list_of_peer_slices, lo, hi) that ORs the peers' bytes of CSs [lo, hi)
                   into this rank's cube (the product passes Cbaa.merge_slice).
    Returns the owned (lo, hi)."""
    import torch
    import torch.distributed as dist

    lo, hi = owned_range(rank, world, n_cs)
    if world == 1:
        return lo, hi
    in_splits = [(owned_range(k, world, n_cs)[1] - owned_range(k, world, n_cs)[0]) * cs_bytes for k in range(world)]
    mine = (hi - lo) * cs_bytes
    out = torch.empty(mine * world, dtype=torch.uint8, device=cube.device)
    dist.all_to_all_single(out, cube, output_split_sizes=[mine] * world, input_split_sizes=in_splits, group=group)
    peers = [out[k * mine:(k + 1) * mine] for k in range(world) if k != rank]
    if mine:
        merge_slices(peers, lo, hi)
    return lo, hi


class PeerExchange:
    """The exchange without a staging collective: every rank's cube lives in torch symmetric memory.
    After the symmetric-memory device barrier the owner either lets the NVSwitch OR all ranks' bytes of
    its CS range (NVLS ``multimem.ld_reduce``, ``cbaa_merge_multicast``) when the buffer has a multicast
    address, or pulls the peers' slices over NVLink and ORs them with its own in one kernel that also
    computes the window-end zero counts (``cbaa_merge_slice_zc``).  A second barrier keeps any rank from
    resetting its cube for the next window while a peer may still be reading it."""

    def __init__(self, nbytes: int, device, group=None):
        import torch
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm_mem

        self.group = group or dist.group.WORLD
        self.buf = symm_mem.empty(nbytes, dtype=torch.uint8, device=device)
        self.hdl = symm_mem.rendezvous(self.buf, self.group)
        self.ptrs = [int(p) for p in self.hdl.buffer_ptrs]
        self.mc = int(getattr(self.hdl, "multicast_ptr", 0) or 0)

    def exchange(self, cb, rank: int, world: int, n_cs: int, cs_bytes: int, stream):
        lo, hi = owned_range(rank, world, n_cs)
        self.hdl.barrier(channel=0)               # every router's update is complete and visible
        if hi > lo and world > 1:
            if self.mc:
                cb.merge_multicast(self.mc, lo, hi, stream=stream)
            else:
                cb.merge_slice_zc([p + lo * cs_bytes for k, p in enumerate(self.ptrs) if k != rank], lo, hi,
                                  stream=stream)
        return lo, hi

    def window_done(self):
        self.hdl.barrier(channel=1)               # peers are done reading before the next reset


class IpcExchange:
    """The pull-OR over CUDA IPC mappings of the peers' library-owned cubes (no torch symmetric memory
    needed; works between processes on one device too).  Synchronisation stays on the device: each cube
    allocation carries a signal area, and ``cbaa_peer_barrier`` (one CTA, stream-ordered after the
    window's update) raises this rank's epoch in every peer's area and waits for theirs — no host
    round trip in the window.  Then the owner's ``cbaa_merge_slice_zc`` reads the peers' slices of its CS
    range over NVLink, ORs them in and records the zero counts; ``window_done`` is a second device
    barrier that fences the next reset.  ``device_barrier=False`` falls back to stream sync + a
    process-group barrier (the round-1 scheme)."""

    def __init__(self, cb, rank: int, world: int, group=None, device_barrier: bool = True):
        import torch.distributed as dist

        self.cb, self.rank, self.world, self.group = cb, rank, world, group
        self.device_barrier = device_barrier
        handles = [None] * world
        dist.all_gather_object(handles, cb.ipc_export(), group=group)
        self.ptrs = [None if k == rank else cb.ipc_open(hd) for k, hd in enumerate(handles)]
        self.epoch = 0

    def _barrier(self, stream):
        import torch.distributed as dist

        if self.device_barrier:
            self.epoch += 1
            self.cb.peer_barrier(self.ptrs, self.world, self.rank, self.epoch, stream=stream)
        else:
            stream.synchronize()
            dist.barrier(group=self.group)

    def exchange(self, cb, rank: int, world: int, n_cs: int, cs_bytes: int, stream):
        lo, hi = owned_range(rank, world, n_cs)
        self._barrier(stream)                     # every router's update is complete and visible
        peers = [p + lo * cs_bytes for p in self.ptrs if p is not None]
        if peers and hi > lo:
            cb.merge_slice_zc(peers, lo, hi, stream=stream)
        return lo, hi

    def window_done(self, stream=None):
        import torch

        self._barrier(stream if stream is not None else torch.cuda.current_stream())   # peers done reading

    def close(self):
        for p in self.ptrs:
            if p is not None:
                self.cb.ipc_close(p)
        self.ptrs = []


def gather_hosts(hosts: np.ndarray, rank: int, world: int, group=None):
    """Collect every rank's host list on rank 0, in the output order of S:418."""
    import torch.distributed as dist

    if world == 1:
        return hosts
    objs = [None] * world if rank == 0 else None
    dist.gather_object(hosts, objs, dst=0, group=group)
    if rank != 0:
        return None
    allh = np.concatenate(objs) if objs else hosts[:0]
    from .cbaa import sort_hosts
    return sort_hosts(allh)   # S:418 order, in the library (cbaa_sort_hosts)
