"""World-size-2/4 gloo tests of the multi-GPU window orchestration (paper_1901_06207_b200/distributed.py) on CPU.

The per-rank compute (update, OR of the received slices, detect) is done by the oracle here, so these
tests check the host logic that the NCCL path shares: CS ownership, all_to_all split sizes, which peer
bytes reach which owner, and the gather of the host lists (the merged CBA of all routers)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O
from paper_1901_06207_b200 import distributed as D
from paper_1901_06207_b200 import workload as W


def small_params():
    p = O.default_params()
    p.update(r=3, g=256, cbn=[10, 10, 10, 9], clbs=[0, 10, 20])   # L=29: ep [10,10,9], cp [0,0,1]
    assert O.validate(p)[0] == 0
    return p


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, policy, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    p = small_params()
    w = W.generate(W.WindowSpec(n=60_000, n_hosts=2000, n_flows=8000, scanners=(600, 900, 1200)), 5)
    part = W.partition(w.src.size, world, policy, w.src, w.dst)
    sel = part == rank
    local, _ = O.update(p, w.src[sel], w.dst[sel])            # this router's cube
    cube = torch.from_numpy(local)
    n_cs = 1 << p["r"]
    cs_bytes = local.size // n_cs

    def merge_slices(peers, lo, hi):
        mine = cube[lo * cs_bytes: hi * cs_bytes].numpy()
        for s in peers:
            O.merge(mine, s.numpy())

    lo, hi = D.exchange_owned(cube, rank, world, n_cs, cs_bytes, merge_slices)
    st, hosts, stats = O.detect(p, cube.numpy(), 128)
    owned = hosts[(hosts["cs"] >= lo) & (hosts["cs"] < hi)]
    allh = D.gather_hosts(owned, rank, world)
    np.save(os.path.join(out_dir, f"slice{rank}.npy"), cube.numpy()[lo * cs_bytes: hi * cs_bytes])
    if rank == 0:
        np.save(os.path.join(out_dir, "hosts.npy"), allh)
    dist.destroy_process_group()


@pytest.mark.parametrize("world, policy", [(2, "hash-by-pair"), (2, "round-robin"), (4, "hash-by-inner"),
                                           (8, "hash-by-pair")])
def test_gloo_exchange_matches_global_oracle(tmp_path, world, policy):
    mp.spawn(_worker, args=(world, _free_port(), policy, str(tmp_path)), nprocs=world, join=True)
    p = small_params()
    w = W.generate(W.WindowSpec(n=60_000, n_hosts=2000, n_flows=8000, scanners=(600, 900, 1200)), 5)
    whole, _ = O.update(p, w.src, w.dst)
    n_cs = 1 << p["r"]
    cs_bytes = whole.size // n_cs
    for rank in range(world):
        lo, hi = D.owned_range(rank, world, n_cs)
        got = np.load(tmp_path / f"slice{rank}.npy")
        assert np.array_equal(got, whole[lo * cs_bytes: hi * cs_bytes])
    st, ref, _ = O.detect(p, whole, 128)
    hosts = np.load(tmp_path / "hosts.npy", allow_pickle=True)
    assert np.array_equal(hosts, ref)
    assert set(w.planted) <= set(hosts["ip"].tolist())


def test_owned_ranges_cover_every_cs():
    for n_cs in (1, 2, 16, 64):
        for world in (1, 2, 3, 4, 8):
            rs = [D.owned_range(k, world, n_cs) for k in range(world)]
            cov = [cs for lo, hi in rs for cs in range(lo, hi)]
            assert cov == list(range(n_cs))
