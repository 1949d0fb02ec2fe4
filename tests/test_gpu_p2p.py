"""Caller-owned cubes (cbaa_create_ext) and the symmetric-memory exchange object on one GPU.

The NVLink pull-OR itself needs ≥ 2 GPUs; here we check what one GPU can: the handle works on memory
it does not own (a torch tensor, a symmetric-memory buffer), and the peer-pointer merge path
(cbaa_merge_slice on raw device addresses) is the same kernel the router-merge parity tests cover."""
import os
import socket

import numpy as np
import pytest

from oracle import oracle as O
from paper_1901_06207_b200 import workload as W

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def test_create_ext_on_torch_memory(paper):
    from paper_1901_06207_b200.cbaa import Cbaa, config_from_dict, cube_bytes
    cfg = config_from_dict(paper)
    buf = torch.full((cube_bytes(cfg),), 0xFF, dtype=torch.uint8, device="cuda")
    cb = Cbaa(cfg, 0, cube=buf)
    assert cb.cube_ptr() == buf.data_ptr()
    assert not buf.any()                           # zeroed by the library
    w = W.generate(W.C1, 8)
    cb.reset()
    cb.update(torch.from_numpy(w.src.view(np.int32)).cuda(), torch.from_numpy(w.dst.view(np.int32)).cuda())
    torch.cuda.synchronize()
    ref, _ = O.update(paper, w.src, w.dst)
    assert np.array_equal(buf.cpu().numpy(), ref)
    cb.close()
    assert np.array_equal(buf.cpu().numpy(), ref)  # caller memory survives the handle


def test_merge_slice_from_raw_addresses(paper):
    from paper_1901_06207_b200.cbaa import Cbaa, config_from_dict
    src, dst = W.random_pairs(400_000, 2)
    a, b, g = (Cbaa(config_from_dict(paper), 0) for _ in range(3))
    for h, sl in ((a, slice(0, 200_000)), (b, slice(200_000, None))):
        h.reset()
        h.update(torch.from_numpy(src[sl].view(np.int32)).cuda(), torch.from_numpy(dst[sl].view(np.int32)).cuda())
    g.reset()
    csb = g.nbytes // 16
    g.merge_slice([a.cube_ptr() + 8 * csb, b.cube_ptr() + 8 * csb], 8, 16)
    torch.cuda.synchronize()
    ref, _ = O.update(paper, src, dst)
    cube = g.cube().cpu().numpy()
    assert np.array_equal(cube[8 * csb:], ref[8 * csb:]) and not cube[: 8 * csb].any()


def test_peer_exchange_single_rank(paper):
    import torch.distributed as dist
    from paper_1901_06207_b200 import distributed as D
    from paper_1901_06207_b200.cbaa import Cbaa, config_from_dict, cube_bytes
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        cfg = config_from_dict(paper)
        try:
            peer = D.PeerExchange(cube_bytes(cfg), torch.device("cuda", 0))
        except Exception as e:
            pytest.skip(f"symmetric memory unavailable: {e}")
        cb = Cbaa(cfg, 0, cube=peer.buf)
        w = W.generate(W.C1, 9)
        stream = torch.cuda.Stream()
        with torch.cuda.stream(stream):
            cb.reset(stream)
            cb.update(torch.from_numpy(w.src.view(np.int32)).cuda(), torch.from_numpy(w.dst.view(np.int32)).cuda(),
                      stream)
            lo, hi = peer.exchange(cb, 0, 1, cb.n_cs, cb.nbytes // cb.n_cs, stream)
            hosts, stats, rc = cb.detect(1024, cs_lo=lo, cs_hi=hi, stream=stream)
            peer.window_done()
        torch.cuda.synchronize()
        ref, _ = O.update(paper, w.src, w.dst)
        assert (lo, hi) == (0, 16)
        assert np.array_equal(peer.buf.cpu().numpy(), ref)
        st, oh, _ = O.detect(paper, ref, 1024)
        assert hosts["ip"].tolist() == oh["ip"].tolist()
    finally:
        dist.destroy_process_group()


def _two_rank_worker(rank, world, port, out_dir, exchange):
    import torch.distributed as dist
    from paper_1901_06207_b200 import distributed as D
    from paper_1901_06207_b200.cbaa import Cbaa, config_from_dict, cube_bytes
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    p = O.default_params()
    w = W.generate(W.WindowSpec(n=600_000, n_hosts=20000, n_flows=120000, scanners=(2000,) * 6), 21,
                   packet_seed=100 + rank)
    cfg = config_from_dict(p)
    if exchange == "p2p":
        peer = D.PeerExchange(cube_bytes(cfg), torch.device("cuda", 0))
        cb = Cbaa(cfg, 0, cube=peer.buf)
    elif exchange in ("ipc", "ipc_host"):
        cb = Cbaa(cfg, 0)
        peer = D.IpcExchange(cb, rank, world, device_barrier=exchange == "ipc")
    else:
        peer, cb = None, Cbaa(cfg, 0)
    stream = torch.cuda.Stream()
    n_cs, cs_bytes = cb.n_cs, cb.nbytes // cb.n_cs
    with torch.cuda.stream(stream):
        cb.reset(stream)
        cb.update(torch.from_numpy(w.src.view(np.int32)).cuda(), torch.from_numpy(w.dst.view(np.int32)).cuda(), stream)
        if peer:
            lo, hi = peer.exchange(cb, rank, world, n_cs, cs_bytes, stream)
        else:   # gloo cannot move CUDA tensors: stage the cube through host memory
            host = cb.cube().cpu()
            def merge(peers, lo_, hi_):
                cb.merge_slice([q.cuda() for q in peers], lo_, hi_, stream=stream)
            lo, hi = D.exchange_owned(host, rank, world, n_cs, cs_bytes, merge)
        hosts, stats, rc = cb.detect(1024, cs_lo=lo, cs_hi=hi, stream=stream)
        if exchange == "p2p":
            peer.window_done()
        elif exchange in ("ipc", "ipc_host"):
            peer.window_done(stream)
    torch.cuda.synchronize()
    if exchange in ("ipc", "ipc_host"):
        assert cb.peer_status() == 0
        peer.close()
    np.save(os.path.join(out_dir, f"src{rank}.npy"), w.src)
    np.save(os.path.join(out_dir, f"dst{rank}.npy"), w.dst)
    np.save(os.path.join(out_dir, f"slice{rank}.npy"), cb.cube().cpu().numpy()[lo * cs_bytes: hi * cs_bytes])
    allh = D.gather_hosts(hosts, rank, world)
    if rank == 0:
        np.save(os.path.join(out_dir, "hosts.npy"), allh)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("exchange", ["ipc", "ipc_host", "p2p", "host"])
def test_two_ranks_one_gpu(tmp_path, exchange):
    """Two router processes sharing one B200: the pull-OR over CUDA IPC mappings of the peer's cube (ipc)
    end to end — handle exchange, barriers, merge_slice reading the peer's memory — the staged path
    (host), and the symmetric-memory variant (p2p; torch refuses two ranks on one device, so it skips),
    each against the oracle of the two streams together."""
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    try:
        mp.spawn(_two_rank_worker, args=(2, port, str(tmp_path), exchange), nprocs=2, join=True)
    except Exception as e:
        if exchange == "p2p" and "symm" in str(e).lower():
            pytest.skip(f"symmetric memory with two processes on one GPU unavailable: {e}")
        raise
    p = O.default_params()
    src = np.concatenate([np.load(tmp_path / f"src{r}.npy") for r in range(2)])
    dst = np.concatenate([np.load(tmp_path / f"dst{r}.npy") for r in range(2)])
    whole, _ = O.update(p, src, dst)
    from paper_1901_06207_b200 import distributed as D
    cs_bytes = whole.size // 16
    for r in range(2):
        lo, hi = D.owned_range(r, 2, 16)
        assert np.array_equal(np.load(tmp_path / f"slice{r}.npy"), whole[lo * cs_bytes: hi * cs_bytes])
    st, ref, _ = O.detect(p, whole, 1024)
    hosts = np.load(tmp_path / "hosts.npy", allow_pickle=True)
    assert hosts["ip"].tolist() == ref["ip"].tolist()
    assert np.allclose(hosts["estimate"], ref["estimate"], rtol=1e-12)


# ------------------------------------------------------------------ device-side barrier, fused pull-OR
def test_peer_barrier_orders_peer_reads(paper):
    """Two routers in one process (two handles, two streams): router 1's merge reads router 0's cube
    right after a cbaa_peer_barrier on each stream; the barrier alone orders router 0's update before
    that read (no host synchronisation between them), for three consecutive epochs."""
    from paper_1901_06207_b200.cbaa import Cbaa, config_from_dict
    a, b = Cbaa(config_from_dict(paper), 0), Cbaa(config_from_dict(paper), 0)
    sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
    csb = a.nbytes // 16
    for epoch, seed in ((1, 3), (2, 4), (3, 5)):
        src, dst = W.random_pairs(3_000_000, seed)
        s_t, d_t = (torch.from_numpy(x.view(np.int32)).cuda() for x in (src, dst))
        torch.cuda.synchronize()
        a.reset(sa)
        b.reset(sb)
        a.update(s_t, d_t, sa)                                    # router 0's window (B has none)
        a.peer_barrier([None, b.cube_ptr()], 2, 0, epoch, sa)
        b.peer_barrier([a.cube_ptr(), None], 2, 1, epoch, sb)
        b.merge_slice([a.cube_ptr() + 8 * csb], 8, 16, sb)        # pulls router 0's CSs 8..15
        torch.cuda.synchronize()
        ref, _ = O.update(paper, src, dst)
        got = b.cube().cpu().numpy()
        assert np.array_equal(got[8 * csb:], ref[8 * csb:]) and not got[: 8 * csb].any()
    assert a.peer_status() == 0 and b.peer_status() == 0


def test_peer_barrier_times_out_instead_of_hanging(paper, monkeypatch):
    """A peer that never arrives: the barrier kernel gives up after CBAA_BARRIER_TIMEOUT_MS and flags it."""
    from paper_1901_06207_b200.cbaa import Cbaa, config_from_dict
    monkeypatch.setenv("CBAA_BARRIER_TIMEOUT_MS", "50")
    a, b = Cbaa(config_from_dict(paper), 0), Cbaa(config_from_dict(paper), 0)
    a.peer_barrier([None, b.cube_ptr()], 2, 0, 1)
    torch.cuda.synchronize()
    assert a.peer_status() == 1 and b.peer_status() == 0


@pytest.mark.parametrize("lo, hi", [(0, 16), (4, 12), (15, 16)])
def test_merge_slice_zc_then_detect(paper, lo, hi):
    """The pull-OR fused with the zero counts: the cube slice, the zero counts and the owned-range detect
    equal the oracle of the OR of both routers' streams; a second detect (counts recomputed) agrees."""
    from paper_1901_06207_b200.cbaa import Cbaa, config_from_dict
    from tests.test_gpu_parity import assert_hosts_equal, assert_stats_equal
    w = W.generate(W.WindowSpec(n=1_200_000, n_hosts=30000, n_flows=200000, scanners=(2500,) * 40), 31)
    part = W.partition(w.src.size, 2, "hash-by-pair", w.src, w.dst)
    hs = [Cbaa(config_from_dict(paper), 0) for _ in range(2)]
    for k, h in enumerate(hs):
        h.reset()
        sel = part == k
        h.update(torch.from_numpy(w.src[sel].view(np.int32)).cuda(), torch.from_numpy(w.dst[sel].view(np.int32)).cuda())
    csb = hs[0].nbytes // 16
    hs[0].merge_slice_zc([hs[1].cube_ptr() + lo * csb], lo, hi)
    h1, s1, rc1 = hs[0].detect(1024, cs_lo=lo, cs_hi=hi)
    h2, s2, rc2 = hs[0].detect(1024, cs_lo=lo, cs_hi=hi)
    torch.cuda.synchronize()
    ref, _ = O.update(paper, w.src, w.dst)
    assert np.array_equal(hs[0].cube().cpu().numpy()[lo * csb: hi * csb], ref[lo * csb: hi * csb])
    st, oh, ostats = O.detect(paper, ref, 1024)
    oh = oh[(oh["cs"] >= lo) & (oh["cs"] < hi)]
    assert_stats_equal(s1, ostats[lo:hi])
    assert_hosts_equal(h1, oh)
    assert_stats_equal(s2, ostats[lo:hi])
    assert_hosts_equal(h2, oh)
