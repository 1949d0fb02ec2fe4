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
    elif exchange == "ipc":
        cb = Cbaa(cfg, 0)
        peer = D.IpcExchange(cb, rank, world)
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
        elif exchange == "ipc":
            peer.window_done(stream)
    torch.cuda.synchronize()
    if exchange == "ipc":
        peer.close()
    np.save(os.path.join(out_dir, f"src{rank}.npy"), w.src)
    np.save(os.path.join(out_dir, f"dst{rank}.npy"), w.dst)
    np.save(os.path.join(out_dir, f"slice{rank}.npy"), cb.cube().cpu().numpy()[lo * cs_bytes: hi * cs_bytes])
    allh = D.gather_hosts(hosts, rank, world)
    if rank == 0:
        np.save(os.path.join(out_dir, "hosts.npy"), allh)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("exchange", ["ipc", "p2p", "host"])
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
