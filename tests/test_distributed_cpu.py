"""Multi-rank partition and exchange logic on CPU (gloo, world size 2).

The product's partition (order_owner, ring_blocks, shard_bins) and its
torch.distributed exchanger (TorchExchange) move data between two CPU
processes; each rank's local SHT stages are computed by the CPU oracle (test
infrastructure).  The gathered result must equal the unsharded oracle SHT.
"""
import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parents[1]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, L, real, scheme, q):
    sys.path.insert(0, str(ROOT))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as orc
        from paper_1211_1680_b200 import distributed as D
        from paper_1211_1680_b200.bench import gaussian_coeffs

        f = gaussian_coeffs(L, np.random.default_rng(L), real_signal=real).coeffs
        full_map = orc.sh_synthesis(f[None], L, real, scheme)            # (1, L, N)
        owner = D.order_owner(L, world)
        blocks = D.ring_blocks(L, world)
        orders = [np.nonzero(owner == r)[0] for r in range(world)]
        bins = [D.shard_bins(L, o, real) for o in orders]
        t0, t1 = blocks[rank]
        ex = D.TorchExchange()
        nb = L if real else 2 * L - 1

        # ---- analysis: my rings -> all-to-all -> my orders
        rows = full_map[:, t0:t1, :]
        gcol = torch.from_numpy(orc.rings_forward(rows, L, real))       # (1, nb, t_me)
        sends = {rank: [gcol[:, torch.as_tensor(bins[q]), :].contiguous() for q in range(world)]}
        sizes = {rank: [len(bins[rank]) * (blocks[q][1] - blocks[q][0]) for q in range(world)]}
        recv = ex.all_to_all(sends, sizes)[rank]
        H = torch.cat([recv[q].view(1, len(bins[rank]), blocks[q][1] - blocks[q][0])
                       for q in range(world)], dim=2).numpy()
        if scheme == "mw":
            H = orc.mw_theta_stage(H, L, real, bins=bins[rank])
        Hfull = np.zeros((1, nb, L), dtype=complex)
        Hfull[:, bins[rank], :] = H
        f_my = orc.legendre_ana(Hfull, L, real, scheme, orc.ring_weights(scheme, L),
                                orders=orders[rank])[0]
        # ---- synthesis: my orders -> all-to-all -> my rings
        G = orc.legendre_synth(f[None], L, real, scheme, orders=orders[rank])  # (1, L, nb)
        glocal = torch.from_numpy(np.ascontiguousarray(G[:, :, bins[rank]]))
        sends = {rank: [glocal[:, blocks[q][0]:blocks[q][1], :].contiguous() for q in range(world)]}
        sizes = {rank: [(t1 - t0) * len(bins[q]) for q in range(world)]}
        recv = ex.all_to_all(sends, sizes)[rank]
        ring = np.zeros((1, t1 - t0, nb), dtype=complex)
        for qq in range(world):
            ring[:, :, bins[qq]] = recv[qq].view(1, t1 - t0, len(bins[qq])).numpy()
        # the MW pole pin applies to the last ring of the grid only (its owner)
        pin = scheme if t1 == L else "gl"
        my_rows = orc.rings_inverse(ring, L, real, pin) if t1 > t0 else ring
        q.put((rank, f_my, orders[rank], my_rows, (t0, t1), f, full_map))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("scheme", ["gl", "mw"])
@pytest.mark.parametrize("real", [False, True])
def test_two_rank_sharded_sht(scheme, real):
    L, world = 17, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, L, real, scheme, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    f = res[0][5]
    full_map = res[0][6]
    got_f = np.zeros_like(f)
    for rank, f_my, orders, rows, (t0, t1), _, _ in res:
        idx = np.concatenate([np.arange(m, L) ** 2 + np.arange(m, L) + s * m
                              for m in orders for s in ((1, -1) if m else (1,))])
        got_f[idx] = f_my[idx]
        if t1 > t0:
            assert np.abs(rows - full_map[:, t0:t1]).max() <= 1e-12
    assert np.abs(got_f - f).max() <= 1e-10


def _xchg_worker(rank, world, port, q):
    sys.path.insert(0, str(ROOT))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1211_1680_b200 import distributed as D

        ex = D.TorchExchange()
        # two keys (two scales of one grouped exchange), blocks of rank-dependent shape
        sends, shapes = {}, {}
        for key, rows in (("s000", 3), ("s001", 2)):
            sends[key] = [torch.full((1, rows + d, 2), complex(10 * rank + d, key == "s001"),
                                     dtype=torch.complex128) for d in range(world)]
            shapes[key] = [(1, rows + rank, 2) for src in range(world)]
        got = ex.exchange({rank: sends}, {rank: shapes})[rank]
        ok = True
        for key in ("s000", "s001"):
            for src in range(world):
                want = complex(10 * src + rank, key == "s001")
                t = got[key][src]
                ok &= bool(torch.all(t == want).item()) and tuple(t.shape)[1] == (3 if key == "s000" else 2) + rank
        buf = torch.full((5,), complex(rank + 1, -rank), dtype=torch.complex128)
        ex.all_reduce({rank: buf})
        ok &= bool(torch.all(buf == complex(3, -1)).item())
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


def test_grouped_exchange_and_all_reduce():
    """TorchExchange.exchange (grouped P2P, one message per key and peer, own
    block by reference) and all_reduce on gloo, world size 2."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_xchg_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res == {0: True, 1: True}


def test_whole_scale_owners_balance():
    from paper_1211_1680_b200 import distributed as D

    bands = [2, 2, 4, 8, 16, 32, 64, 128, 256, 512, 1024, 2048, 4096, 4096]   # C5
    own = D.whole_scale_owners(bands, 8)
    assert sorted(own) == [j for j, k in enumerate(bands) if k <= 256]
    assert own[8] != own[7]                 # the two largest whole scales apart
    assert D.whole_scale_owners(bands, 1) == {j: 0 for j in own}
    assert D.whole_scale_owners([27, 27, 81, 243, 729, 2048, 2048], 4, whole_max=0) == {}
