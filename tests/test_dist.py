"""Multi-process host logic of the head sharding / Ulysses exchange, on CPU with
the gloo backend at world size 2 and 3 (ragged token chunks)."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2502_21079_b200 import dist as D


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, N, H, d, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = torch.Generator().manual_seed(5)
        full = torch.randn(N, H, d, generator=g)          # the global [N, H, d] activation
        sizes = D.seq_splits(N, world)
        off = sum(sizes[:rank])
        local = full[off:off + sizes[rank]].contiguous()   # this rank's token chunk
        got = D.ulysses_in(local)
        Hp = H // world
        want = full[:, rank * Hp:(rank + 1) * Hp]
        ok_in = torch.equal(got, want)
        v = D.as_bhnd(got)
        ok_view = (tuple(v.shape) == (1, Hp, N, d) and v.stride(2) == Hp * d and v.stride(1) == d
                   and torch.equal(v[0, 1 % Hp], full[:, rank * Hp + 1 % Hp]))
        back = D.ulysses_out(got * 2.0, sizes)
        ok_out = torch.equal(back, 2.0 * local)
        q.put((rank, ok_in, ok_view, ok_out))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,N", [(2, 64), (3, 50)])
def test_ulysses_roundtrip_gloo(world, N):
    H, d = 6, 8
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, N, H, d, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ok_in, ok_view, ok_out in res:
        assert ok_in and ok_view and ok_out, (rank, ok_in, ok_view, ok_out)


def test_head_range_partitions():
    for H in (1, 5, 24, 48):
        for w in (1, 2, 3, 8):
            rs = [D.head_range(H, w, r) for r in range(w)]
            assert rs[0][0] == 0 and rs[-1][1] == H
            assert all(rs[i][1] == rs[i + 1][0] for i in range(w - 1))
            assert max(b - a for a, b in rs) - min(b - a for a, b in rs) <= 1


def test_lpt_assign():
    costs = [9, 1, 1, 1, 8, 2, 7, 3]
    parts = D.lpt_assign(costs, 3)
    assert sorted(h for p in parts for h in p) == list(range(8))
    loads = [sum(costs[h] for h in p) for p in parts]
    assert max(loads) - min(loads) <= max(costs)
    assert max(loads) <= sum(costs) / 3 + max(costs)


def _timing_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # rank r: total, K1..K4 ms over 5 steps; kept FLOPs of its own layer
        ms = [100.0 + rank, 50.0 + 3 * rank, 30.0, 0.2, 10.0 + 2 * rank]
        value, tmax = D.reduce_step_timings(ms, 1e12 * (rank + 1), 5)
        q.put((rank, value, tmax))
    finally:
        dist.destroy_process_group()


def test_reduce_step_timings_gloo():
    """bench.py's whole-job aggregation at world size 2: times are the max over ranks (per kernel),
    the work is the sum; value = sum(kept FLOPs) x steps / slowest K4 time."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_timing_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    want_t = [101.0, 53.0, 30.0, 0.2, 12.0]
    want_v = (1e12 + 2e12) * 5 / (12.0 / 1e3) / 1e12
    for _, value, tmax in res:
        assert tmax == pytest.approx(want_t)
        assert value == pytest.approx(want_v)
    v1, t1 = D.reduce_step_timings([1.0, 2.0, 3.0, 4.0, 5.0], 2e12, 2)  # single process
    assert t1 == [1.0, 2.0, 3.0, 4.0, 5.0] and v1 == pytest.approx(2e12 * 2 / 5e-3 / 1e12)


def _random_csr(H, nb, seed):
    """A CSR like adaspa_select_blocks writes: rows (h, p), ascending ids, 1..nb per row."""
    g = torch.Generator().manual_seed(seed)
    rows = []
    for _ in range(H * nb):
        n = int(torch.randint(1, nb + 1, (1,), generator=g))
        rows.append(sorted(torch.randperm(nb, generator=g)[:n].tolist()))
    rp = torch.tensor([0] + [len(r) for r in rows]).cumsum(0).to(torch.int32)
    ci = torch.tensor([j for r in rows for j in r], dtype=torch.int32)
    cap = torch.full((H * nb * nb,), -7, dtype=torch.int32)   # capacity buffer, tail is garbage
    cap[: ci.numel()] = ci
    return rp, cap, rows


def _csr_worker(rank, world, port, H, nb, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        h0, h1 = D.head_range(H, world, rank)
        rp, ci, _ = _random_csr(h1 - h0, nb, seed=100 + rank)
        grp, gci = D.gather_csr(rp, ci)
        # the whole layer's rows, rank by rank, as every rank generated them
        want = []
        for r in range(world):
            a, b = D.head_range(H, world, r)
            want += _random_csr(b - a, nb, seed=100 + r)[2]
        got = [gci[grp[i]:grp[i + 1]].tolist() for i in range(H * nb)]
        ok_gather = got == want and int(grp[-1]) == gci.numel()
        costs = D.head_nnz(grp, nb)
        ok_cost = costs == [sum(len(want[h * nb + p]) for p in range(nb)) for h in range(H)]
        assign = D.lpt_assign(costs, world)
        mine = assign[rank]
        prp, pci = D.pack_heads_csr(grp, gci, mine, nb)
        got_p = [pci[prp[i]:prp[i + 1]].tolist() for i in range(len(mine) * nb)]
        ok_pack = got_p == [want[h * nb + p] for h in mine for p in range(nb)] and prp.dtype == torch.int32
        q.put((rank, ok_gather, ok_cost, ok_pack))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,H", [(2, 5), (3, 7)])
def test_gather_and_pack_csr_gloo(world, H):
    """The LPT rebalancing plumbing: all-gather every rank's CSR (ragged head groups, ragged nnz),
    the per-head kept counts, and the CSR of an LPT head set cut out of the whole-layer CSR."""
    nb = 6
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_csr_worker, args=(r, world, port, H, nb, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, *oks in res:
        assert all(oks), (rank, oks)


def _ulysses_assign_worker(rank, world, port, N, H, d, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = torch.Generator().manual_seed(9)
        full = torch.randn(N, H, d, generator=g)
        sizes = D.seq_splits(N, world)
        off = sum(sizes[:rank])
        local = full[off:off + sizes[rank]].contiguous()
        assign = D.lpt_assign([float((7 * h) % 5 + 1) for h in range(H)], world)   # uneven head counts
        got = D.ulysses_in(local, sizes=sizes, assign=assign)
        ok_in = torch.equal(got, full[:, assign[rank]])
        back = D.ulysses_out(got * 3.0, sizes, assign=assign)
        ok_out = torch.equal(back, 3.0 * local)
        q.put((rank, ok_in, ok_out, len(assign[rank])))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,N,H", [(2, 40, 5), (3, 50, 7)])
def test_ulysses_lpt_assign_roundtrip_gloo(world, N, H):
    """Ulysses exchange with an LPT head set per rank (uneven head counts, non-contiguous heads):
    the a2a send order carries the permutation, O comes back in the global head order."""
    d = 4
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_ulysses_assign_worker, args=(r, world, port, N, H, d, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert sum(r[3] for r in res) == H
    for rank, ok_in, ok_out, _ in res:
        assert ok_in and ok_out, (rank, ok_in, ok_out)


def test_imbalance_and_single_process_helpers():
    costs = [10, 1, 1, 1, 1, 2]
    imb, loads = D.imbalance(costs, D.contiguous_assign(6, 2))
    assert loads == [12.0, 4.0] and imb == pytest.approx(12 / 8)
    imb2, _ = D.imbalance(costs, D.lpt_assign(costs, 2))
    assert imb2 <= imb
    rp, ci, rows = _random_csr(2, 4, seed=3)
    grp, gci = D.gather_csr(rp, ci)                          # no process group: as is
    assert torch.equal(grp, rp) and gci.numel() == int(rp[-1])
    assert D.reduce_max([1.0, 2.0]) == [1.0, 2.0] and D.reduce_sum([3.0]) == [3.0]
    assert D.all_gather_floats([1.0]) == [[1.0]]
