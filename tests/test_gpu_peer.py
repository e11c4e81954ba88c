"""The Ulysses exchange over peer memory (dist.PeerExchange: CUDA IPC-mapped receive buffers,
copy-engine 2-D copies, stream-ordered flags) against the plain re-layout it
must produce: rank r receives all tokens of its head list ([N, H_r, d], token-major), and O goes
back to every rank's token chunk with heads in global order.  World size 1 in-process, and world
sizes 2 and 3 as separate processes sharing this one GPU (CUDA IPC works across processes on one
device, so the handle exchange, the mapped copies and the flag handshake all run for real; only
NVLink itself is not exercised), with uneven token chunks and contiguous and permuted (LPT-style)
head lists, over several epochs (the release handshake)."""

import os
import socket

import pytest
import torch

pytestmark = pytest.mark.gpu


def _global(N, H, d, seed):
    g = torch.Generator().manual_seed(seed)
    return [torch.randn(N, H, d, generator=g).to(torch.bfloat16) for _ in range(3)]


def _run_rank(rank, world, port, N, H, d, assign, epochs, out):
    import torch.distributed as dist
    from paper_2502_21079_b200 import dist as D
    torch.cuda.set_device(0)
    if world > 1:
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    dev = torch.device("cuda", 0)
    sizes = D.seq_splits(N, world)
    off = sum(sizes[:rank])
    ex = D.PeerExchange(N, H, d, sizes, assign, dev)
    st = torch.cuda.current_stream()
    ok = True
    for ep in range(epochs):
        xs_g = _global(N, H, d, 7 + ep)
        xs = [x[off:off + sizes[rank]].contiguous().to(dev) for x in xs_g]
        ex.push_in(xs, st)
        recv = ex.wait_in(st)
        mine = assign[rank]
        for i in range(3):
            want = xs_g[i][:, mine].to(dev)                        # [N, H_r, d]: all tokens, my heads
            ok &= bool(torch.equal(recv[i], want))
        o = recv[0].clone()                                         # "O" = my Q slice, token-major
        ex.release_in(st)
        ex.push_out(o, st)
        back = ex.wait_out(st)
        ok &= bool(torch.equal(back, xs[0]))                       # my token chunk of every head, global order
        ex.release_out(st)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ex.close()
    if world > 1:
        dist.destroy_process_group()
    out[rank] = ok


def _spawn_main(rank, world, port, N, H, d, assign, epochs, q):
    res = {}
    _run_rank(rank, world, port, N, H, d, assign, epochs, res)
    q.put((rank, res[rank]))


def test_peer_exchange_world1():
    """One process: the exchange is local copies; a permuted head list exercises the run logic."""
    N, H, d = 1000, 6, 64
    res = {}
    _run_rank(0, 1, 0, N, H, d, [[3, 4, 0, 1, 5, 2]], 2, res)
    assert res[0]


@pytest.mark.parametrize("world,assign", [
    (2, [[0, 1, 2], [3, 4, 5]]),
    (2, [[1, 4], [0, 2, 3, 5]]),                  # LPT-style: uneven, non-contiguous head sets
    (3, [[5], [0, 1, 2], [3, 4]]),
])
def test_peer_exchange_multiprocess_one_gpu(world, assign):
    import torch.multiprocessing as mp
    N, H, d = 1001, 6, 64                         # uneven token chunks
    so = socket.socket()
    so.bind(("127.0.0.1", 0))
    port = so.getsockname()[1]
    so.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_spawn_main, args=(r, world, port, N, H, d, assign, 3, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = {}
    for _ in range(world):
        r, ok = q.get(timeout=240)
        got[r] = ok
    for p in procs:
        p.join(timeout=60)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    assert got == {r: True for r in range(world)}, got
