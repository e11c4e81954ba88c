"""The multi-GPU paths of bench.py at world size 1 on one B200: the Ulysses exchange
(sequence-sharded [N_p, H, d] -> head-sharded token-major [N, H_r, d], read by the kernels through
the descriptor strides with no staging copy) feeding the whole hot path through HotPath, and the
LPT plumbing (CSR gather + pack for a permuted head set feeding K4), each against the fp64 oracle.
The a2a/CSR bookkeeping at world size 2-3 is covered with gloo on CPU in tests/test_dist.py."""

import math
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist

import oracle
import workloads
from gpu_helpers import compare_out, csr_rows, np64

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pg():
    import paper_2502_21079_b200  # noqa: F401
    assert torch.cuda.is_available(), "gpu tests need a CUDA device"
    so = socket.socket()
    so.bind(("127.0.0.1", 0))
    port = so.getsockname()[1]
    so.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    yield
    dist.destroy_process_group()


def _oracle_check(lay, q_bhnd, k_bhnd, v_bhnd, hp, heads, what):
    blocks = oracle.block_map(lay.n_video, lay.n_text, lay.block, lay.text_first)
    nb = len(blocks)
    rows = csr_rows(hp.csr.row_ptr, hp.csr.col_idx)
    scale = 1 / math.sqrt(lay.head_dim)
    for i, h in enumerate(heads):
        qq, kk, vv = np64(q_bhnd[0, h]), np64(k_bhnd[0, h]), np64(v_bhnd[0, h])
        od, lse = oracle.dense_attention(qq, kk, vv, scale)
        compare_out(hp.o_dense[0, i], od, hp.lse[0, i], lse, what=f"{what} K1 head {h}")
        kept = rows[i * nb:(i + 1) * nb]
        so, _ = oracle.masked_attention(qq, kk, vv, blocks, kept, scale)
        compare_out(hp.o_sparse[0, i], so, what=f"{what} K4 head {h}")


@pytest.mark.parametrize("d,block", [(128, 128), (64, 64)])
def test_ulysses_hot_path_world1(pg, d, block):
    import paper_2502_21079_b200 as ada
    from paper_2502_21079_b200 import dist as D
    from paper_2502_21079_b200.hotpath import HotPath
    lay = workloads.layout_for("tiny", f=3, h=9, w=11, n_text=37, heads=3, head_dim=d, block=block)
    q, k, v = (x.cuda() for x in workloads.generate_qkv(lay))
    N, H = lay.n, lay.heads
    sizes = D.seq_splits(N, 1)
    loc = [x[0].transpose(0, 1).contiguous() for x in (q, k, v)]               # [N, H, d] (one rank's chunk)
    sh = [D.as_bhnd(D.ulysses_in(x, sizes=sizes)) for x in loc]
    assert sh[0].stride() == (H * d, d, H * d, 1)                              # token-major view
    hp = HotPath(1, H, N, d, block, lay.n_text, lay.text_first, mode=ada.SELECT_RECALL, targets=0.9,
                 token_major=True)
    ptr_before = hp.q.data_ptr()
    hp.run(*sh)
    torch.cuda.synchronize()
    assert hp.q.data_ptr() == ptr_before
    _oracle_check(lay, q, k, v, hp, list(range(H)), f"ulysses d{d} B{block}")
    o_loc = D.ulysses_out(hp.o_sparse[0].transpose(0, 1), sizes)               # back to [N, H, d]
    assert torch.equal(o_loc, hp.o_sparse[0].transpose(0, 1))


def test_hotpath_uses_device_inputs_in_place(pg):
    """HotPath.run on CUDA inputs must not stage them (no device-to-device copy of Q/K/V)."""
    import paper_2502_21079_b200 as ada
    from paper_2502_21079_b200.hotpath import HotPath
    lay = workloads.layout_for("tiny", heads=2, head_dim=64, block=64)
    q, k, v = (x.cuda() for x in workloads.generate_qkv(lay))
    hp = HotPath(1, lay.heads, lay.n, 64, 64, lay.n_text, lay.text_first, mode=ada.SELECT_RECALL, targets=0.9,
                 device="cuda")
    assert hp.device == q.device
    st = hp._stage(q, k, v)
    assert all(a.data_ptr() == b.data_ptr() for a, b in zip(st, (q, k, v)))


def test_lpt_pack_feeds_k4_world1(pg):
    """The --lpt path of bench.py at world size 1 with a PERMUTED head set: gather_csr +
    pack_heads_csr give the CSR of heads [2, 0, 1]; K4 on Q/K/V gathered in that order matches the
    oracle's masked attention on the same rows; the Ulysses a2a with that assignment delivers the
    heads in that order."""
    import paper_2502_21079_b200 as ada
    from paper_2502_21079_b200 import dist as D
    from paper_2502_21079_b200.hotpath import HotPath
    lay = workloads.layout_for("tiny", f=2, h=9, w=20, n_text=20, heads=3, head_dim=128, block=128)
    q, k, v = (x.cuda() for x in workloads.generate_qkv(lay))
    hp = HotPath(1, lay.heads, lay.n, 128, 128, lay.n_text, lay.text_first, mode=ada.SELECT_RECALL, targets=0.8)
    hp.search(q, k, v)
    nb = hp.nb
    grp, gci = D.gather_csr(hp.csr.row_ptr, hp.csr.col_idx)
    heads = [2, 0, 1]
    prp, pci = D.pack_heads_csr(grp, gci, heads, nb)
    idx = torch.tensor(heads, device="cuda")
    q4, k4, v4 = (x.index_select(1, idx).contiguous() for x in (q, k, v))
    o4, _ = ada.block_sparse_attn(q4, k4, v4, prp, pci, block_size=128, n_text=lay.n_text)
    loc = q[0].transpose(0, 1).contiguous()
    got = D.ulysses_in(loc, sizes=[lay.n], assign=[heads])
    assert torch.equal(got, loc[:, heads])
    torch.cuda.synchronize()
    blocks = oracle.block_map(lay.n_video, lay.n_text, 128, lay.text_first)
    rows_all = csr_rows(hp.csr.row_ptr, hp.csr.col_idx)
    rows_p = csr_rows(prp, pci)
    scale = 1 / math.sqrt(128)
    for i, h in enumerate(heads):
        assert rows_p[i * nb:(i + 1) * nb] == rows_all[h * nb:(h + 1) * nb]
        qq, kk, vv = np64(q[0, h]), np64(k[0, h]), np64(v[0, h])
        so, _ = oracle.masked_attention(qq, kk, vv, blocks, rows_p[i * nb:(i + 1) * nb], scale)
        compare_out(o4[0, i], so, what=f"lpt head {h}")
    assert np.isfinite(np64(o4)).all()
