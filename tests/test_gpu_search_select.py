"""The whole RECALL-mode search step t_w in one call (adaspa_search_select: the fused dense pass, the
block masses with the fresh LSE and, in the same CTA, the row's selection; then the CSR), checked
against the fp64 oracle: O / LSE as K1, block masses as W_sum_attn with the fresh
LSE (reading R4), and the selection (PAPER.md:228-232 per q-block row, text sink
PAPER.md:549, readings R7-R13, R25) bit-exact against the oracle's greedy on the same fp32 masses --
the criterion of K3's own exact test -- and identical to K3 (adaspa_select_blocks) on those masses."""

import math

import numpy as np
import pytest
import torch

import oracle
import workloads
from gpu_helpers import MASS_REL, compare_out, csr_rows, np64

pytestmark = pytest.mark.gpu

CASES = [
    ("tiny", {}, [0.9, 0.9]),
    ("tiny_tf", {}, [0.5, 0.99]),
    ("tiny", dict(f=5, h=9, w=11, n_text=37, head_dim=128, block=128), [0.8, 0.95]),
    ("tiny_tf", dict(f=3, h=10, w=13, n_text=77, head_dim=64, block=128), [0.9, 1.0]),
    ("tiny", dict(f=4, h=9, w=10, n_text=45, head_dim=128, block=64, heads=3), [0.3, 0.9, 0.97]),
    ("tiny_tf", dict(f=6, h=10, w=21, n_text=77, head_dim=128, block=128, heads=3), [0.9, 0.0, 0.7]),
    ("tiny_tf", dict(f=3, h=7, w=13, n_text=29, head_dim=64, block=64, heads=2), [0.9, 0.6]),  # odd nb
]


@pytest.fixture(scope="module")
def ada():
    import paper_2502_21079_b200 as m
    assert torch.cuda.is_available(), "gpu tests need a CUDA device"
    return m


def _same_csr(a, b):
    assert torch.equal(a.row_ptr, b.row_ptr)
    n = int(a.row_ptr[-1].item())
    assert torch.equal(a.col_idx[:n], b.col_idx[:n])
    assert torch.equal(a.head_nnz, b.head_nnz)
    assert torch.equal(a.head_recall, b.head_recall)


def _row_order_ok(out, rows):
    order = out.row_order.cpu().numpy()
    cnt = np.diff(out.row_ptr.cpu().numpy())
    assert sorted(order.tolist()) == list(range(rows))
    assert (np.diff(cnt[order]) <= 0).all()


def _check(ada, lay, q, k, v, targets, flags=1, batch=1, heads_per_pass=0):
    kw = dict(block_size=lay.block, n_text=lay.n_text, text_first=lay.text_first)
    o, lse, M, out = ada.search_select(q, k, v, target=targets, flags=flags, heads_per_pass=heads_per_pass, **kw)
    torch.cuda.synchronize()
    blocks = oracle.block_map(lay.n_video, lay.n_text, lay.block, lay.text_first)
    nb = len(blocks)
    L = np.array([b.length for b in blocks], dtype=np.float64)
    scale = 1 / math.sqrt(lay.head_dim)
    rows = csr_rows(out.row_ptr, out.col_idx)
    H = lay.heads
    for b in range(batch):
        for h in range(H):
            qq, kk, vv = np64(q[b, h]), np64(k[b, h]), np64(v[b, h])
            ro, rl = oracle.dense_attention(qq, kk, vv, scale)
            compare_out(o[b, h], ro, lse[b, h], rl, what=f"{lay} b{b} h{h}")
            Mo = oracle.block_mass(qq, kk, lse[b, h].double().cpu().numpy(), blocks, scale)
            err = np.abs(M[b, h].double().cpu().numpy() - Mo) / L[:, None]
            assert err.max() <= MASS_REL, f"b{b} h{h}: max |dM|/|qb| = {err.max():.3e}"
        # the selection on the same fp32 masses: bit-exact against the oracle's greedy
        keep, rec, nnz, _ = oracle.select_blocks(M[b].double().cpu().numpy(), blocks, "recall", targets,
                                                 text_sink=bool(flags & 1))
        for h in range(H):
            for p in range(nb):
                exp = np.nonzero(keep[h, p])[0].tolist()
                got = rows[(b * H + h) * nb + p]
                assert got == exp, f"b{b} h{h} row {p}: {got[:8]} vs {exp[:8]}"
        np.testing.assert_array_equal(out.head_nnz[b].cpu().numpy(), nnz)
        np.testing.assert_allclose(out.head_recall[b].cpu().numpy(), rec, rtol=1e-6)
    _row_order_ok(out, batch * H * nb)
    # identical to K3 on the same masses, and the dense pass / masses identical to the two-call path
    ref = ada.select_blocks(M, heads_desc=ada.make_desc(q, lay.block, lay.n_text, lay.text_first),
                            mode=ada.SELECT_RECALL, target=targets, flags=flags)
    o2, l2, M2 = ada.dense_attn_lse_search(q, k, v, heads_per_pass=heads_per_pass, **kw)
    torch.cuda.synchronize()
    _same_csr(out, ref)
    assert torch.equal(o, o2) and torch.equal(lse, l2) and torch.equal(M, M2)
    return o, lse, M, out


@pytest.mark.parametrize("name,over,targets", CASES)
def test_search_select_matches_oracle(ada, name, over, targets):
    lay = workloads.layout_for(name, **over)
    q, k, v = (x.cuda() for x in workloads.generate_qkv(lay))
    _check(ada, lay, q, k, v, targets)


def test_search_select_no_sink_batch2_passes_token_major(ada):
    """Without the text sink; batch 2; [B, N, H, d] storage; one head per pass gives the same bits as
    one pass; block_mass not requested (not written) gives the same CSR."""
    lay = workloads.layout_for("tiny", f=3, h=9, w=11, n_text=37, heads=3, head_dim=128, block=128)
    q, k, v = (x.cuda() for x in workloads.generate_qkv(lay, batch=2))
    qt, kt, vt = (x.transpose(1, 2).contiguous().transpose(1, 2) for x in (q, k, v))
    tg = [0.9, 0.75, 0.99]
    _, _, _, a = _check(ada, lay, qt, kt, vt, tg, flags=0, batch=2, heads_per_pass=1)
    _, _, _, b = _check(ada, lay, q, k, v, tg, flags=0, batch=2, heads_per_pass=0)
    _same_csr(a, b)
    kw = dict(block_size=lay.block, n_text=lay.n_text, text_first=lay.text_first)
    _, _, Mn, c = ada.search_select(q, k, v, target=tg, flags=0, want_block_mass=False, **kw)
    torch.cuda.synchronize()
    assert Mn is None
    _same_csr(b, c)


@pytest.mark.parametrize("nv,nt,B", [(139200, 320, 64), (70000, 77, 64)])
def test_search_select_large_nb(ada, nv, nt, B):
    """nb = 2182 (> 2048: the selection runs as K3's row kernel after the passes) and nb = 1095 (the
    fused epilogue at 35 masses per lane): identical to K3 on the masses the call wrote."""
    lay = workloads.layout_for("tiny", n_text=nt, heads=1, head_dim=64, block=B, f=1, h=1, w=nv)
    q, k, v = (x.cuda() for x in workloads.generate_qkv(lay))
    kw = dict(block_size=B, n_text=nt, text_first=False)
    o, lse, M, out = ada.search_select(q, k, v, target=[0.9], **kw)
    ref = ada.select_blocks(M, heads_desc=ada.make_desc(q, B, nt, False), mode=ada.SELECT_RECALL, target=[0.9])
    torch.cuda.synchronize()
    _same_csr(out, ref)
    # without a requested block_mass the binding still passes one when nb > 2048 (the C ABI requires it)
    _, _, Mx, out2 = ada.search_select(q, k, v, target=[0.9], want_block_mass=False, **kw)
    torch.cuda.synchronize()
    assert (Mx is not None) == (ada.num_blocks(ada.make_desc(q, B, nt, False)) > 2048)
    _same_csr(out, out2)
