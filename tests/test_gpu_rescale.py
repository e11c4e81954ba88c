"""The rare O-rescale path of K1/K4 (the running max grows by more than 2^8 in log2 units after
the first kv tile) driven on purpose: keys whose logits grow along the sequence, so
every row's max keeps moving up across kv tiles (and, at d=64, the softmax's wait for the previous
PV before rescaling O is exercised).  Against the oracle, dense and block-sparse, d = 64 and 128."""

import math

import numpy as np
import pytest
import torch

import oracle
import workloads
from gpu_helpers import compare_out, np64

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ada():
    import paper_2502_21079_b200 as m
    assert torch.cuda.is_available(), "gpu tests need a CUDA device"
    return m


def _growing(lay, seed=3):
    """q . k / sqrt(d) ramps from ~0 to ~+60 along the kv axis (in natural-log units), i.e. the row
    max grows by ~8 log2 units every ~200 keys: several rescales per row."""
    g = torch.Generator().manual_seed(seed)
    H, N, d = lay.heads, lay.n, lay.head_dim
    u = torch.randn(H, 1, d, generator=g)
    u = u / u.norm(dim=-1, keepdim=True)
    q = (u * math.sqrt(d) * 1.0).expand(H, N, d) + 0.05 * torch.randn(H, N, d, generator=g)
    ramp = torch.linspace(0.0, 60.0, N).view(1, N, 1)
    k = u * ramp + 0.3 * torch.randn(H, N, d, generator=g)
    v = torch.randn(H, N, d, generator=g).clamp(-4, 4)
    return tuple(x.unsqueeze(0).to(torch.bfloat16).cuda() for x in (q, k, v))


@pytest.mark.parametrize("d,block", [(64, 64), (128, 128), (128, 64)])
def test_rescale_dense_and_sparse(ada, d, block):
    lay = workloads.layout_for("tiny", f=4, h=9, w=30, n_text=40, head_dim=d, block=block, heads=2)
    q, k, v = _growing(lay)
    kw = dict(block_size=lay.block, n_text=lay.n_text, text_first=lay.text_first)
    scale = 1 / math.sqrt(d)
    o, lse = ada.dense_attn_lse(q, k, v, **kw)
    blocks = oracle.block_map(lay.n_video, lay.n_text, lay.block, lay.text_first)
    nb = len(blocks)
    # sparse: every other kv block plus the last one (the largest logits), so rows see the max move
    rows = [sorted(set(range(0, nb, 2)) | {nb - 1, p}) for _ in range(lay.heads) for p in range(nb)]
    rp = torch.tensor(np.cumsum([0] + [len(r) for r in rows]), dtype=torch.int32, device="cuda")
    ci = torch.tensor([j for r in rows for j in r], dtype=torch.int32, device="cuda")
    os_, ls = ada.block_sparse_attn(q, k, v, rp, ci, want_lse=True, **kw)
    torch.cuda.synchronize()
    for h in range(lay.heads):
        qq, kk, vv = np64(q[0, h]), np64(k[0, h]), np64(v[0, h])
        ro, rl = oracle.dense_attention(qq, kk, vv, scale)
        z = (qq @ kk.T) * scale
        # the workload really moves each row's max by many 2^8 steps after the first kv tile
        assert (z.max(axis=1) - z[:, :128].max(axis=1)).min() > 30.0
        compare_out(o[0, h], ro, lse[0, h], rl, what=f"dense d{d} B{block} h{h}")
        so, sl = oracle.masked_attention(qq, kk, vv, blocks, rows[h * nb:(h + 1) * nb], scale)
        compare_out(os_[0, h], so, ls[0, h], sl, what=f"sparse d{d} B{block} h{h}")


@pytest.mark.parametrize("d,block", [(64, 64), (128, 128), (128, 64)])
def test_rescale_fused_search_step(ada, d, block):
    """The fused search step t_w (adaspa_search_select) on the same ramped logits: every row's max moves
    up by many 2^8 steps, so the block log-sum-exps are written under several running maxima (the
    pass keeps them relative to the row's first max).  O / LSE against the oracle; block masses against
    W_sum_attn with the GPU's LSE; the selection bit-exact against the oracle's
    greedy on the GPU's masses."""
    from gpu_helpers import MASS_REL, csr_rows
    lay = workloads.layout_for("tiny", f=4, h=9, w=30, n_text=40, head_dim=d, block=block, heads=2)
    q, k, v = _growing(lay)
    kw = dict(block_size=lay.block, n_text=lay.n_text, text_first=lay.text_first)
    scale = 1 / math.sqrt(d)
    o, lse, M, out = ada.search_select(q, k, v, target=[0.9, 0.6], **kw)
    torch.cuda.synchronize()
    blocks = oracle.block_map(lay.n_video, lay.n_text, lay.block, lay.text_first)
    nb = len(blocks)
    L = np.array([b.length for b in blocks], dtype=np.float64)
    rows = csr_rows(out.row_ptr, out.col_idx)
    keep, _, _, _ = oracle.select_blocks(M[0].double().cpu().numpy(), blocks, "recall", [0.9, 0.6])
    for h in range(lay.heads):
        qq, kk, vv = np64(q[0, h]), np64(k[0, h]), np64(v[0, h])
        ro, rl = oracle.dense_attention(qq, kk, vv, scale)
        compare_out(o[0, h], ro, lse[0, h], rl, what=f"fused d{d} B{block} h{h}")
        Mo = oracle.block_mass(qq, kk, lse[0, h].double().cpu().numpy(), blocks, scale)
        err = np.abs(M[0, h].double().cpu().numpy() - Mo) / L[:, None]
        # MASS_REL's derivation (gpu_helpers) holds for |S_scaled| <= 32; its leading term grows with
        # the logit magnitude, which reaches ~60 nats here.  The fused pass adds one more term: a block
        # log-sum-exp and the row LSE are stored relative to the row's FIRST running max, and the row max
        # moves up by ~smax here, so each is a log2 value of magnitude ~smax/ln2 rounded to fp32
        # (absolute error <= smax/ln2 * 2^-24, i.e. a relative error <= smax * 2^-24 of 2^value), two
        # of them per mass term
        smax = np.abs(scale * qq @ kk.T).max()
        tol = MASS_REL * max(1.0, smax / 32.0) + 2.0 * smax * 2.0 ** -24
        assert err.max() <= tol, f"h{h}: max |dM|/|qb| = {err.max():.3e} > {tol:.3e} (|S| <= {smax:.1f})"
        for p in range(nb):
            assert rows[h * nb + p] == np.nonzero(keep[h, p])[0].tolist(), f"h{h} row {p}"
