"""The fused search step t_w (adaspa_dense_attn_lse_search: Alg. 1 in one dense pass plus the
HBM-bound block-mass reduction) against the fp64 oracle: O and LSE as K1
(PAPER.md:166-202), block masses as W_sum_attn with the fresh LSE (reading R4),
on layouts spanning several tiles with ragged tails, both text orders, blocks 64/128, d 64/128,
batch 2, token-major strides, and head passes (a workspace smaller than the whole layer)."""

import math

import numpy as np
import pytest
import torch

import oracle
import workloads
from gpu_helpers import MASS_REL, compare_out, np64

pytestmark = pytest.mark.gpu

CASES = [
    ("tiny", {}),
    ("tiny_tf", {}),
    ("tiny", dict(f=5, h=9, w=11, n_text=37, head_dim=128, block=128)),      # 495 + 37 tokens
    ("tiny_tf", dict(f=3, h=10, w=13, n_text=77, head_dim=64, block=128)),   # text first, B=128, d=64
    ("tiny", dict(f=4, h=9, w=10, n_text=45, head_dim=128, block=64, heads=3)),
    ("tiny_tf", dict(f=6, h=10, w=21, n_text=77, head_dim=128, block=128, heads=3)),
    ("tiny_tf", dict(f=3, h=7, w=13, n_text=29, head_dim=64, block=64, heads=2)),  # odd nb at B=64
]


@pytest.fixture(scope="module")
def ada():
    import paper_2502_21079_b200 as m
    assert torch.cuda.is_available(), "gpu tests need a CUDA device"
    return m


def _check(ada, lay, q, k, v, batch=1, heads_per_pass=0):
    kw = dict(block_size=lay.block, n_text=lay.n_text, text_first=lay.text_first)
    o, lse, M = ada.dense_attn_lse_search(q, k, v, heads_per_pass=heads_per_pass, **kw)
    torch.cuda.synchronize()
    blocks = oracle.block_map(lay.n_video, lay.n_text, lay.block, lay.text_first)
    L = np.array([b.length for b in blocks], dtype=np.float64)
    scale = 1 / math.sqrt(lay.head_dim)
    worst = 0.0
    for b in range(batch):
        for h in range(lay.heads):
            qq, kk, vv = np64(q[b, h]), np64(k[b, h]), np64(v[b, h])
            ro, rl = oracle.dense_attention(qq, kk, vv, scale)
            compare_out(o[b, h], ro, lse[b, h], rl, what=f"{lay} b{b} h{h}")
            Mo = oracle.block_mass(qq, kk, lse[b, h].double().cpu().numpy(), blocks, scale)
            err = np.abs(M[b, h].double().cpu().numpy() - Mo) / L[:, None]
            worst = max(worst, err.max())
            assert err.max() <= MASS_REL, f"b{b} h{h}: max |dM|/|qb| = {err.max():.3e}"
            rows = M[b, h].double().cpu().numpy().sum(axis=1) / L                  # exact LSE: rows sum to |qb|
            assert np.abs(rows - 1.0).max() <= 1e-5
    return o, lse, M, worst


@pytest.mark.parametrize("name,over", CASES)
def test_fused_search_matches_oracle(ada, name, over):
    lay = workloads.layout_for(name, **over)
    q, k, v = (x.cuda() for x in workloads.generate_qkv(lay))
    o, lse, M, worst = _check(ada, lay, q, k, v)
    # same O / LSE bits as K1 alone (the fused pass walks the kv blocks of the grid instead of 128-row
    # tiles from token 0, so compare within tolerance, not bitwise)
    o1, l1 = ada.dense_attn_lse(q, k, v, block_size=lay.block, n_text=lay.n_text, text_first=lay.text_first)
    torch.cuda.synchronize()
    assert (o.float() - o1.float()).abs().max().item() <= 2e-2
    assert (lse - l1).abs().max().item() <= 1e-4
    print(f"{name} {over}: max |dM|/|qb| = {worst:.2e}")


def test_fused_search_head_passes_batch2_token_major(ada):
    """A workspace for one head per pass gives the same bits as one pass over all heads; batch 2 and
    [B, N, H, d] storage through the strides."""
    lay = workloads.layout_for("tiny", f=3, h=9, w=11, n_text=37, heads=3, head_dim=128, block=128)
    q, k, v = (x.cuda() for x in workloads.generate_qkv(lay, batch=2))
    qt, kt, vt = (x.transpose(1, 2).contiguous().transpose(1, 2) for x in (q, k, v))
    o_a, l_a, M_a, _ = _check(ada, lay, qt, kt, vt, batch=2, heads_per_pass=1)
    o_b, l_b, M_b, _ = _check(ada, lay, q, k, v, batch=2, heads_per_pass=0)
    assert torch.equal(M_a, M_b) and torch.equal(l_a, l_b) and torch.equal(o_a, o_b)


def test_fused_search_agrees_with_k2(ada):
    """The fused block masses equal K2's (two-pass Alg. 1) within twice the mass tolerance."""
    lay = workloads.layout_for("tiny_tf", f=4, h=10, w=21, n_text=77, head_dim=64, block=64, heads=2)
    q, k, v = (x.cuda() for x in workloads.generate_qkv(lay))
    kw = dict(block_size=lay.block, n_text=lay.n_text, text_first=lay.text_first)
    _, lse, M = ada.dense_attn_lse_search(q, k, v, **kw)
    M2 = ada.lse_cached_search(q, k, lse, **kw)
    torch.cuda.synchronize()
    blocks = oracle.block_map(lay.n_video, lay.n_text, lay.block, lay.text_first)
    L = torch.tensor([b.length for b in blocks], dtype=torch.float64, device="cuda")[:, None]
    assert ((M.double() - M2.double()).abs() / L).max().item() <= 2 * MASS_REL
