"""K1/K4 exactness for ANY logit range (PAPER.md:194-202 online softmax; 415-427 with c = +inf):
masked columns must never enter the running max.  Masked columns are

  * the TMA zero fill past the sequence end in the last dense kv tile (logit 0),
  * the excluded half of a B=64 paired kv tile (a block another q-block of the item keeps),
  * the neighbour tokens loaded behind a partial block (the 128-row tile of a partial block).

Each case puts the kept logits ~100 nats BELOW the masked ones; with the masked columns in the max,
exp(kept - max) underflows and O = 0 / LSE = -inf.  Compared with the fp64 oracle (O max-abs 2e-2,
mean-abs 2e-3, LSE 1e-3).  Also: a caller CSR with an empty row gives O = 0 and LSE = -inf (the
C-ABI's in-band contract for data-dependent errors, include/adaspa.h)."""

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


def _unit(d, g):
    u = torch.randn(d, generator=g, dtype=torch.float64)
    return u / u.norm()


def _bf(x):
    return x.to(torch.bfloat16).unsqueeze(0).cuda()


def _csr(rows):
    rp = torch.tensor(np.cumsum([0] + [len(r) for r in rows]), dtype=torch.int32, device="cuda")
    ci = torch.tensor([j for r in rows for j in r] or [0], dtype=torch.int32, device="cuda")
    return rp, ci


@pytest.mark.parametrize("d", [64, 128])
@pytest.mark.parametrize("n", [37, 200])
def test_dense_all_logits_far_below_zero(ada, d, n):
    """Every logit ~ -100 nats (spread of a few nats); N % 128 != 0, so the last kv tile is zero
    filled by TMA (logit exactly 0 on those columns)."""
    g = torch.Generator().manual_seed(11 + n + d)
    H = 2
    u = torch.stack([_unit(d, g) for _ in range(H)])[:, None, :]           # [H, 1, d]
    a = math.sqrt(100.0 * math.sqrt(d))                                   # a*a/sqrt(d) = 100
    q = a * u + 0.5 * torch.randn(H, n, d, generator=g, dtype=torch.float64)
    k = -a * u + 0.5 * torch.randn(H, n, d, generator=g, dtype=torch.float64)
    v = torch.randn(H, n, d, generator=g, dtype=torch.float64).clamp(-4, 4)
    q, k, v = _bf(q), _bf(k), _bf(v)
    block = 64 if d == 64 else 128
    o, lse = ada.dense_attn_lse(q, k, v, block_size=block, n_text=0)
    torch.cuda.synchronize()
    scale = 1 / math.sqrt(d)
    for h in range(H):
        qq, kk, vv = np64(q[0, h]), np64(k[0, h]), np64(v[0, h])
        z = scale * qq @ kk.T
        assert z.max() < -80.0, z.max()
        ro, rl = oracle.dense_attention(qq, kk, vv, scale)
        compare_out(o[0, h], ro, lse[0, h], rl, what=f"dense N={n} d={d} h{h}")
    # the fused search step on the same inputs: O / LSE as K1, and the block masses of every row sum to
    # the q-block's token count under its exact LSE, however far below zero the logits
    o2, l2, M, _ = ada.search_select(q, k, v, block_size=block, n_text=0, target=[0.9] * H)
    torch.cuda.synchronize()
    blocks = oracle.block_map(n, 0, block, False)
    L = np.array([b.length for b in blocks], dtype=np.float64)
    for h in range(H):
        qq, kk, vv = np64(q[0, h]), np64(k[0, h]), np64(v[0, h])
        ro, rl = oracle.dense_attention(qq, kk, vv, scale)
        compare_out(o2[0, h], ro, l2[0, h], rl, what=f"fused N={n} d={d} h{h}")
        rows = M[0, h].double().cpu().numpy().sum(axis=1) / L
        assert np.isfinite(rows).all() and np.abs(rows - 1.0).max() <= 1e-5, rows


@pytest.mark.parametrize("d", [64, 128])
def test_sparse_b64_excluded_paired_block_dominates(ada, d):
    """B=64: q-block 0 keeps only kv block 0; every other kv block carries logits ~ +100 nats for
    q-block 0's rows.  The item's other q-blocks keep other blocks, so the kv stream pairs block 0
    with an excluded block in one 128-row tile (masked half for q-block 0)."""
    g = torch.Generator().manual_seed(5 + d)
    H, nblk = 2, 6
    n = 64 * nblk
    lay = workloads.layout_for("tiny", f=1, h=nblk, w=64, n_text=0, heads=H, head_dim=d, block=64)
    assert lay.n == n
    u = torch.stack([_unit(d, g) for _ in range(H)])[:, None, :]
    a = math.sqrt(100.0 * math.sqrt(d))
    q = torch.randn(H, n, d, generator=g, dtype=torch.float64)
    k = torch.randn(H, n, d, generator=g, dtype=torch.float64)
    q[:, :64] = a * u + 0.3 * torch.randn(H, 64, d, generator=g, dtype=torch.float64)
    k[:, 64:] = a * u + 0.3 * torch.randn(H, n - 64, d, generator=g, dtype=torch.float64)
    v = torch.randn(H, n, d, generator=g, dtype=torch.float64).clamp(-4, 4)
    q, k, v = _bf(q), _bf(k), _bf(v)
    per_head = [[0], [1], [2, 4], [3], [4], [5, 0]]
    rows = per_head * H
    rp, ci = _csr(rows)
    o, lse = ada.block_sparse_attn(q, k, v, rp, ci, block_size=64, n_text=0, want_lse=True)
    torch.cuda.synchronize()
    blocks = oracle.block_map(lay.n_video, lay.n_text, 64, lay.text_first)
    scale = 1 / math.sqrt(d)
    for h in range(H):
        qq, kk, vv = np64(q[0, h]), np64(k[0, h]), np64(v[0, h])
        z = scale * qq[:64] @ kk.T
        assert z[:, 64:].min() > z[:, :64].max() + 60.0      # the masked columns dominate by > 60 nats
        so, sl = oracle.masked_attention(qq, kk, vv, blocks, per_head, scale)
        compare_out(o[0, h], so, lse[0, h], sl, what=f"B64 paired d={d} h{h}")


@pytest.mark.parametrize("d,block", [(64, 64), (128, 128), (128, 64)])
def test_sparse_partial_block_neighbours_dominate(ada, d, block):
    """Text last, text sink off: the video tail block is partial, so its kv tile also loads the first
    text tokens behind it.  Text keys carry logits ~ +100 nats for every query; rows keep video
    blocks only (no text block), so the loaded text neighbours are masked columns."""
    g = torch.Generator().manual_seed(21 + d + block)
    H = 2
    n_video = 2 * block + 40
    n_text = 30
    lay = workloads.layout_for("tiny", f=1, h=1, w=n_video, n_text=n_text, text_first=False, heads=H,
                               head_dim=d, block=block)
    n = lay.n
    u = torch.stack([_unit(d, g) for _ in range(H)])[:, None, :]
    a = math.sqrt(100.0 * math.sqrt(d))
    q = a * u + 0.3 * torch.randn(H, n, d, generator=g, dtype=torch.float64)
    k = torch.randn(H, n, d, generator=g, dtype=torch.float64)
    k[:, n_video:] = a * u + 0.3 * torch.randn(H, n_text, d, generator=g, dtype=torch.float64)
    v = torch.randn(H, n, d, generator=g, dtype=torch.float64).clamp(-4, 4)
    q, k, v = _bf(q), _bf(k), _bf(v)
    blocks = oracle.block_map(lay.n_video, lay.n_text, block, False)
    nb = len(blocks)
    tail = max(i for i, b in enumerate(blocks) if b.modality == "video")
    assert blocks[tail].length == 40
    per_head = [[tail] if p % 2 == 0 else [0, tail] for p in range(nb)]
    rp, ci = _csr(per_head * H)
    o, lse = ada.block_sparse_attn(q, k, v, rp, ci, block_size=block, n_text=n_text, want_lse=True)
    torch.cuda.synchronize()
    scale = 1 / math.sqrt(d)
    for h in range(H):
        qq, kk, vv = np64(q[0, h]), np64(k[0, h]), np64(v[0, h])
        z = scale * qq @ kk.T
        assert z[:, n_video:].min() > z[:, :n_video].max() + 40.0
        so, sl = oracle.masked_attention(qq, kk, vv, blocks, per_head, scale)
        compare_out(o[0, h], so, lse[0, h], sl, what=f"partial tail d={d} B={block} h{h}")


@pytest.mark.parametrize("block", [64, 128])
def test_sparse_empty_rows(ada, block):
    """A caller CSR with empty rows (K3 never produces one): those rows get O = 0 and LSE = -inf;
    the other rows match the oracle.  Covers a whole item with no entries and a tile of which one
    q-block is empty."""
    lay = workloads.layout_for("tiny", head_dim=64, block=block, heads=2)
    q, k, v = (x.cuda() for x in workloads.generate_qkv(lay))
    blocks = oracle.block_map(lay.n_video, lay.n_text, block, lay.text_first)
    nb = len(blocks)
    empty = {0, 1, nb - 2} if block == 128 else {0, 1, 2, 3, 5}
    per_head = [[] if p in empty else [p, (p + 1) % nb] for p in range(nb)]
    rp, ci = _csr(per_head * lay.heads)
    o = torch.full_like(q, 7.0)
    o, lse = ada.block_sparse_attn(q, k, v, rp, ci, block_size=block, n_text=lay.n_text, o=o, want_lse=True)
    torch.cuda.synchronize()
    scale = 1 / math.sqrt(64)
    for h in range(lay.heads):
        qq, kk, vv = np64(q[0, h]), np64(k[0, h]), np64(v[0, h])
        for p in range(nb):
            bp = blocks[p]
            sl = slice(bp.start, bp.start + bp.length)
            if p in empty:
                assert torch.all(o[0, h, sl] == 0), f"row {p}: O not zero"
                assert torch.all(torch.isneginf(lse[0, h, sl])), f"row {p}: LSE not -inf"
            else:
                so, sll = oracle.masked_attention(qq, kk, vv, blocks, per_head, scale, q_block_ids=[p])
                compare_out(o[0, h, sl], so, lse[0, h, sl], sll, what=f"B={block} h{h} row {p}")
