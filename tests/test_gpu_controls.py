"""Negative controls and invariances of the GPU path (the fault-injection control of
SPEC.md:547, the uniform-LSE-shift invariance of SPEC.md:289/322, reading R8 of DESIGN.md §3).

The controls show that the parity checks of tests/gpu_helpers.py are sharp enough to catch a
plausible kernel mistake: each injects one (a wrong softmax scale, a dropped kv block, swapped
masses) into an otherwise correct GPU run and asserts that the comparison with the oracle FAILS.
"""

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


def _lay():
    return workloads.layout_for("tiny", f=5, h=9, w=11, n_text=37, head_dim=128, block=128)


def _fails(fn):
    try:
        fn()
    except AssertionError:
        return True
    return False


def test_control_wrong_scale_is_caught(ada):
    """K1 run with softmax_scale 2% off 1/sqrt(d) must fail the O / LSE tolerances."""
    lay = _lay()
    q, k, v = (x.cuda() for x in workloads.generate_qkv(lay))
    scale = 1 / math.sqrt(lay.head_dim)
    o, lse = ada.dense_attn_lse(q, k, v, block_size=lay.block, n_text=lay.n_text, softmax_scale=scale * 1.02)
    torch.cuda.synchronize()
    ro, rl = oracle.dense_attention(np64(q[0, 0]), np64(k[0, 0]), np64(v[0, 0]), scale)
    assert _fails(lambda: compare_out(o[0, 0], ro, lse[0, 0], rl, what="wrong scale"))
    # and the unperturbed call passes the same check
    o, lse = ada.dense_attn_lse(q, k, v, block_size=lay.block, n_text=lay.n_text)
    torch.cuda.synchronize()
    compare_out(o[0, 0], ro, lse[0, 0], rl, what="correct scale")


def test_control_dropped_block_is_caught(ada):
    """K4 given a CSR with one kv block dropped from one row must fail against the oracle's masked
    attention over the full row (the q-block's rows change beyond tolerance)."""
    lay = _lay()
    q, k, v = (x.cuda() for x in workloads.generate_qkv(lay))
    blocks = oracle.block_map(lay.n_video, lay.n_text, lay.block, lay.text_first)
    nb = len(blocks)
    scale = 1 / math.sqrt(lay.head_dim)
    qh, kh, vh = np64(q[0, 0]), np64(k[0, 0]), np64(v[0, 0])
    od, lse = oracle.dense_attention(qh, kh, vh, scale)
    p = 1
    M = oracle.block_mass(qh, kh, lse, blocks, scale, q_block_ids=[p])[0]
    full = list(range(nb))
    heavy = int(np.argmax(M))  # drop the heaviest block: the largest effect a dropped entry can have
    rows = [full] * (lay.heads * nb)
    rows[p] = [j for j in full if j != heavy]
    rp = torch.tensor(np.cumsum([0] + [len(r) for r in rows]), dtype=torch.int32, device="cuda")
    ci = torch.tensor([j for r in rows for j in r], dtype=torch.int32, device="cuda")
    o, _ = ada.block_sparse_attn(q, k, v, rp, ci, block_size=lay.block, n_text=lay.n_text)
    torch.cuda.synchronize()
    b = blocks[p]
    r = slice(b.start, b.start + b.length)
    ref, _ = oracle.masked_attention(qh, kh, vh, blocks, {p: full}, scale, q_block_ids=[p])
    assert _fails(lambda: compare_out(o[0, 0, r], ref, what="dropped block"))
    b0 = blocks[0]
    compare_out(o[0, 0, b0.start:b0.start + b0.length], od[b0.start:b0.start + b0.length], what="intact row")


def test_control_swapped_masses_are_caught(ada):
    """K3 on masses where two entries of a row were swapped must disagree with the oracle's
    selection on the original masses (the exact-selection check is sharp)."""
    H, nv, nt, B = 2, 1000, 150, 64
    blocks = oracle.block_map(nv, nt, B, False)
    nb = len(blocks)
    Mt = workloads.random_masses(H * nb, nb, seed=21, ties=False).view(1, H, nb, nb)
    q = torch.empty(1, H, nv + nt, 64, dtype=torch.bfloat16, device="cuda")
    desc = ada.make_desc(q, B, nt, False)
    p = 3
    row = Mt[0, 0, p].double().numpy()
    forced, cands = oracle.row_forced_and_candidates(blocks, p, True)
    exp = oracle.select_row_recall(row, forced, cands, 0.9)
    kept_c = [j for j in exp if j in cands]
    dropped = [j for j in cands if j not in exp]
    assert kept_c and dropped
    bad = Mt.clone()
    a, z = kept_c[0], dropped[0]
    bad[0, 0, p, a], bad[0, 0, p, z] = Mt[0, 0, p, z], Mt[0, 0, p, a]
    out_bad = ada.select_blocks(bad.cuda(), heads_desc=desc, mode=ada.SELECT_RECALL, target=[0.9] * H)
    out_ok = ada.select_blocks(Mt.cuda(), heads_desc=desc, mode=ada.SELECT_RECALL, target=[0.9] * H)
    torch.cuda.synchronize()

    def row_of(out):
        rp = out.row_ptr.cpu().numpy()
        return out.col_idx.cpu().numpy()[rp[p]:rp[p + 1]].tolist()

    assert row_of(out_ok) == exp
    assert row_of(out_bad) != exp


def test_lse_shift_leaves_selection_unchanged(ada):
    """Reading R8: recall is measured against the row total T, so a uniform shift of the cached LSE
    (M -> M e^-delta) leaves the RECALL selection unchanged (up to the tie zone); the masses scale
    by e^-delta within K2's tolerance."""
    lay = _lay()
    q, k, v = (x.cuda() for x in workloads.generate_qkv(lay))
    kw = dict(block_size=lay.block, n_text=lay.n_text, text_first=lay.text_first)
    desc = ada.make_desc(q, lay.block, lay.n_text, lay.text_first)
    _, lse = ada.dense_attn_lse(q, k, v, **kw)
    M0 = ada.lse_cached_search(q, k, lse, **kw)
    delta = 0.75
    M1 = ada.lse_cached_search(q, k, lse + delta, **kw)
    s0 = ada.select_blocks(M0, heads_desc=desc, mode=ada.SELECT_RECALL, target=[0.9] * lay.heads)
    s1 = ada.select_blocks(M1, heads_desc=desc, mode=ada.SELECT_RECALL, target=[0.9] * lay.heads)
    torch.cuda.synchronize()
    ratio = (M1.double() / M0.double().clamp_min(1e-30))[M0 > 1e-20]
    assert torch.allclose(ratio, torch.full_like(ratio, math.exp(-delta)), rtol=2e-5)
    assert torch.equal(s0.row_ptr, s1.row_ptr) and torch.equal(s0.col_idx[:int(s0.row_ptr[-1])],
                                                               s1.col_idx[:int(s1.row_ptr[-1])])
