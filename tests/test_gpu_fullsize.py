"""Full-size parity at the BASELINE.json configurations, in the launch configuration bench.py
times (HotPath: K1 -> K2 -> K3 -> K4 on one seeded layer): sampled q-blocks of sampled heads are
recomputed one by one by the fp64 oracle (DESIGN.md §4 tolerances).  The samples cover the first
and last video blocks (the ragged video tail), every text block, and seeded random blocks, on the
densest, the sparsest and a seeded random head."""

import math

import numpy as np
import pytest
import torch

import oracle
import workloads
from gpu_helpers import MASS_REL, compare_out, np64, selection_ok

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ada():
    import paper_2502_21079_b200 as m
    assert torch.cuda.is_available(), "gpu tests need a CUDA device"
    return m


def _sample_blocks(blocks, rng, n_random=2):
    video = [i for i, b in enumerate(blocks) if b.modality == "video"]
    text = [i for i, b in enumerate(blocks) if b.modality == "text"]
    pick = {video[0], video[-1], *text}
    pick.update(int(x) for x in rng.choice(video, size=n_random, replace=False))
    return sorted(pick)


@pytest.mark.parametrize("name", ["hyv110k", "cogx45k"])
def test_fullsize_hot_path_sampled(ada, name):
    from paper_2502_21079_b200.hotpath import HotPath
    lay = workloads.layout_for(name)
    q, k, v = workloads.generate_qkv(lay, device="cuda")
    hp = HotPath(1, lay.heads, lay.n, lay.head_dim, lay.block, lay.n_text, lay.text_first,
                 mode=ada.SELECT_RECALL, targets=0.9, flags=ada.FLAG_TEXT_SINK)
    o = hp.run(q, k, v)
    # the search step's fused selection epilogue == K3 on the masses it wrote, whole layer, bit for bit
    ref = ada.select_blocks(hp.mass, heads_desc=hp.desc, mode=ada.SELECT_RECALL, target=[0.9] * lay.heads,
                            flags=ada.FLAG_TEXT_SINK)
    torch.cuda.synchronize()
    assert torch.equal(ref.row_ptr, hp.csr.row_ptr)
    assert torch.equal(ref.col_idx[:int(ref.row_ptr[-1])], hp.csr.col_idx[:int(ref.row_ptr[-1])])
    assert torch.equal(ref.head_recall, hp.csr.head_recall)
    blocks = oracle.block_map(lay.n_video, lay.n_text, lay.block, lay.text_first)
    nb = len(blocks)
    assert nb == hp.nb
    scale = 1.0 / math.sqrt(lay.head_dim)
    nnz = hp.csr.head_nnz[0].cpu().numpy()
    rng = np.random.default_rng(7)
    heads = sorted({int(np.argmax(nnz)), int(np.argmin(nnz)), int(rng.integers(lay.heads))})
    rp = hp.csr.row_ptr.cpu().numpy()
    ci = hp.csr.col_idx.cpu().numpy()
    for h in heads:
        qh, kh, vh = np64(q[0, h]), np64(k[0, h]), np64(v[0, h])
        lse_g = hp.lse[0, h].double().cpu().numpy()
        for p in _sample_blocks(blocks, rng):
            b = blocks[p]
            rows = slice(b.start, b.start + b.length)
            od, lse = oracle.dense_attention(qh[rows], kh, vh, scale)                    # a1
            compare_out(hp.o_dense[0, h, rows], od, hp.lse[0, h, rows], lse, what=f"{name} K1 h{h} qb{p}")
            lse_full = np.zeros(lay.n)
            lse_full[rows] = lse
            M = oracle.block_mass(qh, kh, lse_full, blocks, scale, q_block_ids=[p])[0]  # a2
            Mg = hp.mass[0, h, p].double().cpu().numpy()
            err = np.abs(Mg - M).max() / b.length
            # K2 ran on the GPU's LSE: the LSE difference adds |dLSE| relative error per row
            tol = MASS_REL + np.abs(lse_g[rows] - lse).max()
            assert err <= tol, f"{name} K2 h{h} qb{p}: |dM|/|qb| {err:.3e} > {tol:.3e}"
            forced, cands = oracle.row_forced_and_candidates(blocks, p, True)           # a3
            ok_sel = oracle.select_row_recall(M, forced, cands, 0.9)
            row = (0 * lay.heads + h) * nb + p
            g_sel = ci[rp[row]:rp[row + 1]].tolist()
            good, msg = selection_ok(M, forced, cands, 0.9, g_sel, ok_sel)
            assert good, f"{name} K3 h{h} qb{p}: {msg}"
            so, _ = oracle.masked_attention(qh, kh, vh, blocks, {p: g_sel}, scale, q_block_ids=[p])  # a4
            compare_out(o[0, h, rows], so, what=f"{name} K4 h{h} qb{p}")


@pytest.mark.parametrize("name", ["cogx45k", "hyv110k"])
def test_fullsize_sparsity_tiers(ada, name):
    """The paper's default selection at full size: SPARSITY 0.8 with
    head-adaptive tiers and the text sink.  K3 on the GPU's block masses equals the oracle's selection
    on the same masses for EVERY row (tiers need every row: head Recall over the whole matrix, then
    n = min(#{R_h > 0.8}, H/2) heads raised / lowered); the per-head kept counts and Recalls agree;
    sampled rows are also checked against the oracle's OWN masses (sparsity tie-zone rule)."""
    from gpu_helpers import selection_ok_topk
    from paper_2502_21079_b200.hotpath import HotPath
    lay = workloads.layout_for(name)
    q, k, v = workloads.generate_qkv(lay, device="cuda")
    hp = HotPath(1, lay.heads, lay.n, lay.head_dim, lay.block, lay.n_text, lay.text_first,
                 mode=ada.SELECT_SPARSITY, targets=0.8, flags=ada.FLAG_TEXT_SINK | ada.FLAG_HEAD_TIERS)
    hp.search(q, k, v)
    torch.cuda.synchronize()
    blocks = oracle.block_map(lay.n_video, lay.n_text, lay.block, lay.text_first)
    nb = len(blocks)
    H = lay.heads
    Mg = hp.mass[0].double().cpu().numpy()
    keep, rec, nnz, s_h = oracle.select_blocks(Mg, blocks, "sparsity", [0.8] * H, text_sink=True, tiers=True)
    assert sorted(set(np.round(s_h, 12))) != [0.8], "no head was re-tiered"
    rp = hp.csr.row_ptr.cpu().numpy()
    ci = hp.csr.col_idx.cpu().numpy()
    for h in range(H):
        for p in range(nb):
            row = h * nb + p
            assert ci[rp[row]:rp[row + 1]].tolist() == np.nonzero(keep[h, p])[0].tolist(), (name, h, p)
    np.testing.assert_array_equal(hp.csr.head_nnz[0].cpu().numpy(), nnz)
    np.testing.assert_allclose(hp.csr.head_recall[0].cpu().numpy(), rec, rtol=1e-6)
    # sampled rows against the oracle's own masses
    scale = 1.0 / math.sqrt(lay.head_dim)
    rng = np.random.default_rng(11)
    n_cand = sum(1 for b in blocks if b.modality == "video")
    for h in sorted({int(np.argmax(s_h)), int(np.argmin(s_h))}):
        qh, kh = np64(q[0, h]), np64(k[0, h])
        for p in _sample_blocks(blocks, rng, n_random=1):
            b = blocks[p]
            rows = slice(b.start, b.start + b.length)
            _, lse = oracle.dense_attention(qh[rows], kh, np64(v[0, h]), scale)
            lse_full = np.zeros(lay.n)
            lse_full[rows] = lse
            M = oracle.block_mass(qh, kh, lse_full, blocks, scale, q_block_ids=[p])[0]
            forced, cands = oracle.row_forced_and_candidates(blocks, p, True)
            kk = oracle.k_from_sparsity(s_h[h], n_cand)
            exp = oracle.select_row_sparsity(M, forced, cands, kk)
            row = h * nb + p
            good, msg = selection_ok_topk(M, forced, cands, kk, ci[rp[row]:rp[row + 1]].tolist(), exp)
            assert good, f"{name} h{h} qb{p} (s={s_h[h]}): {msg}"
