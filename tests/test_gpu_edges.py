"""Edge cases of the whole hot path (K1 -> K2 -> K3 -> K4 through HotPath) against the oracle:
sequences shorter than one tile, a single token, a one-row tail tile, no text tokens, text-only
sequences (every row is a text row: the sink keeps every block), batch 3, one head, and both
selection modes.  Every head of every batch element is checked end to end."""

import math

import numpy as np
import pytest
import torch

import oracle
import workloads
from gpu_helpers import MASS_REL, compare_out, csr_rows, np64, selection_ok, selection_ok_topk

pytestmark = pytest.mark.gpu

EDGES = [
    # (name, f, h, w, n_text, text_first, heads, d, block, batch)
    ("short", 1, 3, 9, 10, False, 2, 64, 64, 1),        # N = 37 < one tile
    ("single_token", 1, 1, 1, 0, False, 1, 128, 128, 1),  # N = 1
    ("one_row_tail", 1, 1, 129, 0, False, 2, 128, 128, 1),  # N = 129: a 1-row second tile, no text
    ("no_text_b64", 2, 5, 20, 0, True, 3, 64, 64, 3),    # no text tokens, batch 3
    ("text_only", 0, 1, 1, 200, True, 2, 64, 64, 1),     # every token is text
    ("one_head", 3, 7, 11, 19, False, 1, 128, 64, 2),
]


@pytest.fixture(scope="module")
def ada():
    import paper_2502_21079_b200 as m
    assert torch.cuda.is_available(), "gpu tests need a CUDA device"
    return m


@pytest.mark.parametrize("edge", EDGES, ids=[e[0] for e in EDGES])
@pytest.mark.parametrize("mode", ["recall", "sparsity"])
@pytest.mark.parametrize("fused", [True, False], ids=["fused", "twopass"])
def test_hot_path_edges(ada, edge, mode, fused):
    from paper_2502_21079_b200.hotpath import HotPath
    name, f, h, w, nt, tf, H, d, B, batch = edge
    lay = workloads.layout_for("tiny", f=f, h=h, w=w, n_text=nt, text_first=tf, heads=H, head_dim=d, block=B)
    q, k, v = (x.cuda() for x in workloads.generate_qkv(lay, batch=batch))
    kmode = ada.SELECT_RECALL if mode == "recall" else ada.SELECT_SPARSITY
    target = 0.9 if mode == "recall" else 0.5
    hp = HotPath(batch, H, lay.n, d, B, nt, tf, mode=kmode, targets=target)
    o = hp.run(q, k, v, fused=fused)
    torch.cuda.synchronize()
    blocks = oracle.block_map(lay.n_video, lay.n_text, B, tf)
    nb = len(blocks)
    assert nb == hp.nb
    scale = 1 / math.sqrt(d)
    rows = csr_rows(hp.csr.row_ptr, hp.csr.col_idx)
    n_video_blocks = sum(1 for bl in blocks if bl.modality == "video")
    L = np.array([bl.length for bl in blocks], dtype=np.float64)[:, None]
    for b in range(batch):
        for hh in range(H):
            qq, kk, vv = np64(q[b, hh]), np64(k[b, hh]), np64(v[b, hh])
            od, lse = oracle.dense_attention(qq, kk, vv, scale)
            compare_out(hp.o_dense[b, hh], od, hp.lse[b, hh], lse, what=f"{name} b{b} h{hh} K1")
            M = oracle.block_mass(qq, kk, hp.lse[b, hh].double().cpu().numpy(), blocks, scale)
            assert (np.abs(hp.mass[b, hh].double().cpu().numpy() - M) / L).max() <= MASS_REL, f"{name} K2"
            for p in range(nb):
                got = rows[(b * H + hh) * nb + p]
                forced, cands = oracle.row_forced_and_candidates(blocks, p, True)
                if mode == "recall":
                    exp = oracle.select_row_recall(M[p], forced, cands, target)
                    good, msg = selection_ok(M[p], forced, cands, target, got, exp)
                    assert good, f"{name} b{b} h{hh} row {p}: {msg}"
                else:
                    k_top = oracle.k_from_sparsity(target, n_video_blocks)
                    exp = oracle.select_row_sparsity(M[p], forced, cands, k_top)
                    good, msg = selection_ok_topk(M[p], forced, cands, k_top, got, exp)
                    assert good, f"{name} b{b} h{hh} row {p}: {msg}"
                assert got, "no row may be empty"
            kept = [rows[(b * H + hh) * nb + p] for p in range(nb)]
            so, _ = oracle.masked_attention(qq, kk, vv, blocks, kept, scale)
            compare_out(o[b, hh], so, what=f"{name} b{b} h{hh} K4")
