"""Pins for oracle.select / oracle.schedule: brute-force enumeration, paper
formulas and worked examples (tests/golden/*.json, each cited)."""

import itertools
import json
import math
import os

import numpy as np
import pytest

import oracle


def test_topk_2x2_golden(golden_dir):
    g = json.load(open(os.path.join(golden_dir, "topk_2x2.json")))
    S = np.array(g["scores"], dtype=float)
    kept = []
    for p in range(2):
        for j in oracle.select_row_sparsity(S[p], [], [0, 1], 1):
            kept.append([p, j])
    assert kept == g["row_wise_k1_keep"]
    # global top-2 by enumeration of all C(4,2) masks
    cells = [(p, j) for p in range(2) for j in range(2)]
    best = max(itertools.combinations(cells, 2), key=lambda c: sum(S[x] for x in c))
    assert [list(x) for x in best] == g["global_top2_keep"]


def test_recall_ge_boundary_pin():
    # R9: row [4,1], r=0.8 -> 0.8*5 = 4.0 exactly -> one block reaches it
    assert oracle.select_row_recall([4.0, 1.0], [], [0, 1], 0.8) == [0]
    assert oracle.select_row_recall([4.0, 1.0], [], [0, 1], 0.81) == [0, 1]


@pytest.mark.parametrize("seed", range(40))
def test_recall_greedy_is_minimal_bruteforce(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(2, 9))
    m = rng.exponential(size=n) ** rng.uniform(0.5, 4)
    if seed % 5 == 0:
        m[rng.integers(0, n)] = m[0]  # ties
    n_forced = int(rng.integers(0, 3)) if n > 3 else 0
    forced = sorted(rng.choice(n, n_forced, replace=False).tolist())
    cands = [j for j in range(n) if j not in forced]
    r = float(rng.uniform(0.05, 0.99))
    kept = oracle.select_row_recall(m, forced, cands, r)
    size, best = oracle.brute_force_min_set(m, forced, cands, r)
    chosen = [j for j in kept if j not in forced]
    T = math.fsum(m)
    if math.fsum(m[j] for j in forced) >= r * T:
        assert chosen == [] or (not forced and len(chosen) == 1)
    else:
        assert len(chosen) == size
        assert abs(math.fsum(m[j] for j in kept) - best) <= 1e-12 * T
        assert math.fsum(m[j] for j in kept) >= r * T * (1 - 1e-12)
    assert set(forced) <= set(kept)


def test_recall_monotone_and_full():
    rng = np.random.default_rng(7)
    m = rng.exponential(size=30)
    prev = 0
    for r in np.linspace(0.0, 1.0, 41):
        kept = oracle.select_row_recall(m, [], list(range(30)), float(r))
        assert len(kept) >= prev and len(kept) >= 1
        prev = len(kept)
    assert oracle.select_row_recall(m, [], list(range(30)), 1.0) == list(range(30))
    # r <= 0 with no forced set keeps exactly the top block (R25)
    assert oracle.select_row_recall(m, [], list(range(30)), 0.0) == [int(np.argmax(m))]


def test_sparsity_topk_optimal_enumeration():
    """the top-k set has the maximum mass over all k-subsets."""
    rng = np.random.default_rng(3)
    for _ in range(30):
        n = int(rng.integers(3, 8))
        m = np.round(rng.exponential(size=n), 1)  # rounding creates ties
        k = int(rng.integers(1, n + 1))
        kept = oracle.select_row_sparsity(m, [], list(range(n)), k)
        best = max(math.fsum(m[list(c)]) for c in itertools.combinations(range(n), k))
        assert len(kept) == k and abs(math.fsum(m[kept]) - best) < 1e-12
        # tie rule: among equal masses the lower index wins
        order = sorted(range(n), key=lambda j: (-m[j], j))
        assert kept == sorted(order[:k])


def test_k_from_sparsity():
    assert oracle.k_from_sparsity(0.8, 872) == 174
    assert oracle.k_from_sparsity(0.0, 10) == 10
    assert oracle.k_from_sparsity(0.99, 10) == 1
    # R11: (3*0.8-1)/2 is 0.7000000000000002 in fp64 and must round like 0.7
    s = (3 * 0.8 - 1) / 2
    assert s != 0.7
    assert oracle.k_from_sparsity(s, 5) == oracle.k_from_sparsity(0.7, 5) == 2


def test_tiers_golden(golden_dir):
    g = json.load(open(os.path.join(golden_dir, "tiers.json")))
    for c in g["tier_values"]:
        out = oracle.head_tiers([0.99, 0.1], c["s"], 0.8)
        assert abs(out[0] - c["raised"]) < 1e-12 and abs(out[1] - c["lowered"]) < 1e-12
    ex = g["h4_example"]
    out = oracle.head_tiers(ex["recalls"], ex["s"], ex["tau"])
    np.testing.assert_allclose(out, ex["expected"], atol=1e-12)
    assert abs(np.mean(out) - ex["s"]) < 1e-12  # mean sparsity preserved


def test_tiers_rules():
    # n capped at floor(H/2); strict '>' tau; ties by head index
    out = oracle.head_tiers([0.9, 0.9, 0.9], 0.8, 0.8)
    assert out == pytest.approx([0.9, 0.8, 0.7])
    out = oracle.head_tiers([0.8, 0.8], 0.8, 0.8)     # not > 0.8 -> n = 0
    assert out == pytest.approx([0.8, 0.8])
    with pytest.raises(ValueError):
        oracle.head_tiers([0.9, 0.1], 0.3, 0.8)


def _toy_masses(H, blocks, seed):
    rng = np.random.default_rng(seed)
    nb = len(blocks)
    return rng.exponential(size=(H, nb, nb)) ** rng.uniform(1, 3, size=(H, 1, 1))


@pytest.mark.parametrize("tf", [False, True])
def test_text_sink_and_row_wise(tf):
    blocks = oracle.block_map(56, 20, 8, tf)
    M = _toy_masses(3, blocks, 5)
    text = [j for j, b in enumerate(blocks) if b.modality == "text"]
    vid = [j for j, b in enumerate(blocks) if b.modality == "video"]
    keep, rec, nnz, _ = oracle.select_blocks(M, blocks, "sparsity", [0.5, 0.7, 0.9], text_sink=True)
    for h in range(3):
        for p, b in enumerate(blocks):
            assert keep[h, p, text].all()
            if b.modality == "text":
                assert keep[h, p].all()
            else:  # Row Wise: the same count of video blocks in every video row
                assert keep[h, p, vid].sum() == oracle.k_from_sparsity([0.5, 0.7, 0.9][h], len(vid))
    keep2, _, _, _ = oracle.select_blocks(M, blocks, "sparsity", [0.5] * 3, text_sink=False)
    assert (keep2.sum(axis=2) == oracle.k_from_sparsity(0.5, len(blocks))).all()


def test_select_recall_mode_meets_targets_and_head_recall():
    blocks = oracle.block_map(64, 16, 8, False)
    M = _toy_masses(2, blocks, 9)
    keep, rec, nnz, _ = oracle.select_blocks(M, blocks, "recall", [0.9, 0.6], text_sink=True)
    for h, r in enumerate([0.9, 0.6]):
        row_ok = (M[h] * keep[h]).sum(axis=1) >= r * M[h].sum(axis=1) * (1 - 1e-12)
        assert row_ok.all()
        assert abs(rec[h] - (M[h] * keep[h]).sum() / M[h].sum()) < 1e-12
        assert nnz[h] == keep[h].sum()


def test_select_tiers_end_to_end():
    blocks = oracle.block_map(64, 0, 8, False)
    M = _toy_masses(4, blocks, 11)
    M[0] = np.eye(len(blocks)) * 100 + 1e-3   # concentrated head -> high recall
    keep, rec, nnz, tg = oracle.select_blocks(M, blocks, "sparsity", [0.8] * 4, tiers=True)
    base, brec, _, _ = oracle.select_blocks(M, blocks, "sparsity", [0.8] * 4)
    expect = oracle.head_tiers(brec, 0.8, 0.8)
    assert tg == pytest.approx(expect)
    assert abs(np.mean(tg) - 0.8) < 1e-12


def test_csr_roundtrip():
    rng = np.random.default_rng(1)
    keep = rng.random((2, 5, 7)) < 0.4
    rp, ci = oracle.to_csr(keep.reshape(-1, 7))
    assert rp[-1] == keep.sum()
    back = np.zeros((10, 7), dtype=bool)
    for r in range(10):
        seg = ci[rp[r]:rp[r + 1]]
        assert (np.diff(seg) > 0).all()
        back[r, seg] = True
    np.testing.assert_array_equal(back, keep.reshape(-1, 7))


def test_schedule_golden(golden_dir):
    g = json.load(open(os.path.join(golden_dir, "schedule.json")))
    tr = oracle.schedule_trace(g["n_steps"], g["t_w"], g["key_steps"])
    runs = []
    for m in tr:
        if runs and runs[-1][0] == m:
            runs[-1][1] += 1
        else:
            runs.append([m, 1])
    assert runs == g["runs"]
    assert oracle.schedule_trace(20, 5, [5]).count("cached-search+sparse") == 0
    with pytest.raises(ValueError):
        oracle.schedule_trace(50, 10, [12, 30])


def test_head_recall_equals_token_level_recall():
    """Independent pin of the whole-matrix Recall (the share of the attention weight
    matrix A that the mask keeps): computed at TOKEN level from an explicit softmax matrix (torch,
    fp64) with the block mask expanded to tokens, it must equal what select_blocks reports from the
    block masses."""
    import torch
    rng = np.random.default_rng(5)
    nv, nt, B, d, H = 70, 13, 8, 16, 2
    blocks = oracle.block_map(nv, nt, B, False)
    N = nv + nt
    scale = 1 / math.sqrt(d)
    q = rng.standard_normal((H, N, d)) * 1.5
    k = rng.standard_normal((H, N, d)) * 1.5
    M = np.stack([oracle.block_mass(q[h], k[h], np.log(np.exp(scale * q[h] @ k[h].T).sum(axis=1)), blocks, scale)
                  for h in range(H)])
    keep, rec, _, _ = oracle.select_blocks(M, blocks, "recall", [0.7, 0.95], text_sink=True)
    for h in range(H):
        A = torch.softmax(torch.tensor(scale * q[h] @ k[h].T, dtype=torch.float64), dim=-1).numpy()
        tok = np.zeros((N, N), dtype=bool)
        for p, bp in enumerate(blocks):
            for j, bj in enumerate(blocks):
                if keep[h, p, j]:
                    tok[bp.start:bp.start + bp.length, bj.start:bj.start + bj.length] = True
        assert abs((A * tok).sum() / A.sum() - rec[h]) < 1e-12


def test_tiers_composition_hand_example():
    """The tiered selection worked by hand from PAPER.md:527-533 (readings R11, R16, R17) on two
    heads with one 4-block row each (no text):
      head 0 masses [0.75, 0.10, 0.10, 0.05], head 1 [0.25]*4, base sparsity s = 0.5;
      base k = floor(0.5*4 + 0.5 + 1e-9) = 2 -> Recall 0.85 (head 0) and 0.50 (head 1);
      n = min(#{R > 0.8} = 1, floor(2/2) = 1): head 0 -> (1+s)/2 = 0.75, head 1 -> (3s-1)/2 = 0.25;
      k = floor(0.25*4 + 0.5) = 1 (head 0 keeps block 0) and floor(0.75*4 + 0.5) = 3 (head 1 keeps
      blocks 0, 1, 2: equal masses, ids ascending, R10)."""
    blocks = oracle.block_map(4 * 8, 0, 8, False)
    M = np.array([[[0.75, 0.10, 0.10, 0.05]] * 4, [[0.25] * 4] * 4])
    keep, rec, nnz, tg = oracle.select_blocks(M, blocks, "sparsity", [0.5, 0.5], tiers=True)
    assert tg == pytest.approx([0.75, 0.25])
    for p in range(4):
        assert keep[0, p].tolist() == [True, False, False, False]
        assert keep[1, p].tolist() == [True, True, True, False]
    assert rec[0] == pytest.approx(0.75) and rec[1] == pytest.approx(0.75)
    assert nnz.tolist() == [4, 12]
