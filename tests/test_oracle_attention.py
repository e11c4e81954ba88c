"""Pins for oracle.attention / oracle.blocks against things other than the
oracle itself: torch's SDPA (library routine), scipy's softmax/logsumexp,
closed forms, brute-force loops and paper-printed geometry."""

import json
import math
import os

import numpy as np
import pytest
import torch
from scipy.special import logsumexp, softmax

import oracle
from oracle import Block


def _rand(shape, seed, scale=1.0):
    return np.random.default_rng(seed).standard_normal(shape) * scale


def _sdpa_fp64(q, k, v, mask=None):
    tq, tk, tv = (torch.from_numpy(np.ascontiguousarray(x))[None, None] for x in (q, k, v))
    m = None if mask is None else torch.from_numpy(mask)[None, None]
    return torch.nn.functional.scaled_dot_product_attention(tq, tk, tv, attn_mask=m)[0, 0].numpy()


# ---------------------------------------------------------------- block map

def test_layout_geometry_golden(golden_dir):
    cases = json.load(open(os.path.join(golden_dir, "layouts.json")))["cases"]
    for c in cases:
        nv = c["f"] * c["h"] * c["w"]
        assert nv + c["t"] == c["L"]
        if "B" in c:
            for tf in (False, True):
                blocks = oracle.block_map(nv, c["t"], c["B"], tf)
                vids = [b for b in blocks if b.modality == "video"]
                txts = [b for b in blocks if b.modality == "text"]
                assert len(vids) == c["nb_video"] and len(txts) == c["nb_text"]
                assert vids[-1].length == c["video_tail"]
                assert oracle.num_blocks(nv, c["t"], c["B"]) == len(blocks)


@pytest.mark.parametrize("tf", [False, True])
def test_block_map_partitions_and_no_straddle(tf):
    nv, nt, B = 100, 37, 16
    blocks = oracle.block_map(nv, nt, B, tf)
    tok = oracle.token_block_of(blocks)
    assert len(tok) == nv + nt
    # contiguous cover in order
    pos = 0
    for b in blocks:
        assert b.start == pos and 1 <= b.length <= B
        pos += b.length
    # no block mixes modalities
    text_lo = 0 if tf else nv
    for b in blocks:
        is_text = [text_lo <= t < text_lo + nt for t in range(b.start, b.start + b.length)]
        assert all(is_text) or not any(is_text)
        assert (b.modality == "text") == is_text[0]


# ---------------------------------------------------------------- dense

@pytest.mark.parametrize("seed", range(4))
def test_dense_matches_torch_sdpa(seed):
    N, d = 97, 32
    q, k, v = (_rand((N, d), seed * 3 + i) for i in range(3))
    o, lse = oracle.dense_attention(q, k, v, 1.0 / math.sqrt(d))
    np.testing.assert_allclose(o, _sdpa_fp64(q, k, v), rtol=0, atol=1e-12)
    z = (q @ k.T) / math.sqrt(d)
    np.testing.assert_allclose(lse, logsumexp(z, axis=1), rtol=0, atol=1e-12)


def test_dense_special_cases():
    # L = 1: W = [[1]], O = V
    q, k, v = _rand((1, 8), 1), _rand((1, 8), 2), _rand((1, 8), 3)
    o, lse = oracle.dense_attention(q, k, v, 0.3)
    np.testing.assert_allclose(o, v, atol=1e-15)
    assert abs(lse[0] - 0.3 * float(q[0] @ k[0])) < 1e-12
    # Q = 0: uniform weights, O = column mean of V, lse = log N
    N = 50
    k, v = _rand((N, 8), 4), _rand((N, 8), 5)
    o, lse = oracle.dense_attention(np.zeros((3, 8)), k, v, 0.125)
    np.testing.assert_allclose(o, np.tile(v.mean(axis=0), (3, 1)), atol=1e-14)
    np.testing.assert_allclose(lse, np.log(N), atol=1e-14)
    # logits [1000, 1000]: lse = 1000 + ln 2, no overflow
    o, lse = oracle.dense_attention(np.array([[1000.0]]), np.array([[1.0], [1.0]]),
                                    np.array([[1.0], [3.0]]), 1.0)
    assert abs(lse[0] - (1000.0 + math.log(2.0))) < 1e-12
    assert abs(o[0, 0] - 2.0) < 1e-12


def test_dense_key_permutation_invariance():
    N, d = 40, 16
    q, k, v = (_rand((N, d), 10 + i) for i in range(3))
    perm = np.random.default_rng(0).permutation(N)
    o1, l1 = oracle.dense_attention(q, k, v, 0.25)
    o2, l2 = oracle.dense_attention(q, k[perm], v[perm], 0.25)
    np.testing.assert_allclose(o1, o2, atol=1e-13)
    np.testing.assert_allclose(l1, l2, atol=1e-13)


# ---------------------------------------------------------------- block mass

def _bruteforce_mass(q, k, lse, blocks, scale):
    """Nested loops: token -> block by walking the block list, weights by
    math.exp per element (SPEC.md:149 nested-loop oracle)."""
    tok = oracle.token_block_of(blocks)
    nb = len(blocks)
    M = [[0.0] * nb for _ in range(nb)]
    for i in range(q.shape[0]):
        for j in range(k.shape[0]):
            s = scale * sum(float(q[i, t]) * float(k[j, t]) for t in range(q.shape[1]))
            M[tok[i]][tok[j]] += math.exp(s - float(lse[i]))
    return np.array(M)


@pytest.mark.parametrize("tf", [False, True])
def test_block_mass_nested_loops(tf):
    # H=1, N=16 (+ partial blocks), B=4 -- SPEC.md:149
    nv, nt, B, d = 13, 5, 4, 8
    blocks = oracle.block_map(nv, nt, B, tf)
    q, k = _rand((nv + nt, d), 21), _rand((nv + nt, d), 22)
    scale = 1 / math.sqrt(d)
    lse = logsumexp(scale * q @ k.T, axis=1)
    M = oracle.block_mass(q, k, lse, blocks, scale)
    np.testing.assert_allclose(M, _bruteforce_mass(q, k, lse, blocks, scale), rtol=1e-12, atol=1e-14)


def test_block_mass_equals_softmax_block_sums_and_recall():
    """W_sum_attn = block sums of softmax(QK^T/sqrt(d)) from scipy,
    and block-level recall equals element-level Recall of the expanded mask
    (PAPER.md:230)."""
    nv, nt, B, d = 40, 9, 8, 16
    blocks = oracle.block_map(nv, nt, B, False)
    q, k, v = (_rand((nv + nt, d), 30 + i, 1.5) for i in range(3))
    scale = 1 / math.sqrt(d)
    W = softmax(scale * q @ k.T, axis=1)
    _, lse = oracle.dense_attention(q, k, v, scale)
    M = oracle.block_mass(q, k, lse, blocks, scale)
    tok = np.array(oracle.token_block_of(blocks))
    for p in range(len(blocks)):
        for j in range(len(blocks)):
            ref = W[np.ix_(tok == p, tok == j)].sum()
            assert abs(M[p, j] - ref) < 1e-13
    keep = M > np.median(M)
    el = oracle.expand_block_mask(keep, blocks)
    assert abs(W[el].sum() / W.sum() - M[keep].sum() / M.sum()) < 1e-13


def test_block_mass_rowsum_exact_lse():
    """Per-row block masses sum to |qb| under the exact LSE (north_star's oracle
    self-check: 'per-row block masses sum to 1' after dividing by |qb|)."""
    nv, nt, B, d = 70, 11, 16, 32
    blocks = oracle.block_map(nv, nt, B, True)
    q, k, v = (_rand((nv + nt, d), 40 + i, 2.0) for i in range(3))
    _, lse = oracle.dense_attention(q, k, v, 1 / math.sqrt(d))
    M = oracle.block_mass(q, k, lse, blocks, 1 / math.sqrt(d))
    np.testing.assert_allclose(M.sum(axis=1), [b.length for b in blocks], rtol=1e-12)


def test_block_mass_uniform_and_shift():
    nv, nt, B, d = 30, 10, 8, 8
    N = nv + nt
    blocks = oracle.block_map(nv, nt, B, False)
    k = _rand((N, d), 50)
    # uniform logits: M = |qb||kb|/N
    q0 = np.zeros((N, d))
    M = oracle.block_mass(q0, k, np.full(N, math.log(N)), blocks, 0.5)
    L = np.array([b.length for b in blocks], dtype=float)
    np.testing.assert_allclose(M, np.outer(L, L) / N, rtol=1e-13)
    # uniform LSE shift delta scales every mass by exp(-delta)
    q = _rand((N, d), 51)
    lse = logsumexp(0.5 * q @ k.T, axis=1)
    M1 = oracle.block_mass(q, k, lse, blocks, 0.5)
    M2 = oracle.block_mass(q, k, lse + 0.7, blocks, 0.5)
    np.testing.assert_allclose(M2, M1 * math.exp(-0.7), rtol=1e-13)


def test_block_mass_subset_rows():
    nv, nt, B, d = 50, 14, 8, 8
    blocks = oracle.block_map(nv, nt, B, False)
    q, k = _rand((nv + nt, d), 60), _rand((nv + nt, d), 61)
    lse = logsumexp(q @ k.T * 0.3, axis=1)
    full = oracle.block_mass(q, k, lse, blocks, 0.3)
    sub = oracle.block_mass(q, k, lse, blocks, 0.3, q_block_ids=[7, 2])
    np.testing.assert_array_equal(sub, full[[7, 2]])


# ---------------------------------------------------------------- masked attention

def test_masked_full_mask_is_dense():
    nv, nt, B, d = 45, 19, 16, 16
    blocks = oracle.block_map(nv, nt, B, False)
    q, k, v = (_rand((nv + nt, d), 70 + i) for i in range(3))
    nb = len(blocks)
    o, lse = oracle.masked_attention(q, k, v, blocks, [range(nb)] * nb, 0.25)
    od, ld = oracle.dense_attention(q, k, v, 0.25)
    np.testing.assert_allclose(o, od, atol=1e-12)
    np.testing.assert_allclose(lse, ld, atol=1e-12)


@pytest.mark.parametrize("seed", range(3))
def test_masked_matches_sdpa_with_large_bias(seed):
    """c = +inf exclusion vs SDPA with an additive -1e9 bias."""
    nv, nt, B, d = 40, 24, 8, 16
    blocks = oracle.block_map(nv, nt, B, seed % 2 == 1)
    nb = len(blocks)
    rng = np.random.default_rng(seed)
    keep = rng.random((nb, nb)) < 0.35
    keep[np.arange(nb), rng.integers(0, nb, nb)] = True
    q, k, v = (_rand((nv + nt, d), 80 + 3 * seed + i, 2.0) for i in range(3))
    scale = 1 / math.sqrt(d)
    o, lse = oracle.masked_attention(q, k, v, blocks, [np.nonzero(r)[0] for r in keep], scale)
    bias = np.where(oracle.expand_block_mask(keep, blocks), 0.0, -1e9)
    np.testing.assert_allclose(o, _sdpa_fp64(q, k, v, bias), atol=1e-12)
    z = scale * q @ k.T + bias
    np.testing.assert_allclose(lse, logsumexp(z, axis=1), atol=1e-10)


def test_masked_identity_and_locality():
    # B = 1 and each token keeps only its own block -> O = V
    N, d = 12, 4
    blocks = oracle.block_map(N, 0, 1, False)
    q, k, v = (_rand((N, d), 90 + i) for i in range(3))
    o, _ = oracle.masked_attention(q, k, v, blocks, [[i] for i in range(N)], 0.5)
    np.testing.assert_allclose(o, v, atol=1e-15)
    # block-diagonal mask: perturbing V outside the kept blocks leaves O unchanged
    blocks = oracle.block_map(32, 8, 8, False)
    q, k, v = (_rand((40, d), 95 + i) for i in range(3))
    kept = [[p] for p in range(len(blocks))]
    o1, _ = oracle.masked_attention(q, k, v, blocks, kept, 0.5, q_block_ids=[1])
    v2 = v.copy()
    v2[:8] += 10.0
    v2[16:] -= 3.0
    o2, _ = oracle.masked_attention(q, k, v2, blocks, kept, 0.5, q_block_ids=[1])
    np.testing.assert_array_equal(o1, o2)
