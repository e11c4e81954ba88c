"""GPU parity of the four C-ABI calls against the fp64 oracle on seeded inputs
(small sizes that still span several tiles plus ragged tails).  Run on a B200:
    python -m pytest tests -m gpu -x -q
"""

import math

import numpy as np
import pytest
import torch

import oracle
import workloads
from gpu_helpers import (MASS_REL, O_MAX_ABS, compare_out, csr_rows, np64, selection_ok)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ada():
    import paper_2502_21079_b200.build as b
    b.build()
    import paper_2502_21079_b200 as m
    assert torch.cuda.is_available(), "gpu tests need a CUDA device"
    return m


def _qkv(lay, seed=workloads.synth.BASE_SEED, heads=None, batch=1):
    q, k, v = workloads.generate_qkv(lay, batch=batch, seed=seed, heads=heads)
    return q.cuda(), k.cuda(), v.cuda()


CASES = [
    # name, overrides (layouts chosen to span several 128-row tiles with ragged tails)
    ("tiny", {}),
    ("tiny_tf", {}),
    ("tiny", dict(f=5, h=9, w=11, n_text=37, head_dim=128, block=128)),      # 495 + 37 tokens, d=128
    ("tiny_tf", dict(f=3, h=10, w=13, n_text=77, head_dim=64, block=128)),   # text first, B=128
    ("tiny", dict(f=4, h=9, w=10, n_text=45, head_dim=128, block=64, heads=3)),
    # d=128 at block 128 runs on the CTA pair: several 512-row items per head, ragged last item
    ("tiny_tf", dict(f=6, h=10, w=21, n_text=77, head_dim=128, block=128, heads=3)),  # 77 + 1260 tokens
]


def _lay(name, over):
    return workloads.layout_for(name, **over)


@pytest.mark.parametrize("name,over", CASES)
def test_dense_attn_lse(ada, name, over):
    lay = _lay(name, over)
    q, k, v = _qkv(lay)
    o, lse = ada.dense_attn_lse(q, k, v, block_size=lay.block, n_text=lay.n_text, text_first=lay.text_first)
    torch.cuda.synchronize()
    scale = 1 / math.sqrt(lay.head_dim)
    for h in range(lay.heads):
        ro, rl = oracle.dense_attention(np64(q[0, h]), np64(k[0, h]), np64(v[0, h]), scale)
        compare_out(o[0, h], ro, lse[0, h], rl, what=f"{name} h{h}")


def test_dense_token_major_layout(ada):
    """[B, N, H, d] storage (Ulysses layout) through the stride arguments."""
    lay = _lay("tiny", dict(heads=3, head_dim=128, block=128))
    q, k, v = _qkv(lay, batch=2)
    qt, kt, vt = (x.transpose(1, 2).contiguous().transpose(1, 2) for x in (q, k, v))
    assert qt.stride(2) == 3 * 128
    o, lse = ada.dense_attn_lse(qt, kt, vt, block_size=128, n_text=lay.n_text)
    o2, lse2 = ada.dense_attn_lse(q, k, v, block_size=128, n_text=lay.n_text)
    torch.cuda.synchronize()
    assert torch.equal(o, o2) and torch.equal(lse, lse2)
    ro, rl = oracle.dense_attention(np64(q[1, 2]), np64(k[1, 2]), np64(v[1, 2]), 1 / math.sqrt(128))
    compare_out(o[1, 2], ro, lse[1, 2], rl, what="token-major b1 h2")


@pytest.mark.parametrize("name,over", CASES)
def test_search_block_mass(ada, name, over):
    """K2 with the oracle's exact LSE as the cached LSE: masses vs the explicit fp64 matrix,
    and row sums = |q-block|."""
    lay = _lay(name, over)
    q, k, v = _qkv(lay)
    scale = 1 / math.sqrt(lay.head_dim)
    blocks = oracle.block_map(lay.n_video, lay.n_text, lay.block, lay.text_first)
    lse_ref = []
    for h in range(lay.heads):
        _, rl = oracle.dense_attention(np64(q[0, h]), np64(k[0, h]), np64(v[0, h]), scale)
        lse_ref.append(rl)
    lse_t = torch.tensor(np.stack(lse_ref)[None], dtype=torch.float32, device="cuda")
    M = ada.lse_cached_search(q, k, lse_t, block_size=lay.block, n_text=lay.n_text, text_first=lay.text_first)
    torch.cuda.synchronize()
    L = np.array([b.length for b in blocks], dtype=np.float64)
    for h in range(lay.heads):
        # the oracle takes the same fp32 LSE the kernel reads
        Mo = oracle.block_mass(np64(q[0, h]), np64(k[0, h]), lse_t[0, h].double().cpu().numpy(), blocks, scale)
        err = np.abs(M[0, h].double().cpu().numpy() - Mo) / L[:, None]
        assert err.max() <= MASS_REL, f"{name} h{h}: max |dM|/|qb| = {err.max():.3e}"
        rs = M[0, h].double().cpu().numpy().sum(axis=1) / L
        assert np.abs(rs - Mo.sum(axis=1) / L).max() <= 1e-5


@pytest.mark.parametrize("tf", [False, True])
@pytest.mark.parametrize("mode", ["recall", "sparsity", "tiers", "nosink"])
def test_select_blocks_exact(ada, tf, mode):
    """K3 alone: identical fp32 masses on both sides -> identical CSR (bit-exact)."""
    H, nv, nt, B = 6, 1000, 150, 64
    blocks = oracle.block_map(nv, nt, B, tf)
    nb = len(blocks)
    Mt = workloads.random_masses(H * nb, nb, seed=7 + tf).view(1, H, nb, nb)
    q = torch.empty(1, H, nv + nt, 64, dtype=torch.bfloat16, device="cuda")
    desc = ada.make_desc(q, B, nt, tf)
    sink = mode != "nosink"
    if mode in ("recall", "nosink"):
        targets = [0.5, 0.8, 0.9, 0.95, 0.99, 1.0]
        kmode, flags = ada.SELECT_RECALL, (1 if sink else 0)
    elif mode == "sparsity":
        targets = [0.0, 0.5, 0.7, 0.8, 0.9, 0.95]
        kmode, flags = ada.SELECT_SPARSITY, 1
    else:
        targets = [0.8] * H
        kmode, flags = ada.SELECT_SPARSITY, 3
    out = ada.select_blocks(Mt.cuda(), heads_desc=desc, mode=kmode, target=targets, flags=flags, tier_tau=0.8)
    torch.cuda.synchronize()
    M64 = Mt[0].double().numpy()
    keep, rec, nnz, _ = oracle.select_blocks(M64, blocks, "recall" if kmode == 0 else "sparsity", targets,
                                             text_sink=sink, tiers=(mode == "tiers"))
    rows = csr_rows(out.row_ptr, out.col_idx)
    for h in range(H):
        for p in range(nb):
            exp = np.nonzero(keep[h, p])[0].tolist()
            assert rows[h * nb + p] == exp, f"h{h} row {p}: {rows[h * nb + p][:8]} vs {exp[:8]}"
    np.testing.assert_array_equal(out.head_nnz[0].cpu().numpy(), nnz)
    np.testing.assert_allclose(out.head_recall[0].cpu().numpy(), rec, rtol=1e-6)
    order = out.row_order.cpu().numpy()
    cnt = np.diff(out.row_ptr.cpu().numpy())
    assert sorted(order.tolist()) == list(range(H * nb))
    assert (np.diff(cnt[order]) <= 0).all()


@pytest.mark.parametrize("nv,nt", [(70000, 226), (150000, 256), (261000, 256), (349000, 256), (392900, 256)])
@pytest.mark.parametrize("mode", ["recall", "sparsity"])
def test_select_blocks_exact_large_nb(ada, nv, nt, mode):
    """K3 at nb > 1024 (more than 32 kv-blocks per warp lane: nb = 1098 / 2348 / 4082 at block 64, and
    the KPL=192 instantiation at nb = 5458 (the 24 s length-sweep point) and 6144 (the limit)); sampled rows (every text row, the first and last video
    rows, seeded random rows) bit-exact against the oracle's per-row selection."""
    H, B = 2, 64
    blocks = oracle.block_map(nv, nt, B, False)
    nb = len(blocks)
    Mt = workloads.random_masses(H * nb, nb, seed=11).view(1, H, nb, nb)
    q = torch.empty(1, H, nv + nt, 64, dtype=torch.bfloat16, device="cuda")
    desc = ada.make_desc(q, B, nt, False)
    targets = [0.9, 0.5] if mode == "recall" else [0.9, 0.8]
    kmode = ada.SELECT_RECALL if mode == "recall" else ada.SELECT_SPARSITY
    out = ada.select_blocks(Mt.cuda(), heads_desc=desc, mode=kmode, target=targets, flags=1)
    torch.cuda.synchronize()
    rp = out.row_ptr.cpu().numpy()
    ci = out.col_idx.cpu().numpy()
    rng = np.random.default_rng(3)
    text = [i for i, b in enumerate(blocks) if b.modality == "text"]
    sample = sorted({0, nb - len(text) - 1, *text, *rng.choice(nb, 40, replace=False).tolist()})
    for h in range(H):
        for p in sample:
            forced, cands = oracle.row_forced_and_candidates(blocks, p, True)
            m = Mt[0, h, p].double().numpy()
            if mode == "recall":
                exp = oracle.select_row_recall(m, forced, cands, targets[h])
            else:
                exp = oracle.select_row_sparsity(m, forced, cands, oracle.k_from_sparsity(targets[h], nb - len(text)))
            row = h * nb + p
            got = ci[rp[row]:rp[row + 1]].tolist()
            assert got == exp, f"nb={nb} {mode} h{h} row {p}: {len(got)} kept vs {len(exp)} (first {got[:6]} / {exp[:6]})"


@pytest.mark.parametrize("levels", [3, 24, 400])
@pytest.mark.parametrize("mode", ["recall", "sparsity"])
def test_select_blocks_heavy_ties(ada, mode, levels):
    """K3 when many candidates share the cut value: masses drawn from `levels` distinct values, so the
    bisection's bracket can end with more than 32 equal masses (the exact-walk / tie-count fallback
    of select_row) or with a handful (the in-bracket resolution).  Ties are taken in ascending id
    order (the (mass desc, id asc) greedy, PAPER.md:436-448 / reading R10); bit-exact against the
    oracle on identical masses, both modes, with and without the text sink."""
    H, nv, nt, B = 4, 40000, 150, 64
    blocks = oracle.block_map(nv, nt, B, False)
    nb = len(blocks)
    g = torch.Generator().manual_seed(5 + levels)
    vals = torch.rand(levels, generator=g, dtype=torch.float64) * 3.0 + 0.01
    Mt = vals[torch.randint(0, levels, (1, H, nb, nb), generator=g)].float()
    q = torch.empty(1, H, nv + nt, 64, dtype=torch.bfloat16, device="cuda")
    desc = ada.make_desc(q, B, nt, False)
    targets = [0.3, 0.7, 0.9, 0.97]
    kmode = ada.SELECT_RECALL if mode == "recall" else ada.SELECT_SPARSITY
    for sink in (True, False):
        out = ada.select_blocks(Mt.cuda(), heads_desc=desc, mode=kmode, target=targets, flags=int(sink))
        torch.cuda.synchronize()
        keep, _, nnz, _ = oracle.select_blocks(Mt[0].double().numpy(), blocks, mode, targets, text_sink=sink)
        rows = csr_rows(out.row_ptr, out.col_idx)
        for h in range(H):
            for p in range(nb):
                exp = np.nonzero(keep[h, p])[0].tolist()
                assert rows[h * nb + p] == exp, f"{mode} L{levels} sink{sink} h{h} row {p}: {rows[h * nb + p][:8]} vs {exp[:8]}"
        np.testing.assert_array_equal(out.head_nnz[0].cpu().numpy(), nnz)


@pytest.mark.parametrize("mode", ["recall", "sparsity"])
def test_select_blocks_extreme_masses(ada, mode):
    """K3 on masses spread log-uniformly over the whole fp32 range (denormals up to 2^100 in one row)
    and targets close to 0 and 1: the bisection's first probe (budget / ncand), the counted bracket
    and the exact fp64 resolution at extreme scales.  Bit-exact against the oracle on identical masses."""
    H, nv, nt, B = 4, 50000, 150, 64
    blocks = oracle.block_map(nv, nt, B, False)
    nb = len(blocks)
    g = torch.Generator().manual_seed(13)
    e = torch.rand(1, H, nb, nb, generator=g, dtype=torch.float64) * 250.0 - 149.0   # 2^-149 .. 2^101
    Mt = torch.exp2(e).float()
    Mt[Mt == 0] = 1e-45
    q = torch.empty(1, H, nv + nt, 64, dtype=torch.bfloat16, device="cuda")
    desc = ada.make_desc(q, B, nt, False)
    targets = [1e-6, 0.5, 0.999999, 0.9] if mode == "recall" else [0.001, 0.5, 0.99, 0.9]
    kmode = ada.SELECT_RECALL if mode == "recall" else ada.SELECT_SPARSITY
    out = ada.select_blocks(Mt.cuda(), heads_desc=desc, mode=kmode, target=targets, flags=1)
    torch.cuda.synchronize()
    keep, _, nnz, _ = oracle.select_blocks(Mt[0].double().numpy(), blocks, mode, targets, text_sink=True)
    rows = csr_rows(out.row_ptr, out.col_idx)
    for h in range(H):
        for p in range(nb):
            exp = np.nonzero(keep[h, p])[0].tolist()
            assert rows[h * nb + p] == exp, f"{mode} h{h} row {p}: {rows[h * nb + p][:8]} vs {exp[:8]}"
    np.testing.assert_array_equal(out.head_nnz[0].cpu().numpy(), nnz)


@pytest.mark.parametrize("mode", ["recall", "sparsity"])
def test_select_blocks_zero_masses(ada, mode):
    """K3 on rows where most candidate masses are exactly 0 (fp32 underflow of far blocks in sharp
    heads): SPARSITY budgets larger than the non-zero count must take zero-mass blocks in ascending
    id order (reading R10), RECALL must stop at the non-zero prefix; all-zero rows keep the forced
    set / the first candidate (R25).  Bit-exact against the oracle on identical masses."""
    H, nv, nt, B = 3, 3000, 150, 64
    blocks = oracle.block_map(nv, nt, B, False)
    nb = len(blocks)
    Mt = workloads.random_masses(H * nb, nb, seed=9).view(1, H, nb, nb).clone()
    g = torch.Generator().manual_seed(4)
    zero = torch.rand(1, H, nb, nb, generator=g) < 0.9
    Mt[zero] = 0.0
    Mt[0, 1, 5] = 0.0   # one all-zero row
    q = torch.empty(1, H, nv + nt, 64, dtype=torch.bfloat16, device="cuda")
    desc = ada.make_desc(q, B, nt, False)
    targets = [0.9, 0.5, 0.99] if mode == "recall" else [0.5, 0.8, 0.95]
    kmode = ada.SELECT_RECALL if mode == "recall" else ada.SELECT_SPARSITY
    out = ada.select_blocks(Mt.cuda(), heads_desc=desc, mode=kmode, target=targets, flags=1)
    torch.cuda.synchronize()
    M64 = Mt[0].double().numpy()
    keep, _, _, _ = oracle.select_blocks(M64, blocks, mode, targets, text_sink=True)
    rows = csr_rows(out.row_ptr, out.col_idx)
    for h in range(H):
        for p in range(nb):
            exp = np.nonzero(keep[h, p])[0].tolist()
            assert rows[h * nb + p] == exp, f"{mode} h{h} row {p}: {rows[h * nb + p][:8]} vs {exp[:8]}"


def _random_csr(H, nb, density, seed):
    g = np.random.default_rng(seed)
    keep = g.random((H, nb, nb)) < density
    keep[:, np.arange(nb), g.integers(0, nb, nb)] = True
    rp = [0]
    ci = []
    for r in keep.reshape(-1, nb):
        ids = np.nonzero(r)[0].tolist()
        ci += ids
        rp.append(len(ci))
    return keep, torch.tensor(rp, dtype=torch.int32, device="cuda"), torch.tensor(ci, dtype=torch.int32, device="cuda")


@pytest.mark.parametrize("name,over", CASES)
@pytest.mark.parametrize("density", [0.05, 0.3, 1.0])
def test_block_sparse_attn(ada, name, over, density):
    """K4 vs oracle masked attention (c = +inf) on the same CSR."""
    lay = _lay(name, over)
    q, k, v = _qkv(lay)
    blocks = oracle.block_map(lay.n_video, lay.n_text, lay.block, lay.text_first)
    nb = len(blocks)
    keep, rp, ci = _random_csr(lay.heads, nb, density, 11)
    o, lse = ada.block_sparse_attn(q, k, v, rp, ci, block_size=lay.block, n_text=lay.n_text,
                                   text_first=lay.text_first, want_lse=True)
    torch.cuda.synchronize()
    scale = 1 / math.sqrt(lay.head_dim)
    for h in range(lay.heads):
        kept = [np.nonzero(keep[h, p])[0] for p in range(nb)]
        ro, rl = oracle.masked_attention(np64(q[0, h]), np64(k[0, h]), np64(v[0, h]), blocks, kept, scale)
        # masked_attention returns rows in q-block order = token order
        compare_out(o[0, h], ro, lse[0, h], rl, what=f"{name} d={density} h{h}")


def test_block_sparse_attn_large_nb(ada):
    """K4 with block ids above 4095 (16-bit ids in the kv stream): nb = 4202 at block 64, a seeded
    CSR of ~1.5% density in which every sampled row also keeps blocks >= 4096; sampled q-blocks
    against the oracle's masked attention (one q-block at a time)."""
    lay = workloads.layout_for("tiny", f=16, h=16, w=1050, n_text=77, head_dim=64, block=64, heads=1)
    q, k, v = _qkv(lay)
    blocks = oracle.block_map(lay.n_video, lay.n_text, lay.block, lay.text_first)
    nb = len(blocks)
    assert nb > 4096
    g = np.random.default_rng(17)
    rows = []
    for p in range(nb):
        ids = set(g.choice(nb, 60, replace=False).tolist())
        ids.add(int(g.integers(4096, nb)))
        rows.append(sorted(ids))
    rp = torch.tensor(np.cumsum([0] + [len(r) for r in rows]), dtype=torch.int32, device="cuda")
    ci = torch.tensor([j for r in rows for j in r], dtype=torch.int32, device="cuda")
    o, lse = ada.block_sparse_attn(q, k, v, rp, ci, block_size=lay.block, n_text=lay.n_text,
                                   text_first=lay.text_first, want_lse=True)
    torch.cuda.synchronize()
    scale = 1 / math.sqrt(lay.head_dim)
    qh, kh, vh = np64(q[0, 0]), np64(k[0, 0]), np64(v[0, 0])
    for p in sorted({0, 4095, 4096, nb - 1, *g.choice(nb, 8, replace=False).tolist()}):
        b = blocks[p]
        r = slice(b.start, b.start + b.length)
        ro, rl = oracle.masked_attention(qh, kh, vh, blocks, {p: rows[p]}, scale, q_block_ids=[p])
        compare_out(o[0, 0, r], ro, lse[0, 0, r], rl, what=f"large-nb K4 qb{p}")


@pytest.mark.parametrize("tf,block,d", [(False, 128, 128), (True, 64, 64), (True, 128, 64), (False, 64, 128)])
def test_hot_path_batch2(ada, tf, block, d):
    """K1 -> K2 -> K3 -> K4 through HotPath at batch 2 (per-(b,h) items, row offsets and the
    per-batch head tiers of K3 span both batch elements): every head of both batch elements against
    the oracle pipeline (K2 with the GPU's LSE; K4 on the GPU's CSR)."""
    from paper_2502_21079_b200.hotpath import HotPath
    lay = _lay("tiny_tf" if tf else "tiny", dict(f=4, h=9, w=10, n_text=45, head_dim=d, block=block, heads=3))
    q, k, v = _qkv(lay, batch=2)
    hp = HotPath(2, lay.heads, lay.n, lay.head_dim, lay.block, lay.n_text, lay.text_first, targets=0.9)
    o = hp.run(q, k, v)
    torch.cuda.synchronize()
    blocks = oracle.block_map(lay.n_video, lay.n_text, lay.block, lay.text_first)
    nb = len(blocks)
    scale = 1 / math.sqrt(lay.head_dim)
    rows = csr_rows(hp.csr.row_ptr, hp.csr.col_idx)
    for b in range(2):
        for h in range(lay.heads):
            qq, kk, vv = np64(q[b, h]), np64(k[b, h]), np64(v[b, h])
            od, lse = oracle.dense_attention(qq, kk, vv, scale)
            compare_out(hp.o_dense[b, h], od, hp.lse[b, h], lse, what=f"b{b} h{h} K1")
            M = oracle.block_mass(qq, kk, hp.lse[b, h].double().cpu().numpy(), blocks, scale)
            Mg = hp.mass[b, h].double().cpu().numpy()
            L = np.array([bl.length for bl in blocks], dtype=np.float64)[:, None]
            assert (np.abs(Mg - M) / L).max() <= MASS_REL, f"b{b} h{h} K2"
            for p in range(nb):
                forced, cands = oracle.row_forced_and_candidates(blocks, p, True)
                ok = oracle.select_row_recall(M[p], forced, cands, 0.9)
                good, msg = selection_ok(M[p], forced, cands, 0.9, rows[(b * lay.heads + h) * nb + p], ok)
                assert good, f"b{b} h{h} row {p}: {msg}"
            kept = [rows[(b * lay.heads + h) * nb + p] for p in range(nb)]
            so, _ = oracle.masked_attention(qq, kk, vv, blocks, kept, scale)
            compare_out(o[b, h], so, what=f"b{b} h{h} K4")


@pytest.mark.parametrize("block,d,tf", [(128, 128, False), (64, 128, True), (64, 64, False)])
def test_block_sparse_attn_midsize_random(ada, block, d, tf):
    """K4 with many work items per head (N = 16.5K tokens, H = 3: hundreds of items through the
    dynamic queue in LPT order) on a random CSR with ragged row lengths (1 to ~40% of the blocks,
    plus rows that keep every block); sampled q-blocks of every head against the oracle."""
    lay = _lay("tiny_tf" if tf else "tiny", dict(f=8, h=16, w=128, n_text=77, head_dim=d, block=block, heads=3))
    q, k, v = _qkv(lay)
    blocks = oracle.block_map(lay.n_video, lay.n_text, lay.block, lay.text_first)
    nb = len(blocks)
    g = np.random.default_rng(block + d)
    rows = []
    for r in range(lay.heads * nb):
        kind = g.random()
        if kind < 0.05:
            ids = list(range(nb))
        else:
            n = int(g.integers(1, max(2, int(0.4 * nb))))
            ids = sorted(g.choice(nb, n, replace=False).tolist())
        rows.append(ids)
    rp = torch.tensor(np.cumsum([0] + [len(r) for r in rows]), dtype=torch.int32, device="cuda")
    ci = torch.tensor([j for r in rows for j in r], dtype=torch.int32, device="cuda")
    o, lse = ada.block_sparse_attn(q, k, v, rp, ci, block_size=lay.block, n_text=lay.n_text,
                                   text_first=lay.text_first, want_lse=True)
    torch.cuda.synchronize()
    scale = 1 / math.sqrt(lay.head_dim)
    for h in range(lay.heads):
        qh, kh, vh = np64(q[0, h]), np64(k[0, h]), np64(v[0, h])
        for p in sorted({0, nb - 1, *g.choice(nb, 12, replace=False).tolist()}):
            b = blocks[p]
            r = slice(b.start, b.start + b.length)
            ro, rl = oracle.masked_attention(qh, kh, vh, blocks, {p: rows[h * nb + p]}, scale, q_block_ids=[p])
            compare_out(o[0, h, r], ro, lse[0, h, r], rl, what=f"mid B{block} d{d} h{h} qb{p}")


def test_end_to_end_tiny(ada):
    """K1 -> K2 (fresh LSE) -> K3 (recall 0.9) -> K4 against the oracle pipeline, both text orders."""
    for name in ("tiny", "tiny_tf"):
        lay = workloads.layout_for(name)
        q, k, v = _qkv(lay)
        kw = dict(block_size=lay.block, n_text=lay.n_text, text_first=lay.text_first)
        o_d, lse = ada.dense_attn_lse(q, k, v, **kw)
        M = ada.lse_cached_search(q, k, lse, **kw)
        desc = ada.make_desc(q, lay.block, lay.n_text, lay.text_first)
        out = ada.select_blocks(M, heads_desc=desc, mode=ada.SELECT_RECALL, target=[0.9] * lay.heads)
        o_s, _ = ada.block_sparse_attn(q, k, v, out.row_ptr, out.col_idx, **kw)
        torch.cuda.synchronize()
        blocks = oracle.block_map(lay.n_video, lay.n_text, lay.block, lay.text_first)
        nb = len(blocks)
        scale = 1 / math.sqrt(lay.head_dim)
        rows = csr_rows(out.row_ptr, out.col_idx)
        for h in range(lay.heads):
            qq, kk, vv = np64(q[0, h]), np64(k[0, h]), np64(v[0, h])
            ro, rl = oracle.dense_attention(qq, kk, vv, scale)
            compare_out(o_d[0, h], ro, lse[0, h], rl, what=f"{name} dense h{h}")
            Mo = oracle.block_mass(qq, kk, rl, blocks, scale)
            for p in range(nb):
                forced, cands = oracle.row_forced_and_candidates(blocks, p, True)
                ok = oracle.select_row_recall(Mo[p], forced, cands, 0.9)
                good, msg = selection_ok(Mo[p], forced, cands, 0.9, rows[h * nb + p], ok)
                assert good, f"{name} h{h} row {p}: {msg}"
            gk = [rows[h * nb + p] for p in range(nb)]
            so, _ = oracle.masked_attention(qq, kk, vv, blocks, gk, scale)
            compare_out(o_s[0, h], so, what=f"{name} sparse h{h}")


def test_run_sparse_host_matches_device(ada):
    """HotPath.run_sparse_host (H2D per head group, K4 on the cached CSR, D2H) == the device K4."""
    from paper_2502_21079_b200.hotpath import HotPath, tapered_groups
    lay = _lay("tiny", dict(heads=5, head_dim=128, block=128, f=5, h=9, w=11, n_text=37))
    q, k, v = _qkv(lay)
    hp = HotPath(1, lay.heads, lay.n, lay.head_dim, lay.block, lay.n_text, lay.text_first, targets=0.9)
    hp.run(q, k, v)
    ref = hp.o_sparse.clone()
    qh, kh, vh = (x.cpu().pin_memory() for x in (q, k, v))
    oh = torch.empty_like(qh).pin_memory()
    for groups in (3, [1, 2, 1, 1], tapered_groups(lay.heads)):   # equal groups, explicit sizes, the bench's
        oh.zero_()
        hp.run_sparse_host(qh, kh, vh, oh, groups=groups)
        torch.cuda.synchronize()
        assert torch.equal(oh, ref.cpu()), groups
    with pytest.raises(ValueError):
        hp.run_sparse_host(qh, kh, vh, oh, groups=[2, 2])            # sizes must cover every head
