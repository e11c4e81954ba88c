"""Host schedule: the driver's step modes against the golden trace
(PAPER.md:400-403 with the defaults of PAPER.md:547, 588, 581) and the oracle's trace for every
search strategy of the ablation (tbl:search); on the GPU, a short drifting
schedule through the C-ABI against the oracle pipeline with the t_w LSE cached (R18, R19)."""

import json
import math
import os

import numpy as np
import pytest
import torch

import oracle
import workloads
from paper_2502_21079_b200 import schedule as S


def test_trace_golden(golden_dir):
    g = json.load(open(os.path.join(golden_dir, "schedule.json")))
    tr = S.trace(g["n_steps"], g["t_w"], g["key_steps"])
    runs = []
    for m in tr:
        if runs and runs[-1][0] == m:
            runs[-1][1] += 1
        else:
            runs.append([m, 1])
    assert runs == g["runs"]


@pytest.mark.parametrize("ks", [[10], [10, 30], [10, 20, 30], [10, 20, 30, 40]])
def test_trace_matches_oracle(ks):
    assert S.trace(50, 10, ks) == oracle.schedule_trace(50, 10, ks)


def test_trace_rejects_bad_key_steps():
    with pytest.raises(ValueError):
        S.trace(50, 10, [20, 30])
    with pytest.raises(ValueError):
        S.trace(50, 10, [10, 60])


@pytest.mark.gpu
@pytest.mark.parametrize("fused", [True, False])
def test_schedule_gpu_matches_oracle_pipeline(fused):
    from gpu_helpers import compare_out, csr_rows, np64, selection_ok
    lay = workloads.layout_for("tiny")
    n_steps, t_w, ks = 6, 2, [2, 4]
    sch = S.AdaSpaSchedule(block_size=lay.block, n_text=lay.n_text, text_first=lay.text_first,
                           n_steps=n_steps, t_w=t_w, key_steps=ks, targets=0.9, fused_search=fused)
    blocks = oracle.block_map(lay.n_video, lay.n_text, lay.block, lay.text_first)
    nb = len(blocks)
    scale = 1 / math.sqrt(lay.head_dim)
    lse_cache = None
    for t in range(1, n_steps + 1):
        q, k, v = (x.cuda() for x in workloads.generate_qkv(lay, sigma=0.05, step=t))
        o = sch.attention(0, t, q, k, v)
        torch.cuda.synchronize()
        mode = oracle.schedule_trace(n_steps, t_w, ks)[t - 1]
        c = sch.cache(0)
        for h in range(lay.heads):
            qq, kk, vv = np64(q[0, h]), np64(k[0, h]), np64(v[0, h])
            od, lse = oracle.dense_attention(qq, kk, vv, scale)
            if mode in ("full", "full+search"):
                compare_out(o[0, h], od, what=f"t{t} h{h} dense")
            if mode == "full+search":
                lse_cache = lse_cache if lse_cache is not None else {}
                lse_cache[h] = lse
            if mode in ("full+search", "cached-search+sparse"):
                M = oracle.block_mass(qq, kk, lse_cache[h], blocks, scale)
                rows = csr_rows(c.csr.row_ptr, c.csr.col_idx)
                for p in range(nb):
                    forced, cands = oracle.row_forced_and_candidates(blocks, p, True)
                    ok = oracle.select_row_recall(M[p], forced, cands, 0.9)
                    good, msg = selection_ok(M[p], forced, cands, 0.9, rows[h * nb + p], ok)
                    assert good, f"t{t} h{h} row {p}: {msg}"
            if mode in ("sparse", "cached-search+sparse"):
                rows = csr_rows(c.csr.row_ptr, c.csr.col_idx)
                so, _ = oracle.masked_attention(qq, kk, vv, blocks, [rows[h * nb + p] for p in range(nb)], scale)
                compare_out(o[0, h], so, what=f"t{t} h{h} sparse")
    assert [m for (_, _, m) in sch.calls] == oracle.schedule_trace(n_steps, t_w, ks)


def test_tapered_groups_cover_every_head():
    """run_sparse_host's head groups (host logic, no GPU): sizes >= 1 covering every head once, one-head
    groups at both ends once there are enough heads."""
    from paper_2502_21079_b200.hotpath import tapered_groups
    for h in range(1, 200):
        g = tapered_groups(h)
        assert sum(g) == h and min(g) >= 1
        if h >= 12:
            assert g[:4] == [1] * 4 and g[-4:] == [1] * 4 and max(g) == 2
    assert tapered_groups(24) == [1, 1, 1, 1] + [2] * 8 + [1, 1, 1, 1]
