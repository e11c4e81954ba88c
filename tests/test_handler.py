"""The plug-and-play handler (paper_2502_21079_b200/handler.py): call-order
bookkeeping on the CPU, and on the GPU a two-layer run through the paper's default mode (sparsity
with head tiers, text sink) in the [B, N, H, d] layout, checked against the oracle."""

import math

import numpy as np
import pytest
import torch

import oracle
import workloads


def test_handler_call_order_and_defaults():
    import paper_2502_21079_b200 as ada
    h = ada.adaspa_attention_handler(num_layers=3, n_text=256)
    s = h.schedule
    assert (s.kw["block_size"], s.n_steps, s.t_w, s.key_steps) == (64, 50, 10, [10, 30])
    assert s.mode == ada.SELECT_SPARSITY and s.targets == 0.8
    assert s.flags == ada.FLAG_TEXT_SINK | ada.FLAG_HEAD_TIERS
    assert [h.position(c) for c in range(7)] == [(1, 0), (1, 1), (1, 2), (2, 0), (2, 1), (2, 2), (3, 0)]
    assert h.position(150) == (1, 0)  # a new generation after n_steps * num_layers calls
    modes = [h.mode_of(t) for t in range(1, 51)]
    assert modes == oracle.schedule_trace(50, 10, [10, 30])
    with pytest.raises(ValueError):
        ada.adaspa_attention_handler(num_layers=2, n_text=8, warmup=10, key_steps=(12, 30))
    r = ada.adaspa_attention_handler(num_layers=1, n_text=8, mode="recall", recall=0.95)
    assert r.schedule.mode == ada.SELECT_RECALL and r.schedule.flags == ada.FLAG_TEXT_SINK


@pytest.mark.gpu
def test_handler_two_layers_token_major_matches_oracle():
    import paper_2502_21079_b200 as ada
    from gpu_helpers import compare_out, csr_rows, np64
    lay = workloads.layout_for("tiny", f=5, h=9, w=11, n_text=37, heads=4)
    n_steps, L = 5, 2
    attn = ada.adaspa_attention_handler(num_layers=L, n_text=lay.n_text, text_first=lay.text_first,
                                        n_steps=n_steps, warmup=2, key_steps=(2, 4), layout="bnhd")
    blocks = oracle.block_map(lay.n_video, lay.n_text, lay.block, lay.text_first)
    nb = len(blocks)
    scale = 1 / math.sqrt(lay.head_dim)
    for t in range(1, n_steps + 1):
        for layer in range(L):
            q, k, v = workloads.generate_qkv(lay, seed=workloads.synth.BASE_SEED + 31 * layer, sigma=0.05, step=t)
            qt, kt, vt = (x.transpose(1, 2).contiguous().cuda() for x in (q, k, v))  # [B, N, H, d]
            o = attn(qt, kt, vt)
            torch.cuda.synchronize()
            assert o.shape == qt.shape and o.stride() == qt.stride()
            mode = attn.mode_of(t)
            c = attn.schedule.cache(layer)
            if mode in ("full+search", "cached-search+sparse"):
                # K3 with tiers on the GPU's masses == the oracle's selection on the same masses
                keep, _, _, _ = oracle.select_blocks(c.mass[0].double().cpu().numpy(), blocks, "sparsity",
                                                     [0.8] * lay.heads, text_sink=True, tiers=True)
                rows = csr_rows(c.csr.row_ptr, c.csr.col_idx)
                for h in range(lay.heads):
                    for p in range(nb):
                        assert rows[h * nb + p] == np.nonzero(keep[h, p])[0].tolist(), (t, layer, h, p)
            for h in range(lay.heads):
                qq, kk, vv = np64(q[0, h]), np64(k[0, h]), np64(v[0, h])
                if mode in ("full", "full+search"):
                    ref, _ = oracle.dense_attention(qq, kk, vv, scale)
                else:
                    rows = csr_rows(c.csr.row_ptr, c.csr.col_idx)
                    ref, _ = oracle.masked_attention(qq, kk, vv, blocks, [rows[h * nb + p] for p in range(nb)], scale)
                compare_out(o[0, :, h], ref, what=f"t{t} layer{layer} h{h} {mode}")
    assert attn.calls == n_steps * L
