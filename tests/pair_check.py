"""Test infrastructure (run by tests/test_gpu_pair.py with ADASPA_PAIR=1): parity of the CTA-pair kernel:
K1 dense and K4 block-sparse at d=128, block 128, several 256-row pair items per head, both text
orders, batch 2, against the fp64 oracle (tolerances of tests/gpu_helpers.py)."""
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import torch

import oracle
import workloads
import paper_2502_21079_b200 as ada
from gpu_helpers import compare_out, np64

assert os.environ.get("ADASPA_PAIR") == "1", "run with ADASPA_PAIR=1"
case = sys.argv[1] if len(sys.argv) > 1 else "dense"
for tf in (False, True):
    lay = workloads.layout_for("tiny_tf" if tf else "tiny", f=6, h=10, w=21, n_text=77, head_dim=128,
                               block=128, heads=3)
    q, k, v = (x.cuda() for x in workloads.generate_qkv(lay, batch=2))
    kw = dict(block_size=lay.block, n_text=lay.n_text, text_first=lay.text_first)
    scale = 1 / math.sqrt(lay.head_dim)
    blocks = oracle.block_map(lay.n_video, lay.n_text, lay.block, lay.text_first)
    nb = len(blocks)
    if case == "dense":
        o, lse = ada.dense_attn_lse(q, k, v, **kw)
        torch.cuda.synchronize()
        for b in range(2):
            for h in range(lay.heads):
                ro, rl = oracle.dense_attention(np64(q[b, h]), np64(k[b, h]), np64(v[b, h]), scale)
                compare_out(o[b, h], ro, lse[b, h], rl, what=f"pair dense tf={tf} b{b} h{h}")
    else:
        g = np.random.default_rng(5)
        keep = g.random((2 * lay.heads, nb, nb)) < 0.25
        keep[:, np.arange(nb), g.integers(0, nb, nb)] = True
        rp, ci = [0], []
        for r in keep.reshape(-1, nb):
            ci += np.nonzero(r)[0].tolist()
            rp.append(len(ci))
        rp = torch.tensor(rp, dtype=torch.int32, device="cuda")
        ci = torch.tensor(ci, dtype=torch.int32, device="cuda")
        o, lse = ada.block_sparse_attn(q, k, v, rp, ci, want_lse=True, **kw)
        torch.cuda.synchronize()
        for b in range(2):
            for h in range(lay.heads):
                kept = [np.nonzero(keep[b * lay.heads + h, p])[0] for p in range(nb)]
                ro, rl = oracle.masked_attention(np64(q[b, h]), np64(k[b, h]), np64(v[b, h]), blocks, kept, scale)
                compare_out(o[b, h], ro, lse[b, h], rl, what=f"pair sparse tf={tf} b{b} h{h}")
print("pair ok", case)
