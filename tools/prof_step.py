"""One bench step on a BASELINE config for ncu captures (diagnostic; not the bench contract):
K1 alone, the search step t_w in one call (dense BLSE pass, block mass + selection epilogue, CSR), K4,
K2 with the cached LSE, K3 on its masses -- the kernels in that launch order (attn_fwd_kernel: dense,
then BLSE, then sparse).

    python tools/prof_step.py [config] [runs] [heads_per_pass]

heads_per_pass > 0 splits the search step's dense pass into launches of that many heads (smaller
block-LSE scratch: ncu's replay has to save and restore what a launch writes).
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import workloads
import paper_2502_21079_b200 as ada
from paper_2502_21079_b200.hotpath import HotPath

name = sys.argv[1] if len(sys.argv) > 1 else "hyv110k"
runs = int(sys.argv[2]) if len(sys.argv) > 2 else 1
hpp = int(sys.argv[3]) if len(sys.argv) > 3 else 0
lay = workloads.layout_for(name)
q, k, v = workloads.generate_qkv(lay, device="cuda")
hp = HotPath(1, lay.heads, lay.n, lay.head_dim, lay.block, lay.n_text, lay.text_first,
             mode=ada.SELECT_RECALL, targets=0.9, flags=ada.FLAG_TEXT_SINK)
hp.heads_per_pass = hpp
o = torch.empty_like(q)
for _ in range(runs):
    hp.dense(q, k, v, o=o)
    hp.search(q, k, v)
    hp.sparse(q, k, v)
    hp.select(hp.cached_search(q, k))
torch.cuda.synchronize()
print("done", name, runs)
