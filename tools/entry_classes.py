"""Share of K4 kv-stream entries (block 128) needed by both q-blocks of an item vs by one only."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import workloads
import paper_2502_21079_b200 as ada
from paper_2502_21079_b200.hotpath import HotPath

for name, tgt in (("hyv110k", 0.9),):
    lay = workloads.layout_for(name)
    q, k, v = workloads.generate_qkv(lay, device="cuda")
    hp = HotPath(1, lay.heads, lay.n, lay.head_dim, lay.block, lay.n_text, lay.text_first, targets=tgt)
    hp.run(q, k, v)
    rp = hp.csr.row_ptr.cpu().numpy(); ci = hp.csr.col_idx.cpu().numpy(); nb = hp.nb
    both = single = paired = excess = 0
    for h in range(lay.heads):
        for p in range(0, nb, 2):
            a = set(ci[rp[h * nb + p]:rp[h * nb + p + 1]].tolist())
            b = set(ci[rp[h * nb + p + 1]:rp[h * nb + p + 2]].tolist()) if p + 1 < nb else set()
            n1, n2 = len(a - b), len(b - a)
            both += len(a & b); single += n1 + n2
            paired += 2 * min(n1, n2); excess += abs(n1 - n2)
    E = both + single
    print(f"{name} recall {tgt}: entries {E}: both {both / E:.3f}, single alternating {paired / E:.3f}, "
          f"single excess (one tile only) {excess / E:.3f}")
