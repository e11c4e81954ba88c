"""How much of K4's MMA work is on kept blocks: emulates the kv-stream packing of
sparse_stream_kernel (attn_fwd.cu: pattern-grouped pairs at block 64; ID_ORDER=1 for id order) on a real CSR and reports executed / kept FLOPs.

    python tools/sparse_efficiency.py [config] [recall|sparsity] [target]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import workloads
import paper_2502_21079_b200 as ada
from bench import block_lengths

ID_ORDER = os.environ.get("ID_ORDER") == "1"  # emulate the former ascending-id pairing
name = sys.argv[1] if len(sys.argv) > 1 else "cogx45k"
mode = sys.argv[2] if len(sys.argv) > 2 else "recall"
target = float(sys.argv[3]) if len(sys.argv) > 3 else 0.9
lay = workloads.layout_for(name, **({"block": int(sys.argv[4])} if len(sys.argv) > 4 else {}))
q, k, v = workloads.generate_qkv(lay, device="cuda")
kw = dict(block_size=lay.block, n_text=lay.n_text, text_first=lay.text_first)
desc = ada.make_desc(q, lay.block, lay.n_text, lay.text_first)
o, lse = ada.dense_attn_lse(q, k, v, **kw)
M = ada.lse_cached_search(q, k, lse, **kw)
out = ada.select_blocks(M, heads_desc=desc, mode=ada.SELECT_RECALL if mode == "recall" else ada.SELECT_SPARSITY,
                        target=[target] * lay.heads)
rp = out.row_ptr.cpu().numpy()
ci = out.col_idx.cpu().numpy()
L = np.array(block_lengths(lay), dtype=np.float64)
nb = len(L)
two = lay.block == 64
nq = 4 if two else 2
kept = executed = 0.0
n_ent_tot = 0
for bh in range(lay.heads):
    for p in range((nb + nq - 1) // nq):
        rows = [p * nq + s for s in range(nq) if p * nq + s < nb]
        lists = [set(ci[rp[bh * nb + r]:rp[bh * nb + r + 1]].tolist()) for r in rows]
        for r, s in zip(rows, lists):
            kept += L[r] * sum(L[j] for j in s)
        memb = lambda j: sum(1 << m for m in range(len(lists)) if j in lists[m])  # noqa: E731
        uni = sorted(set().union(*lists), key=(lambda j: (memb(j), j)) if two and not ID_ORDER else None)
        ents = [uni[i:i + 2] for i in range(0, len(uni), 2)] if two else [[j] for j in uni]
        n_ent_tot += len(ents)
        for e in ents:
            for t in range(2):  # q tile t: q-blocks (2t, 2t+1) at B=64, q-block t at B=128
                members = [2 * t, 2 * t + 1] if two else [t]
                need = any(m < len(lists) and any(j in lists[m] for j in e) for m in members)
                executed += 128.0 * 128.0 if need else 0.0
print(f"{name} {mode} {target}: kept pair work {kept:.4g}, executed MMA tile work {executed:.4g}, "
      f"efficiency {kept / executed:.3f}, entries {n_ent_tot}")
