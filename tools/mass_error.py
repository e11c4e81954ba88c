"""Measured block-mass error at a full-size BASELINE config: max |dM|/T over sampled
q-block rows of every head, for the fused search (K1+K2 in one dense pass) and for K2 on the same
fp32 LSE, against the fp64 oracle's block mass with that LSE.  Prints one JSON line."""
import json, math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import oracle
import workloads
import paper_2502_21079_b200 as ada

name = sys.argv[1] if len(sys.argv) > 1 else "hyv110k"
per_head = int(sys.argv[2]) if len(sys.argv) > 2 else 2
lay = workloads.layout_for(name)
q, k, v = workloads.generate_qkv(lay, device="cuda")
kw = dict(block_size=lay.block, n_text=lay.n_text, text_first=lay.text_first)
_, lse, Mf = ada.dense_attn_lse_search(q, k, v, **kw)
M2 = ada.lse_cached_search(q, k, lse, **kw)
torch.cuda.synchronize()
blocks = oracle.block_map(lay.n_video, lay.n_text, lay.block, lay.text_first)
nb = len(blocks)
scale = 1.0 / math.sqrt(lay.head_dim)
rng = np.random.default_rng(5)
worst = {"fused": 0.0, "k2": 0.0}
n = 0
for h in range(lay.heads):
    qh, kh = q[0, h].float().double().cpu().numpy(), k[0, h].float().double().cpu().numpy()
    lg = lse[0, h].double().cpu().numpy()
    for p in rng.choice(nb, per_head, replace=False).tolist() + ([nb - 1] if h == 0 else []):
        M = oracle.block_mass(qh, kh, lg, blocks, scale, q_block_ids=[p])[0]
        T = M.sum()
        for key, G in (("fused", Mf), ("k2", M2)):
            e = np.abs(G[0, h, p].double().cpu().numpy() - M).max() / T
            worst[key] = max(worst[key], float(e))
        n += 1
print(json.dumps({"config": name, "rows_sampled": n, "max_dM_over_T": worst}))
