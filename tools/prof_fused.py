"""One fused search (K1+K2 in one dense pass + block-mass reduction) and one K1 + K2 on a BASELINE
config, for an ncu launch list (diagnostic)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import workloads
import paper_2502_21079_b200 as ada
name = sys.argv[1] if len(sys.argv) > 1 else "hyv110k"
lay = workloads.layout_for(name)
q, k, v = workloads.generate_qkv(lay, device="cuda")
kw = dict(block_size=lay.block, n_text=lay.n_text, text_first=lay.text_first)
o, lse, M = ada.dense_attn_lse_search(q, k, v, **kw)
o1, l1 = ada.dense_attn_lse(q, k, v, **kw)
M2 = ada.lse_cached_search(q, k, l1, **kw)
torch.cuda.synchronize()
print("ok")
