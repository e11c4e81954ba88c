"""Sweep the synthetic sharpness range and report per-head kept density at recall 0.9."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, workloads
import paper_2502_21079_b200 as ada
name = sys.argv[1]
lay = workloads.layout_for(name)
for lo, hi in [(1.5, 4.0), (2.5, 5.0), (3.0, 6.0), (3.5, 6.5), (4.0, 7.0), (4.5, 8.0)]:
    q, k, v = workloads.generate_qkv(lay, device="cuda", sharp=(lo, hi))
    kw = dict(block_size=lay.block, n_text=lay.n_text, text_first=lay.text_first)
    o, lse = ada.dense_attn_lse(q, k, v, **kw)
    M = ada.lse_cached_search(q, k, lse, **kw)
    desc = ada.make_desc(q, lay.block, lay.n_text, lay.text_first)
    nb = ada.num_blocks(desc)
    out = ada.select_blocks(M, heads_desc=desc, mode=ada.SELECT_RECALL, target=[0.9] * lay.heads)
    dens = (out.head_nnz[0].double() / (nb * nb)).cpu()
    s = (q[0, :, :2048].float() @ k[0, :, :4096].float().transpose(1, 2)) / lay.head_dim ** 0.5
    print(f"{name} A=[{lo},{hi}] mean density {dens.mean():.3f} min {dens.min():.3f} max {dens.max():.3f} "
          f"spread {dens.max()/dens.min():.1f} max|S|~{s.abs().max().item():.1f}", flush=True)
    del q, k, v, o, lse, M
