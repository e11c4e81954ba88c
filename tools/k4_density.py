import os, sys, json
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), 'tools'))
import torch, workloads, paper_2502_21079_b200 as ada
from bench import kept_flops
from schedule_bench import time_call
for mode, tgt in (("sparsity", 0.9), ("recall", 0.9), ("recall", 0.7)):
    lay = workloads.layout_for("hyv110k")
    q, k, v = workloads.generate_qkv(lay, device="cuda")
    kw = dict(block_size=lay.block, n_text=lay.n_text, text_first=lay.text_first)
    desc = ada.make_desc(q, lay.block, lay.n_text, lay.text_first)
    o, lse = ada.dense_attn_lse(q, k, v, **kw)
    M = ada.lse_cached_search(q, k, lse, **kw)
    out = ada.select_blocks(M, heads_desc=desc, mode=ada.SELECT_SPARSITY if mode == "sparsity" else ada.SELECT_RECALL, target=[tgt] * lay.heads)
    ws = torch.empty(ada.sparse_workspace_bytes(desc), dtype=torch.uint8, device="cuda")
    t = time_call(lambda: ada.block_sparse_attn(q, k, v, out.row_ptr, out.col_idx, o=o, workspace=ws, **kw), 5)
    fl, nnz = kept_flops(lay, out, lay.head_dim)
    print(os.environ.get("TAG"), mode, tgt, f"density {nnz/(lay.heads*ada.num_blocks(desc)**2):.3f} K4 {t:.2f} ms {fl/t/1e9:.1f} TF")
