"""First full-size timing of K1..K4 on a BASELINE config (not the bench contract; see bench.py)."""
import math, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import workloads
import paper_2502_21079_b200 as ada

name = sys.argv[1] if len(sys.argv) > 1 else "hyv110k"
recall = float(sys.argv[2]) if len(sys.argv) > 2 else 0.9
lay = workloads.layout_for(name)
t0 = time.time()
q, k, v = workloads.generate_qkv(lay, device="cuda")
torch.cuda.synchronize()
print(f"{lay} gen {time.time()-t0:.1f}s", flush=True)
kw = dict(block_size=lay.block, n_text=lay.n_text, text_first=lay.text_first)
desc = ada.make_desc(q, lay.block, lay.n_text, lay.text_first)
N, H, d = lay.n, lay.heads, lay.head_dim

def timeit(fn, it=5):
    fn(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    for _ in range(it): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / it

o, lse = ada.dense_attn_lse(q, k, v, **kw)
t1 = timeit(lambda: ada.dense_attn_lse(q, k, v, o=o, lse=lse, **kw), 3)
fl = 4.0 * N * N * d * H
print(f"K1 dense: {t1:.2f} ms  {fl/t1/1e9:.1f} TFLOP/s", flush=True)
M = ada.lse_cached_search(q, k, lse, **kw)
t2 = timeit(lambda: ada.lse_cached_search(q, k, lse, block_mass=M, **kw), 3)
print(f"K2 search: {t2:.2f} ms  {fl/2/t2/1e9:.1f} TFLOP/s(QK)  exp/s {N*N*H/t2/1e9:.2f} T", flush=True)
out = ada.select_blocks(M, heads_desc=desc, mode=ada.SELECT_RECALL, target=[recall]*H)
t3 = timeit(lambda: ada.select_blocks(M, heads_desc=desc, mode=ada.SELECT_RECALL, target=[recall]*H, out=out), 5)
nnz = out.head_nnz.sum().item()
nb = ada.num_blocks(desc)
print(f"K3 select: {t3*1000:.1f} us  nnz {nnz} density {nnz/(H*nb*nb):.3f} per-head {[round(x/(nb*nb),3) for x in out.head_nnz[0].tolist()]}", flush=True)
print("head recall", [round(x, 4) for x in out.head_recall[0].tolist()])
ws = torch.empty(ada.sparse_workspace_bytes(desc), dtype=torch.uint8, device="cuda")
o2, _ = ada.block_sparse_attn(q, k, v, out.row_ptr, out.col_idx, workspace=ws, **kw)
t4 = timeit(lambda: ada.block_sparse_attn(q, k, v, out.row_ptr, out.col_idx, o=o2, workspace=ws, **kw), 5)
# kept FLOPs: 4 d sum |qb||kb| over kept pairs
from bench import kept_flops
kept = kept_flops(lay, out, 1)[0] / 4.0
kfl = 4.0 * d * kept
print(f"K4 sparse: {t4:.2f} ms  effective {kfl/t4/1e9:.1f} TFLOP/s (kept FLOPs {kfl/1e12:.2f} TF)", flush=True)
print(f"search overhead (K2+K3)/K1 = {(t2+t3)/t1:.3f}")
