"""Small runs of the whole path for compute-sanitizer (memcheck / racecheck / synccheck): HotPath.run
(K1-free search step: the fused dense pass + block masses with the selection epilogue + CSR, then K4),
K1 alone and K2 + K3 (the cached search), at d = 128 and 64, blocks 128 and 64, both text orders, two
items per head -- every softmax layout (row per thread; 16 rows per warp for dense d=64); then K3 alone at
nb = 862 in every selection mode, with and without heavy ties."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import workloads
from paper_2502_21079_b200.hotpath import HotPath

for d, tf, block in ((128, False, 128), (128, True, 128), (128, False, 64), (64, True, 64), (64, False, 128)):
    lay = workloads.layout_for("tiny_tf" if tf else "tiny", f=6, h=10, w=11, n_text=77, head_dim=d,
                               block=block, heads=2)
    q, k, v = (x.cuda() for x in workloads.generate_qkv(lay))
    hp = HotPath(1, lay.heads, lay.n, lay.head_dim, lay.block, lay.n_text, lay.text_first, targets=0.9)
    o = hp.run(q, k, v)
    od = hp.dense(q, k, v, lse=torch.empty_like(hp.lse))
    hp.select(hp.cached_search(q, k))
    torch.cuda.synchronize()
    assert torch.isfinite(o.float()).all() and torch.isfinite(od.float()).all()
# K3 alone at a larger nb (KPL = 28 rows in registers, every selection mode, heavy ties so the
# walk fallback runs too): random masses, no attention
import paper_2502_21079_b200 as ada
for levels in (3, 0):
    nv, nt, B, H = 55000, 150, 64, 2
    nb = -(-nv // B) + -(-nt // B)
    g = torch.Generator().manual_seed(3 + levels)
    if levels:
        vals = torch.rand(levels, generator=g, dtype=torch.float64) + 0.01
        M = vals[torch.randint(0, levels, (1, H, nb, nb), generator=g)].float()
    else:
        M = workloads.random_masses(H * nb, nb, seed=5).view(1, H, nb, nb)
    qd = torch.empty(1, H, nv + nt, 64, dtype=torch.bfloat16, device="cuda")
    desc = ada.make_desc(qd, B, nt, False)
    for mode, flags, tgt in ((ada.SELECT_RECALL, 1, [0.9, 0.5]), (ada.SELECT_SPARSITY, 1, [0.8, 0.9]),
                             (ada.SELECT_SPARSITY, 3, [0.8, 0.8]), (ada.SELECT_RECALL, 0, [0.95, 0.7])):
        ada.select_blocks(M.cuda(), heads_desc=desc, mode=mode, target=tgt, flags=flags)
    torch.cuda.synchronize()
print("sanitize case ok")
