"""e2e sparse step from pinned host memory vs the number of head groups of HotPath.run_sparse_host,
plus the raw pinned H2D bandwidth (the bound of that step)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import workloads
import paper_2502_21079_b200 as ada
from paper_2502_21079_b200.hotpath import HotPath

lay = workloads.layout_for("hyv110k")
q, k, v = workloads.generate_qkv(lay, device="cuda")
hp = HotPath(1, lay.heads, lay.n, lay.head_dim, lay.block, lay.n_text, lay.text_first, targets=0.9)
hp.run(q, k, v)
qh, kh, vh = (x.cpu().pin_memory() for x in (q, k, v))
oh = torch.empty_like(qh).pin_memory()
torch.cuda.synchronize()
def t(fn, it=5):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    for _ in range(it): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / it
h2d = t(lambda: [d.copy_(h, non_blocking=True) for d, h in ((hp.q, qh), (hp.k, kh), (hp.v, vh))])
print(f"H2D 3 x {qh.numel()*2/1e9:.3f} GB: {h2d:.2f} ms = {3*qh.numel()*2/h2d/1e6:.1f} GB/s")
# arguments: a number of equal groups, or comma-separated head counts (e.g. 1,1,2,4,4,4,4,2,1,1)
for arg in (sys.argv[1:] or ["4", "8", "12", "24"]):
    g = [int(x) for x in arg.split(",")] if "," in arg else int(arg)
    ms = t(lambda: hp.run_sparse_host(qh, kh, vh, oh, groups=g))
    print(f"groups {arg}: {ms:.2f} ms per sparse step")
