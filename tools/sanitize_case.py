"""Small K1 -> K2 -> K3 -> K4 runs for compute-sanitizer (memcheck / racecheck / synccheck):
d = 128 at blocks 128 and 64, both text orders, two items per head."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import workloads
from paper_2502_21079_b200.hotpath import HotPath

for tf, block in ((False, 128), (True, 128), (False, 64)):
    lay = workloads.layout_for("tiny_tf" if tf else "tiny", f=6, h=10, w=11, n_text=77, head_dim=128,
                               block=block, heads=2)
    q, k, v = (x.cuda() for x in workloads.generate_qkv(lay))
    hp = HotPath(1, lay.heads, lay.n, lay.head_dim, lay.block, lay.n_text, lay.text_first, targets=0.9)
    o = hp.run(q, k, v)
    torch.cuda.synchronize()
    assert torch.isfinite(o.float()).all()
print("sanitize case ok")
