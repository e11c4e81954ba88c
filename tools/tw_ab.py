"""Search step t_w variants on one config, CUDA events (diagnostic; not the bench contract):
one call (adaspa_search_select, selection epilogue), fused dense pass + block mass then K3, K3 alone
(warm, on the masses just written), K3 cold (after a 512 MB L2 flush).

    python tools/tw_ab.py [config] [reps]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import workloads
import paper_2502_21079_b200 as ada
from paper_2502_21079_b200.hotpath import HotPath

name = sys.argv[1] if len(sys.argv) > 1 else "hyv110k"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
lay = workloads.layout_for(name)
q, k, v = workloads.generate_qkv(lay, device="cuda")
hp = HotPath(1, lay.heads, lay.n, lay.head_dim, lay.block, lay.n_text, lay.text_first,
             mode=ada.SELECT_RECALL, targets=0.9, flags=ada.FLAG_TEXT_SINK)
flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")


def t(fn, pre=None):
    out = []
    for i in range(reps + 1):
        if pre:
            pre()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        if i:
            out.append(a.elapsed_time(b))
    out.sort()
    return out[len(out) // 2]


r = {}
if hasattr(ada, "search_select"):
    r["one_call_ms"] = t(lambda: hp.search(q, k, v, fused=True))
    r["mass_then_k3_ms"] = t(lambda: hp.search(q, k, v, fused="mass"))
else:   # an older library build: the masses from the two-call fused path
    r["mass_then_k3_ms"] = t(lambda: hp.search(q, k, v, fused=True))
r["k3_warm_ms"] = t(lambda: hp.select(hp.mass))
r["k3_cold_ms"] = t(lambda: hp.select(hp.mass), pre=lambda: flush.zero_())
print(name, {k_: round(v_, 4) for k_, v_ in r.items()}, flush=True)
