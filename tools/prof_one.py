"""Run the hot path a fixed number of times on one BASELINE config (for ncu captures).

    python tools/prof_one.py [config] [runs]

Under ncu use -k regex:<kernel> -s <skip> -c <count> to pick launches; every run() launches
K1, K2, K3 (3 kernels), K4 (prep 2 + attention 1) in that order.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import workloads
import paper_2502_21079_b200 as ada
from paper_2502_21079_b200.hotpath import HotPath

name = sys.argv[1] if len(sys.argv) > 1 else "hyv110k"
runs = int(sys.argv[2]) if len(sys.argv) > 2 else 2
lay = workloads.layout_for(name)
q, k, v = workloads.generate_qkv(lay, device="cuda")
hp = HotPath(1, lay.heads, lay.n, lay.head_dim, lay.block, lay.n_text, lay.text_first,
             mode=ada.SELECT_RECALL, targets=0.9, flags=ada.FLAG_TEXT_SINK)
for _ in range(runs):
    hp.run(q, k, v)
torch.cuda.synchronize()
print("done", name, runs)
