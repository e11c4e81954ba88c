"""K3 alone on real block masses (diagnostic; not the bench contract).

    python tools/k3_bench.py [config] [reps]

Runs the search step once (LSE), K2 with that LSE (the masses a later key step selects on), then
times K3 (adaspa_select_blocks) `reps` times per selection mode with CUDA events on the current
stream behind a sleep kernel (the host's launch cost hidden, as inside a bench step), warm (M resident in L2 after the previous call) -- median / min ms and the HBM rate of the
algorithmic bytes (DESIGN.md §6 K3).  Under ncu pass reps=1.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import workloads
import paper_2502_21079_b200 as ada
from paper_2502_21079_b200.hotpath import HotPath

name = sys.argv[1] if len(sys.argv) > 1 else "hyv110k"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 50
lay = workloads.layout_for(name)
q, k, v = workloads.generate_qkv(lay, device="cuda")
hp = HotPath(1, lay.heads, lay.n, lay.head_dim, lay.block, lay.n_text, lay.text_first,
             mode=ada.SELECT_RECALL, targets=0.9, flags=ada.FLAG_TEXT_SINK)
hp.search(q, k, v)
m2 = hp.cached_search(q, k)
del q, k, v
torch.cuda.synchronize()
H, nb = lay.heads, m2.shape[-1]
modes = {
    "recall0.9": dict(mode=ada.SELECT_RECALL, target=[0.9] * H, flags=ada.FLAG_TEXT_SINK),
    "recall0.9_no_row_order": dict(mode=ada.SELECT_RECALL, target=[0.9] * H, flags=ada.FLAG_TEXT_SINK,
                                   want_row_order=False),
    "sparsity0.8": dict(mode=ada.SELECT_SPARSITY, target=[0.8] * H, flags=ada.FLAG_TEXT_SINK),
    "sparsity0.8_tiers": dict(mode=ada.SELECT_SPARSITY, target=[0.8] * H,
                              flags=ada.FLAG_TEXT_SINK | ada.FLAG_HEAD_TIERS),
}
for key, kw in modes.items():
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(1_000_000)  # keep the GPU busy while the host enqueues: device time only
        a.record()
        ada.select_blocks(m2, heads_desc=hp.desc, tier_tau=0.8, out=None if kw.get('want_row_order') is False else hp.csr, **kw)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    nnz = int(hp.csr.row_ptr[-1].item())
    rows = H * nb
    byts = 4 * rows * nb + 4 * (rows + 1) + 4 * nnz + 4 * rows
    med = ts[len(ts) // 2]
    print(f"{name} {key}: nb {nb} rows {rows} nnz {nnz} median {med:.4f} ms min {ts[0]:.4f} ms "
          f"-> {byts / (med / 1e3) / 1e9:.1f} GB/s", flush=True)
