"""K4 pipeline ceiling: time K4 on a real HYV-110K CSR with a diagnostic library.

    python tools/k4_ablate.py save /tmp/csr.pt             # CSR from the product library (K1 -> K2 -> K3)
    ADASPA_LIB=<lib built with -DADASPA_ABLATE=4> python tools/k4_ablate.py time /tmp/csr.pt

The second call loads the saved CSR and times K4 alone (kept-block TFLOP/s as bench.py counts it)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import workloads
import paper_2502_21079_b200 as ada
from paper_2502_21079_b200.hotpath import HotPath
from bench import kept_flops

mode, path = sys.argv[1], sys.argv[2]
name = sys.argv[3] if len(sys.argv) > 3 else "hyv110k"
lay = workloads.layout_for(name)
q, k, v = workloads.generate_qkv(lay, device="cuda")
kw = dict(block_size=lay.block, n_text=lay.n_text, text_first=lay.text_first)
if mode == "save":
    hp = HotPath(1, lay.heads, lay.n, lay.head_dim, lay.block, lay.n_text, lay.text_first, targets=0.9)
    hp.run(q, k, v)
    torch.save({"row_ptr": hp.csr.row_ptr.cpu(), "col_idx": hp.csr.col_idx.cpu()}, path)
    print("saved", path)
    sys.exit(0)
d = torch.load(path)
rp, ci = d["row_ptr"].cuda(), d["col_idx"].cuda()
desc = ada.make_desc(q, lay.block, lay.n_text, lay.text_first)
nb = ada.num_blocks(desc)
ws = torch.empty(ada.sparse_workspace_bytes(desc), dtype=torch.uint8, device="cuda")
o = torch.empty_like(q)

class _Csr:
    row_ptr, col_idx = rp, ci
fl, _ = kept_flops(lay, _Csr, lay.head_dim)  # as bench.py counts them
for _ in range(2):
    ada.block_sparse_attn(q, k, v, rp, ci, o=o, workspace=ws, **kw)
torch.cuda.synchronize()
s, e = torch.cuda.Event(True), torch.cuda.Event(True)
s.record()
for _ in range(5):
    ada.block_sparse_attn(q, k, v, rp, ci, o=o, workspace=ws, **kw)
e.record(); torch.cuda.synchronize()
ms = s.elapsed_time(e) / 5
print(f"{name} lib={os.environ.get('ADASPA_LIB') or 'default'}: K4 {ms:.2f} ms  {fl / ms / 1e9:.1f} TFLOP/s on kept blocks")
