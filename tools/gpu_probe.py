"""Quick per-kernel probe for bring-up on the GPU box: prints error metrics instead of
asserting, one kernel per process (so a hang only costs its own timeout).
    python tools/gpu_probe.py dense|search|select|sparse|e2e [name]
"""
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import torch

import oracle
import workloads
import paper_2502_21079_b200 as ada
from gpu_helpers import np64, csr_rows

what = sys.argv[1]
name = sys.argv[2] if len(sys.argv) > 2 else "tiny"
over = eval(sys.argv[3]) if len(sys.argv) > 3 else {}
lay = workloads.layout_for(name, **over)
q, k, v = (x.cuda() for x in workloads.generate_qkv(lay))
kw = dict(block_size=lay.block, n_text=lay.n_text, text_first=lay.text_first)
scale = 1 / math.sqrt(lay.head_dim)
blocks = oracle.block_map(lay.n_video, lay.n_text, lay.block, lay.text_first)
nb = len(blocks)
print(f"{what} {lay}", flush=True)
t0 = time.time()
if what == "dense":
    o, lse = ada.dense_attn_lse(q, k, v, **kw)
    torch.cuda.synchronize()
    print("kernel done", time.time() - t0, flush=True)
    for h in range(lay.heads):
        ro, rl = oracle.dense_attention(np64(q[0, h]), np64(k[0, h]), np64(v[0, h]), scale)
        d = np.abs(np64(o[0, h]) - ro)
        dl = np.abs(lse[0, h].double().cpu().numpy() - rl)
        print(f"h{h} O maxabs {d.max():.3e} meanabs {d.mean():.3e} lse maxabs {dl.max():.3e}")
        if d.max() > 0.02:
            bad = np.argwhere(d > 0.02)
            print(" bad rows", np.unique(bad[:, 0])[:40])
elif what == "search":
    lse_ref = np.stack([oracle.dense_attention(np64(q[0, h]), np64(k[0, h]), np64(v[0, h]), scale)[1]
                        for h in range(lay.heads)])
    lse_t = torch.tensor(lse_ref[None], dtype=torch.float32, device="cuda")
    M = ada.lse_cached_search(q, k, lse_t, **kw)
    torch.cuda.synchronize()
    print("kernel done", time.time() - t0, flush=True)
    L = np.array([b.length for b in blocks], float)
    for h in range(lay.heads):
        Mo = oracle.block_mass(np64(q[0, h]), np64(k[0, h]), lse_t[0, h].double().cpu().numpy(), blocks, scale)
        Mg = M[0, h].double().cpu().numpy()
        err = np.abs(Mg - Mo) / L[:, None]
        print(f"h{h} max|dM|/|qb| {err.max():.3e} rowsum err {np.abs(Mg.sum(1)/L - 1).max():.3e}")
        if err.max() > 1e-4:
            print(" bad cells", np.argwhere(err > 1e-4)[:20].tolist())
elif what == "select":
    H = 4
    Mt = workloads.random_masses(H * nb, nb, seed=3).view(1, H, nb, nb)
    desc = ada.make_desc(torch.empty(1, H, lay.n, lay.head_dim, dtype=torch.bfloat16, device="cuda"),
                         lay.block, lay.n_text, lay.text_first)
    out = ada.select_blocks(Mt.cuda(), heads_desc=desc, mode=ada.SELECT_RECALL, target=[0.5, 0.8, 0.9, 0.99])
    torch.cuda.synchronize()
    keep, rec, nnz, _ = oracle.select_blocks(Mt[0].double().numpy(), blocks, "recall", [0.5, 0.8, 0.9, 0.99])
    rows = csr_rows(out.row_ptr, out.col_idx)
    bad = sum(rows[h * nb + p] != np.nonzero(keep[h, p])[0].tolist() for h in range(H) for p in range(nb))
    print("rows mismatching", bad, "of", H * nb, "nnz", out.head_nnz.cpu().tolist(), nnz.tolist())
elif what == "sparse":
    g = np.random.default_rng(1)
    keep = g.random((lay.heads, nb, nb)) < float(os.environ.get("DENS", "0.3"))
    keep[:, np.arange(nb), g.integers(0, nb, nb)] = True
    rp, ci = [0], []
    for r in keep.reshape(-1, nb):
        ci += np.nonzero(r)[0].tolist()
        rp.append(len(ci))
    rp = torch.tensor(rp, dtype=torch.int32, device="cuda")
    ci = torch.tensor(ci, dtype=torch.int32, device="cuda")
    o, lse = ada.block_sparse_attn(q, k, v, rp, ci, want_lse=True, **kw)
    torch.cuda.synchronize()
    print("kernel done", time.time() - t0, flush=True)
    for h in range(lay.heads):
        ro, rl = oracle.masked_attention(np64(q[0, h]), np64(k[0, h]), np64(v[0, h]), blocks,
                                         [np.nonzero(keep[h, p])[0] for p in range(nb)], scale)
        d = np.abs(np64(o[0, h]) - ro)
        dl = np.abs(lse[0, h].double().cpu().numpy() - rl)
        print(f"h{h} O maxabs {d.max():.3e} meanabs {d.mean():.3e} lse maxabs {dl.max():.3e}")
        if d.max() > 0.02:
            bad = np.argwhere(d > 0.02)
            print(" bad rows", np.unique(bad[:, 0])[:40])
print("elapsed", time.time() - t0)
