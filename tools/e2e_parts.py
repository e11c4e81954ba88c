"""Where the e2e sparse step's time goes beyond the pinned-H2D bound (12 head groups, HYV-110K):
H2D alone, H2D with the per-group D2H of O overlapped (no K4), K4 alone per group, and the full
HotPath.run_sparse_host step."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import workloads
import paper_2502_21079_b200 as ada
from paper_2502_21079_b200 import _lib as L
from paper_2502_21079_b200.hotpath import HotPath

lay = workloads.layout_for("hyv110k")
q, k, v = workloads.generate_qkv(lay, device="cuda")
hp = HotPath(1, lay.heads, lay.n, lay.head_dim, lay.block, lay.n_text, lay.text_first, targets=0.9)
hp.run(q, k, v)
qh, kh, vh = (x.cpu().pin_memory() for x in (q, k, v))
oh = torch.empty_like(qh).pin_memory()
torch.cuda.synchronize()
G, H = 12, lay.heads
bounds = [H * g // G for g in range(G + 1)]
cs, os_ = torch.cuda.Stream(), torch.cuda.Stream()


def t(fn, it=5):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    for _ in range(it): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / it


def h2d_d2h(with_d2h):
    cur = torch.cuda.current_stream()
    cs.wait_stream(cur); os_.wait_stream(cur)
    for g in range(G):
        h0, h1 = bounds[g], bounds[g + 1]
        with torch.cuda.stream(cs):
            for dev, host in ((hp.q, qh), (hp.k, kh), (hp.v, vh)):
                dev[:, h0:h1].copy_(host[:, h0:h1], non_blocking=True)
        if with_d2h:
            with torch.cuda.stream(os_):
                oh[:, h0:h1].copy_(hp.o_sparse[:, h0:h1], non_blocking=True)
    cur.wait_stream(cs); cur.wait_stream(os_)


def k4_groups():
    for g in range(G):
        h0, h1 = bounds[g], bounds[g + 1]
        rp = hp.csr.row_ptr[h0 * hp.nb: h1 * hp.nb + 1]
        L.block_sparse_attn(hp.q[:, h0:h1], hp.k[:, h0:h1], hp.v[:, h0:h1], rp, hp.csr.col_idx,
                            o=hp.o_sparse[:, h0:h1], workspace=hp.ws, **hp.kw)


print(f"H2D only (12 groups): {t(lambda: h2d_d2h(False)):.2f} ms")
print(f"H2D + D2H overlapped, no K4: {t(lambda: h2d_d2h(True)):.2f} ms")
print(f"K4 per group, 12 launches: {t(k4_groups):.2f} ms")
print(f"K4 one launch (all heads): {t(lambda: L.block_sparse_attn(hp.q, hp.k, hp.v, hp.csr.row_ptr, hp.csr.col_idx, o=hp.o_sparse, workspace=hp.ws, **hp.kw)):.2f} ms")
print(f"full run_sparse_host(12): {t(lambda: hp.run_sparse_host(qh, kh, vh, oh, groups=12)):.2f} ms")
