"""Pinned-host copy rates on the box: H2D of Q,K,V alone, D2H of O alone, and both at once on two
streams (the floor of the end-to-end sparse step, which must move both)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import workloads
lay = workloads.layout_for("hyv110k")
shape = (1, lay.heads, lay.n, lay.head_dim)
dq = [torch.empty(shape, dtype=torch.bfloat16, device="cuda") for _ in range(4)]
hq = [torch.empty(shape, dtype=torch.bfloat16).pin_memory() for _ in range(4)]
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn, it=5):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    for _ in range(it): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / it
def h2d():
    for i in range(3): dq[i].copy_(hq[i], non_blocking=True)
def d2h():
    hq[3].copy_(dq[3], non_blocking=True)
def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur); s2.wait_stream(cur)
    with torch.cuda.stream(s1): h2d()
    with torch.cuda.stream(s2): d2h()
    cur.wait_stream(s1); cur.wait_stream(s2)
gb_in, gb_out = 3 * dq[0].numel() * 2 / 1e9, dq[0].numel() * 2 / 1e9
a, b, c = t(h2d), t(d2h), t(both)
print(f"H2D {gb_in:.2f} GB: {a:.2f} ms ({gb_in / a * 1e3:.1f} GB/s); D2H {gb_out:.2f} GB: {b:.2f} ms "
      f"({gb_out / b * 1e3:.1f} GB/s); both at once: {c:.2f} ms")
