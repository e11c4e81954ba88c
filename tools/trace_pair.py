"""clock64 trace of the CTA-pair kernel (diagnostic build with -DADASPA_TRACE, ADASPA_PAIR=1)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import workloads
import paper_2502_21079_b200 as ada
from paper_2502_21079_b200 import _lib

name = sys.argv[1] if len(sys.argv) > 1 else "hyv110k"
lay = workloads.layout_for(name)
q, k, v = workloads.generate_qkv(lay, device="cuda")
kw = dict(block_size=lay.block, n_text=lay.n_text, text_first=lay.text_first)
o, lse = ada.dense_attn_lse(q, k, v, **kw)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * (3 * 4096))()
assert _lib._lib.adaspa_debug_trace_pair(buf, 3 * 4096) == 0
a = np.frombuffer(buf, dtype=np.uint64).astype(np.int64).reshape(3, 4096)[:, :4000].reshape(3, 1000, 4)
mm, s0, s1 = a[0], a[1], a[2]
sl = slice(100, 900)
def st(nm, x):
    print(f"  {nm:40s} median {np.median(x):7.0f}  p10 {np.percentile(x,10):7.0f}  p90 {np.percentile(x,90):7.0f}")
print("MMA thread (leader SM clock):")
st("period (P seen -> next P seen)", np.diff(mm[:, 0])[sl])
st("P(e) seen -> V(e) full", (mm[:, 1] - mm[:, 0])[sl])
st("P seen+V full -> K(e+2) full", (mm[:, 2] - mm[:, 1])[sl])
st("K full -> PV(e)+QK(e+2) issued", (mm[:, 3] - mm[:, 2])[sl])
st("QK done -> next P seen", (mm[1:, 0] - mm[:-1, 3])[sl])
for r, s in ((0, s0), (1, s1)):
    print(f"softmax warp 4, CTA {r}:")
    st("period", np.diff(s[:, 0])[sl])
    st("S seen -> S loaded", (s[:, 1] - s[:, 0])[sl])
    st("S loaded -> P stored", (s[:, 2] - s[:, 1])[sl])
    st("P stored -> arrived", (s[:, 3] - s[:, 2])[sl])
    st("arrived -> next S seen", (s[1:, 0] - s[:-1, 3])[sl])
print("CTA0 same-clock: S(e) seen (softmax) relative to MMA 'QK(e) signalled' (step e-3's stamp 3):")
st("S(e) seen - QK(e) signalled", (s0[3:, 0] - mm[:-3, 3])[sl])
st("P(e) seen by MMA - CTA0 warp4 arrived", (mm[:, 0] - s0[:, 3])[sl])
