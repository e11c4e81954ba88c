"""Per-tile clock64 trace of K1 on one config (diagnostic build, see ADASPA_TRACE in attn_fwd.cu).
    nvcc ... -DADASPA_TRACE -o /tmp/libadaspa_trace.so && ADASPA_LIB=/tmp/libadaspa_trace.so python tools/trace_probe.py
"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import workloads
import paper_2502_21079_b200 as ada
from paper_2502_21079_b200 import _lib

name = sys.argv[1] if len(sys.argv) > 1 else "hyv110k"
which = sys.argv[2] if len(sys.argv) > 2 else "dense"
lay = workloads.layout_for(name)
q, k, v = workloads.generate_qkv(lay, device="cuda")
kw = dict(block_size=lay.block, n_text=lay.n_text, text_first=lay.text_first)
o, lse = ada.dense_attn_lse(q, k, v, **kw)
if which in ("sparse", "sparse2"):
    M = ada.lse_cached_search(q, k, lse, **kw)
    desc = ada.make_desc(q, lay.block, lay.n_text, lay.text_first)
    out = ada.select_blocks(M, heads_desc=desc, mode=ada.SELECT_RECALL, target=[0.9] * lay.heads)
    ada.block_sparse_attn(q, k, v, out.row_ptr, out.col_idx, **kw)
    if which == "sparse2":  # a second launch right after the first (its K/V warm in L2): its trace overwrites
        ada.block_sparse_attn(q, k, v, out.row_ptr, out.col_idx, **kw)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * 16384)()
assert _lib._lib.adaspa_debug_trace(buf, 16384) == 0
a = np.frombuffer(buf, dtype=np.uint64).astype(np.int64)
sm = a[:4000].reshape(1000, 4)
mm = a[4096:4096 + 4000].reshape(1000, 4)
mk = a[8192:8192 + 4000].reshape(1000, 4)  # [V kv_full seen, next K kv_full seen]
tp = a[12288:12288 + 4000].reshape(1000, 4)  # producer: [K wait start, K slot free, V wait start, V slot free]
n = int((sm[:, 3] > 0).sum())
sm = sm[:n]
print(f"{name} {which}: softmax warp 4 (tile 0, half 0), {n} tiles")
ld = sm[:, 1] - sm[:, 0]; mx = sm[:, 2] - sm[:, 1]; ex = sm[:, 3] - sm[:, 2]
wait = sm[1:, 0] - sm[:-1, 3]; period = np.diff(sm[:, 0])
for nm, x in (("LDTM", ld), ("max+xchg barrier", mx), ("rescale+exp+P store", ex), ("wait for next S", wait), ("period", period)):
    x = x[10:-10] if len(x) > 40 else x
    print(f"  {nm:22s} median {np.median(x):8.0f}  p10 {np.percentile(x,10):8.0f}  p90 {np.percentile(x,90):8.0f}  mean {np.mean(x):8.0f}")
print(f"  periods above 2x median: {int((period > 2 * np.median(period)).sum())} of {len(period)}, "
      f"{(period[period > 2 * np.median(period)].sum()) / period.sum() * 100:.1f}% of the traced time")
m = int((mm[:, 3] > 0).sum())
mm = mm[:m]
if m < 40:
    sys.exit(0)
print(f"MMA issuer: {m} entries")
names = ["p_full0 seen", "QK0 issued", "p_full1 seen", "QK1 issued"]
for i in range(4):
    d = np.diff(mm[:, i])[10:-10]
    print(f"  period of '{names[i]}': median {np.median(d):.0f}")
for i, j in ((0, 1), (1, 2), (2, 3)):
    d = (mm[:, j] - mm[:, i])[10:-10]
    print(f"  '{names[i]}' -> '{names[j]}': median {np.median(d):.0f}  p90 {np.percentile(d,90):.0f}")
d = (mm[1:, 0] - mm[:-1, 3])[10:-10]
print(f"  'QK1 issued' -> next 'p_full0 seen': median {np.median(d):.0f}")

# cross timeline: align MMA-thread stamps with softmax warp 4 (tile 0) stamps, same SM clock
print("timeline (cycles relative to 'p_full0 seen' of MMA entry i):")
print("  i  QK0iss  pf1seen  QK1iss  Vfull Knext | sm0:EV0(S0 seen) EV1 EV2 EV3(P0 done) | next pf0seen")
ev0 = sm[:, 0]
for i in range(100, 106):
    base = mm[i, 0]
    # softmax tile 0 event that follows QK0 issue of entry i
    j = int(np.searchsorted(ev0, mm[i, 1]))
    print(f"  {i} {mm[i,1]-base:7d} {mm[i,2]-base:8d} {mm[i,3]-base:7d} {mk[i,0]-base:6d} {mk[i,1]-base:6d} | {sm[j,0]-base:7d} {sm[j,1]-base:6d} "
          f"{sm[j,2]-base:6d} {sm[j,3]-base:6d} | {mm[i+1,0]-base:7d}")

print("producer (same frame): entry i+1's K slot wait start / K slot free / V wait start / V slot free")
for i in range(100, 106):
    base = mm[i, 0]
    # producer entry index: the producer runs ahead; find the entry whose K slot frees closest after QK0 of i
    k = int(np.searchsorted(tp[:, 1], mm[i, 1]))
    print(f"  {i}: prod entry {k}: " + " ".join(f"{tp[k, c] - base:7d}" for c in range(4)))

print("merged event list (absolute, relative to MMA entry 100 'p_full0 seen'):")
base = mm[100, 0]
evs = []
for i in range(98, 106):
    for c, nm in enumerate(["pf0seen", "QK0iss", "pf1seen", "QK1iss"]):
        evs.append((mm[i, c] - base, f"MMA e{i} {nm}"))
    evs.append((mk[i, 0] - base, f"MMA e{i} V(prev) full seen"))
    evs.append((mk[i, 1] - base, f"MMA e{i} K(next) full seen"))
for k in range(95, 110):
    for c, nm in enumerate(["K slot wait", "K slot free->issue", "V slot wait", "V slot free->issue"]):
        evs.append((tp[k, c] - base, f"  TMA p{k} {nm}"))
for t, nm in sorted(evs):
    if -3000 < t < 9000:
        print(f"  {t:7d}  {nm}")
