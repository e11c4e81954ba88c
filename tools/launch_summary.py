"""Summarise an ncu launch list (--metrics gpu__time_duration.sum) of bench.py into profiles/:
per-kernel mean time and share of our kernels' total, to compare with bench.py's CUDA-event shares."""
import csv
import os
import sys

src, out = sys.argv[1], sys.argv[2]
rows = [r for r in csv.reader(open(src)) if len(r) > 5]
h = rows[0]
ik, iv, iu = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
agg = {}
for r in rows[1:]:
    if "adaspa" not in r[ik]:
        continue
    name = r[ik].split("(")[0].replace("void ", "").replace("adaspa::<unnamed>::", "").replace("adaspa::", "")
    scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6, "ms": 1.0, "msecond": 1.0}.get(r[iu], 1e-6)
    agg.setdefault(name, []).append(float(r[iv].replace(",", "")) * scale)
tot = sum(sum(v) for v in agg.values())
desc = sys.argv[3] if len(sys.argv) > 3 else "python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e (HYV-110K)"
lines = [f"# ncu launch list summary: {os.path.basename(src)}", "",
         f"`ncu --metrics gpu__time_duration.sum --clock-control none` over `{desc}`. "
         "Per-launch times are cold-cache and serialised: compare shares.", "",
         "| kernel | launches | mean ms | share of our kernels |", "|---|---|---|---|"]
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    lines.append(f"| `{k}` | {len(v)} | {sum(v)/len(v):.4f} | {sum(v)/tot*100:.2f}% |")
open(out, "w").write("\n".join(lines) + "\n")
print("\n".join(lines))
