"""Summarise `ncu --set full` reports into profiles/ (markdown table + ncu_traffic.json for bench.py).

    python tools/ncu_summary.py TAG K1=gpurun_out/a.ncu-rep K2=... K3=... K4=...
    python tools/ncu_summary.py TAG K1=gpurun_out/x.raw.csv@0 FS=gpurun_out/x.raw.csv@1 ...

A `.raw.csv` (ncu -i rep --page raw --csv, exported on the GPU box) with `@i` picks its i-th launch.

traffic = dram__bytes_read.sum + dram__bytes_write.sum per launch (bench.py's roofline.traffic).
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % peak"),
    ("sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", "tensor pipe % (realtime)"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU) inst %"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA inst %"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU inst %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def raw(rep):
    idx = 0
    if "@" in rep:
        rep, idx = rep.rsplit("@", 1)
        idx = int(idx)
    if rep.endswith(".csv"):
        out = open(rep).read()
    else:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = [r for r in csv.reader(io.StringIO(out)) if len(r) > 5]
    h, units, vals = rows[0], rows[1], rows[2 + idx]
    d = {}
    for k, u, v in zip(h, units, vals):
        d[k] = (v, u)
        d.setdefault(k.split(".", 2)[-1] if k.count(".") >= 4 and k.split(".")[0].isupper() else k, (v, u))
    return d, vals[h.index("Kernel Name")]


def main():
    tag = sys.argv[1]
    items = [a.split("=", 1) for a in sys.argv[2:]]
    lines = [f"# ncu --set full summary ({tag})", "",
             "One launch per kernel, `ncu --set full --clock-control none` (tools/gpu_ncu_step.sh over "
             "tools/prof_step.py, or tools/prof_one.py for r01 tags); "
             "cold-cache, serialised replays: use for shares and counters, not for bench values.", ""]
    traffic = {}
    table = {}
    names = {}
    for key, rep in items:
        d, kname = raw(rep)
        names[key] = kname
        table[key] = d
        rd = float(d.get("dram__bytes_read.sum", ("0", ""))[0].replace(",", "").replace("-nan", "nan") or 0)
        wr = float(d.get("dram__bytes_write.sum", ("0", ""))[0].replace(",", "").replace("-nan", "nan") or 0)
        unit_r = d.get("dram__bytes_read.sum", ("", "byte"))[1]
        unit_w = d.get("dram__bytes_write.sum", ("", "byte"))[1]
        mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        traffic[key] = rd * mult.get(unit_r, 1) + wr * mult.get(unit_w, 1)
    cols = [k for k, _ in items]
    lines.append("| metric | " + " | ".join(cols) + " |")
    lines.append("|---|" + "---|" * len(cols))
    lines.append("| kernel | " + " | ".join(names[c].split("(")[0][-48:] for c in cols) + " |")
    for m, label in KEYS:
        row = []
        for c in cols:
            v, u = table[c].get(m, ("n/a", ""))
            row.append(f"{v} {u}".strip())
        lines.append(f"| {label} (`{m}`) | " + " | ".join(row) + " |")
    lines.append("| traffic = DRAM read + write (bytes) | " + " | ".join(f"{traffic[c]:.4g}" for c in cols) + " |")
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    with open(os.path.join(ROOT, "profiles", f"{tag}_ncu_summary.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    tj = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    old = json.load(open(tj)) if os.path.exists(tj) else {}
    old.update({k: round(v) for k, v in traffic.items() if v == v})
    old["_source"] = f"tools/ncu_summary.py {tag}: dram__bytes_read.sum + dram__bytes_write.sum per launch"
    json.dump(old, open(tj, "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
