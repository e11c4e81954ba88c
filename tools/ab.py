"""A/B timing of library builds on the same box (diagnostic; not the bench contract).

    python tools/ab.py [--config hyv110k] [--reps 3] [--what k1,k2,k4] LIB [LIB ...]

Each (rep, lib) runs in its own process (ADASPA_LIB=LIB), alternating A B A B ..., so clock and power
drift hit every build alike.  K4 runs on the CSR the FIRST library selects (saved once), so every
build times the same kept blocks.  Prints one line per run and a median summary per library."""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

CHILD = r'''
import json, os, sys, torch
sys.path.insert(0, %(root)r)
import workloads
import paper_2502_21079_b200 as ada
from paper_2502_21079_b200.hotpath import HotPath
from bench import kept_flops
lay = workloads.layout_for(%(config)r, **%(over)r)
q, k, v = workloads.generate_qkv(lay, device="cuda")
kw = dict(block_size=lay.block, n_text=lay.n_text, text_first=lay.text_first)
N, H, d = lay.n, lay.heads, lay.head_dim
csr_path = %(csr)r
if not os.path.exists(csr_path):
    hp = HotPath(1, H, N, d, lay.block, lay.n_text, lay.text_first, targets=0.9)
    hp.run(q, k, v)
    torch.save({"row_ptr": hp.csr.row_ptr.cpu(), "col_idx": hp.csr.col_idx.cpu()}, csr_path)
c = torch.load(csr_path)
rp, ci = c["row_ptr"].cuda(), c["col_idx"].cuda()
class _C: row_ptr, col_idx = rp, ci
kfl, _ = kept_flops(lay, _C, d)
def timeit(fn, it):
    fn(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    for _ in range(it): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / it
out = {}
what = %(what)r.split(",")
o = torch.empty_like(q); lse = torch.empty(1, H, N, dtype=torch.float32, device="cuda")
if "k1" in what:
    t = timeit(lambda: ada.dense_attn_lse(q, k, v, o=o, lse=lse, **kw), 5)
    out["k1_ms"] = t; out["k1_tflops"] = 4.0 * N * N * d * H / t / 1e9
if "k2" in what:
    ada.dense_attn_lse(q, k, v, o=o, lse=lse, **kw)
    M = ada.lse_cached_search(q, k, lse, **kw)
    t = timeit(lambda: ada.lse_cached_search(q, k, lse, block_mass=M, **kw), 5)
    out["k2_ms"] = t
if "fs" in what:
    desc0 = ada.make_desc(q, lay.block, lay.n_text, lay.text_first)
    nb = ada.num_blocks(desc0)
    wsf = torch.empty(ada.fused_search_workspace_bytes(desc0, 0), dtype=torch.uint8, device="cuda")
    Mf = torch.empty(1, H, nb, nb, dtype=torch.float32, device="cuda")
    t = timeit(lambda: ada.dense_attn_lse_search(q, k, v, o=o, lse=lse, block_mass=Mf, workspace=wsf, **kw), 3)
    out["fs_ms"] = t
    del wsf
if "k4" in what:
    desc = ada.make_desc(q, lay.block, lay.n_text, lay.text_first)
    ws = torch.empty(ada.sparse_workspace_bytes(desc), dtype=torch.uint8, device="cuda")
    t = timeit(lambda: ada.block_sparse_attn(q, k, v, rp, ci, o=o, workspace=ws, **kw), 10)
    out["k4_ms"] = t; out["k4_tflops"] = kfl / t / 1e9
print("RESULT " + json.dumps(out))
'''


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("libs", nargs="+")
    ap.add_argument("--config", default="hyv110k")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--what", default="k1,k4")
    ap.add_argument("--block", type=int, default=0, help="override the config's block size")
    a = ap.parse_args()
    over = {"block": a.block} if a.block else {}
    csr = f"/tmp/ab_csr_{a.config}_{a.block}.pt"
    if os.path.exists(csr):
        os.unlink(csr)
    res = {lib: [] for lib in a.libs}
    for r in range(a.reps):
        for lib in a.libs:
            env = dict(os.environ, ADASPA_LIB=os.path.abspath(lib))
            code = CHILD % dict(root=ROOT, config=a.config, csr=csr, what=a.what, over=over)
            p = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
            line = [x for x in p.stdout.splitlines() if x.startswith("RESULT ")]
            if p.returncode or not line:
                print(f"{lib} rep {r}: FAILED\n{p.stdout[-2000:]}\n{p.stderr[-3000:]}", flush=True)
                continue
            d = json.loads(line[0][7:])
            res[lib].append(d)
            print(f"{os.path.basename(lib)} rep {r}: " + "  ".join(f"{k} {v:.2f}" for k, v in d.items()), flush=True)
    print("median:")
    for lib, rows in res.items():
        if not rows:
            continue
        keys = rows[0].keys()
        med = {k: sorted(x[k] for x in rows)[len(rows) // 2] for k in keys}
        print(f"  {os.path.basename(lib)}: " + "  ".join(f"{k} {v:.2f}" for k, v in med.items()), flush=True)


if __name__ == "__main__":
    main()
