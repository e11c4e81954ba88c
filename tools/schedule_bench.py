"""Schedule-level measurements on one B200 (BASELINE.json configs[4] and SURVEY.md §8(f) f2).

    python tools/schedule_bench.py schedule [--key-steps 10,30 ...]   # 50-step run, HYV-110K
    python tools/schedule_bench.py sweep                               # length-scaling sweep

schedule: one HunyuanVideo-shaped layer (HYV-110K) driven through the AdaSpa schedule
    (paper_2502_21079_b200.schedule.AdaSpaSchedule: warm-up K1, K1+K2+K3 at t_w, K4 with the cached
    CSR, K2(t_w LSE)+K3+K4 at later key steps).  Every step uses drifted
    inputs x_t = sqrt(1-s^2) x + s rms(x) noise_t, s = 0.05, generated before the
    step's timed region; each step's attention is timed with CUDA events on the launching stream.
    Reports per-mode ms, the layer's attention time over 50 steps, the all-dense time (50 x K1) and
    the ratio, for the T_s variants of PAPER.md:703-708.
sweep: the kernel-level analogue of the scaling study (sparsity 0.9,
    block 64; T_s = {10, 30} since {0, 30} contradicts t_key^1 = t_w, reading R20): HunyuanVideo
    720p at 5/8/16/24 s (latent frames f = 4 s + 1 at 16 fps, 45 x 80 patches, 256 text tokens),
    blocks 64 and 128.  Per-mode times are measured (3 timed runs each after one warm-up) and the
    50-step schedule time is composed from them: 9 full + 1 full+search + sparse + cached-search
    steps (t_w: the fused dense pass + K3).  Reports K1 / K4 TFLOP/s, kept density and the schedule
    speedup over all-dense.
"""
import argparse
import json
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import workloads
import paper_2502_21079_b200 as ada
from paper_2502_21079_b200 import schedule as S
from bench import kept_flops  # block geometry and kept-pair FLOPs, as bench.py counts them


def drift(base, sigma, gen):
    keep = math.sqrt(1.0 - sigma * sigma)
    out = []
    for x in base:
        rms = x.float().pow(2).mean().sqrt()
        n = torch.randn(x.shape, generator=gen, device=x.device, dtype=torch.float32)
        out.append((keep * x.float() + sigma * rms * n).to(torch.bfloat16))
    return out


def run_schedule(args, emit=True):
    lay = workloads.layout_for("hyv110k")
    dev = "cuda"
    q0, k0, v0 = workloads.generate_qkv(lay, device=dev)
    gen = torch.Generator(device=dev)
    results = []
    for ks in args.key_steps:
        key_steps = [int(x) for x in ks.split(",")]
        sch = S.AdaSpaSchedule(block_size=lay.block, n_text=lay.n_text, text_first=lay.text_first,
                               n_steps=50, t_w=key_steps[0], key_steps=key_steps, targets=args.recall)
        o = torch.empty_like(q0)
        per_mode = {}
        total = 0.0
        gen.manual_seed(workloads.synth.BASE_SEED)
        for t in range(1, 51):
            q, k, v = drift((q0, k0, v0), 0.05, gen)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record()
            sch.attention(0, t, q, k, v, o=o)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            mode = S.step_mode(t, sch.t_w, sch.key_steps)
            per_mode.setdefault(mode, []).append(ms)
            total += ms
        c = sch.cache(0)
        dens = c.csr.head_nnz.sum().item() / (lay.heads * ada.num_blocks(ada.make_desc(q0, lay.block, lay.n_text,
                                                                                           lay.text_first)) ** 2)
        full = sum(per_mode[S.FULL]) / len(per_mode[S.FULL])
        rec = {"workload": "hyv110k", "n_steps": 50, "t_w": key_steps[0], "key_steps": key_steps,
               "selection": f"recall {args.recall} per head, text sink", "drift_sigma": 0.05,
               "ms_per_mode": {m: round(sum(v) / len(v), 3) for m, v in per_mode.items()},
               "steps_per_mode": {m: len(v) for m, v in per_mode.items()},
               "attention_ms_per_layer": round(total, 1), "all_dense_ms_per_layer": round(50 * full, 1),
               "speedup_vs_dense": round(50 * full / total, 3), "final_mask_density": round(dens, 4)}
        if emit:
            print(json.dumps(rec), flush=True)
        results.append(rec)
    return results


def time_call(fn, it=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(it):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / it


def run_sweep(args, blocks=(64, 128), seconds=(5, 8, 16, 24), emit=True):
    results = []
    for block in blocks:
        for secs in seconds:
            f = 4 * secs + 1
            lay = workloads.layout_for("hyv110k", f=f, block=block)
            t0 = time.time()
            q, k, v = workloads.generate_qkv(lay, device="cuda")
            kw = dict(block_size=lay.block, n_text=lay.n_text, text_first=lay.text_first)
            desc = ada.make_desc(q, lay.block, lay.n_text, lay.text_first)
            nb = ada.num_blocks(desc)
            H, N, d = lay.heads, lay.n, lay.head_dim
            o, lse = ada.dense_attn_lse(q, k, v, **kw)
            M = ada.lse_cached_search(q, k, lse, **kw)
            out = ada.select_blocks(M, heads_desc=desc, mode=ada.SELECT_SPARSITY, target=[0.9] * H)
            ws = torch.empty(ada.sparse_workspace_bytes(desc), dtype=torch.uint8, device="cuda")
            t_full = time_call(lambda: ada.dense_attn_lse(q, k, v, o=o, lse=lse, **kw))
            t_search = time_call(lambda: ada.lse_cached_search(q, k, lse, block_mass=M, **kw))
            # the search step t_w: the fused dense pass (block LSEs + masses, in head passes whose
            # scratch stays under 32 GB) then K3 (SPARSITY mode has no fused selection epilogue)
            per_head = ada.fused_search_workspace_bytes(desc, 1)
            hpp = max(1, min(H, (32 << 30) // per_head))
            fws = torch.empty(ada.fused_search_workspace_bytes(desc, hpp), dtype=torch.uint8, device="cuda")
            Mf = torch.empty_like(M)
            t_fused = time_call(lambda: ada.dense_attn_lse_search(q, k, v, o=o, lse=lse, block_mass=Mf, workspace=fws,
                                                                  **kw))
            del fws, Mf
            t_sel = time_call(lambda: ada.select_blocks(M, heads_desc=desc, mode=ada.SELECT_SPARSITY,
                                                        target=[0.9] * H, out=out))
            t_sparse = time_call(lambda: ada.block_sparse_attn(q, k, v, out.row_ptr, out.col_idx, o=o,
                                                               workspace=ws, **kw))
            fl, nnz = kept_flops(lay, out, d)
            dense_fl = 4.0 * N * N * d * H
            modes = S.trace(50, 10, [10, 30])
            sched = sum({S.FULL: t_full, S.FULL_SEARCH: t_fused + t_sel, S.SPARSE: t_sparse,
                         S.CACHED_SEARCH_SPARSE: t_search + t_sel + t_sparse}[m] for m in modes)
            rec = {"video_s": secs, "latent_frames": f, "seq_len": N, "block": block, "nb": nb,
                   "selection": "sparsity 0.9 per head (row-wise top-k + text sink)",
                   "K1_ms": round(t_full, 2), "K1_tflops": round(dense_fl / t_full / 1e9, 1),
                   "K2_ms": round(t_search, 2), "K3_ms": round(t_sel, 3), "fused_search_ms": round(t_fused, 2),
                   "fused_heads_per_pass": hpp,
                   "K4_ms": round(t_sparse, 2), "K4_tflops_kept": round(fl / t_sparse / 1e9, 1),
                   "kept_density": round(nnz / (H * nb * nb), 4),
                   "schedule_ms_per_layer": round(sched, 1), "all_dense_ms_per_layer": round(50 * t_full, 1),
                   "speedup_vs_dense": round(50 * t_full / sched, 3), "gen_s": round(time.time() - t0, 1)}
            if emit:
                print(json.dumps(rec), flush=True)
            results.append(rec)
            del q, k, v, o, lse, M, out, ws
            torch.cuda.empty_cache()
    return results


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("what", choices=["schedule", "sweep"])
    ap.add_argument("--key-steps", nargs="+", default=["10", "10,30", "10,20,30", "10,20,30,40"])
    ap.add_argument("--recall", type=float, default=0.9)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    assert torch.cuda.is_available()
    res = run_schedule(args) if args.what == "schedule" else run_sweep(args)
    if args.out:
        json.dump(res, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
