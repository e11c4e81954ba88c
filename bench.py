#!/usr/bin/env python
"""bench.py -- AdaSpa hot path on B200 (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config hyv110k]
                    [--lpt] [--ulysses] [--no-variants]

A step is one pass of the whole hot path over one HunyuanVideo-shaped layer
(BASELINE.json configs[2]: H=24, d=128, ~110K tokens, block 128, head-adaptive recall 0.9):
K1 dense attention + LSE -> K2 LSE-cached block-mass search -> K3 selection -> K4 block-sparse
forward.  metric = BASELINE.json's metric; `value` = effective TFLOP/s of the block-sparse forward
on kept blocks (4*d*sum_kept |qb||kb| / K4 time), whole job: sum over ranks / max over ranks.
ms/layer, the search overhead and every kernel's roofline (median / p90 per kernel) are extra keys;
`variants` holds the paper's default selection (sparsity 0.8 + head tiers) on the same layer and the
CogVideoX-shaped layer (configs[1]).

Multi-GPU (`--gpus N` spawns N ranks through torch.distributed.run unless already under torchrun):
ONE layer, head-sharded -- strong scaling.  Rank p runs the search on its
contiguous head group (equal dense work); `--lpt` then all-gathers the CSRs (NCCL, timed as
`exchange`) and runs K4 on a longest-processing-time head set by kept tiles; `--ulysses` adds the
sequence->head all-to-all of Q/K/V in and O out (BASELINE configs[3]).
`--impl reference`: the fp64 oracle (oracle/) timed on the host cores on a bounded sample.
"""

import argparse
import json
import math
import os
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

METRIC = "block-sparse attn effective TFLOP/s & ms/layer @110K tok; search overhead ms"
UNIT = "TFLOP/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="hyv110k")
    ap.add_argument("--recall", type=float, default=0.9)
    ap.add_argument("--mode", default="recall", choices=["recall", "sparsity-tiers"])
    ap.add_argument("--lpt", action="store_true",
                    help="K4 on an LPT head set by kept tiles (CSRs all-gathered after the search)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-variants", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--ulysses", action="store_true",
                    help="BASELINE configs[3]: sequence-sharded activations, NCCL all-to-all to head shards "
                         "and back around the search step and around the sparse step (strong scaling)")
    ap.add_argument("--p2p", action="store_true",
                    help="with --ulysses: the exchange over peer memory (dist.PeerExchange: IPC-mapped buffers, "
                         "copy-engine copies, stream-ordered flags) instead of NCCL all-to-all")
    return ap.parse_args()


def maybe_spawn(args):
    """`--gpus N` outside torchrun: re-launch this command as N ranks (one per GPU) through
    torch.distributed.run on 127.0.0.1 and return its exit code; None when nothing was spawned."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ or args.impl == "reference":
        return None
    n_dev = torch.cuda.device_count()
    if n_dev < args.gpus and os.environ.get("ADASPA_BENCH_BACKEND", "nccl") == "nccl":
        print(json.dumps({"error": f"--gpus {args.gpus} but {n_dev} CUDA devices visible"}), flush=True)
        return 2
    import socket
    so = socket.socket()
    so.bind(("127.0.0.1", 0))
    port = so.getsockname()[1]
    so.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "sm_max_mhz": 1965.0}, \
        "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region (B200_PROFILING.md)."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, dev):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(dev), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except OSError:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        self.p.wait()
        self.f.flush()
        rows = [r.split(",") for r in open(self.f.name).read().strip().splitlines() if r.count(",") >= 6]
        os.unlink(self.f.name)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        sm, mx, reasons = [], None, set()
        for r in rows:
            try:
                sm.append(float(r[0]))
                mx = float(r[1])
            except ValueError:
                continue
            for i, n in enumerate(names):
                if "Active" in r[3 + i] and "Not" not in r[3 + i]:
                    reasons.add(n)
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def block_lengths(lay):
    """Valid token count of each block of the modality-aware grid."""
    B = lay.block
    n_first = lay.n_text if lay.text_first else lay.n_video
    out = []
    for start, stop in ((0, n_first), (n_first, lay.n)):
        for s in range(start, stop, B):
            out.append(min(B, stop - s))
    return out


def kept_flops(lay, csr, d):
    """4 * d * sum over kept (q-block, kv-block) pairs of |qb| * |kb| (partial blocks counted exactly)."""
    L = torch.tensor(block_lengths(lay), dtype=torch.float64, device=csr.row_ptr.device)
    nbk = L.numel()
    rp = csr.row_ptr.long()
    nnz = int(rp[-1].item())
    rows = torch.repeat_interleave(torch.arange(rp.numel() - 1, device=rp.device), rp[1:] - rp[:-1])
    ci = csr.col_idx[:nnz].long()
    return 4.0 * d * float((L[rows % nbk] * L[ci]).sum().item()), nnz


def roofline_entry(bound, achieved, peak, unit, traffic=None, **extra):
    e = {"bound": bound, "achieved": round(achieved, 3), "peak": round(peak, 3), "unit": unit,
         "frac": round(achieved / peak, 4) if peak else None, "traffic": traffic}
    e.update(extra)
    return e


def load_traffic():
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(p):
        try:
            return json.load(open(p))
        except ValueError:
            return {}
    return {}


def cpu_baseline_sample(lay, q, k, v, csr, seconds):
    """The oracle's block-sparse forward (masked attention) with the GPU's CSR on a
    bounded sample of the same workload: q-blocks visited round-robin over all heads (seeded order)
    until `seconds` of CPU time are spent; value = effective TFLOP/s on the kept blocks it processed."""
    import numpy as np
    import oracle
    try:
        from threadpoolctl import threadpool_info
        cores = max((i.get("num_threads", 1) for i in threadpool_info()), default=1)
    except Exception:  # noqa: BLE001
        cores = os.cpu_count()
    blocks = oracle.block_map(lay.n_video, lay.n_text, lay.block, lay.text_first)
    nb = len(blocks)
    H = lay.heads
    rp = csr.row_ptr.cpu().numpy()
    ci = csr.col_idx[: int(rp[-1])].cpu().numpy()
    scale = 1.0 / math.sqrt(lay.head_dim)
    order = np.random.default_rng(5).permutation(nb)
    cache = {}
    flops, done, heads_seen = 0.0, 0, set()
    i = 0
    dt = 0.0
    while dt < seconds and i < H * nb:
        h, p = i % H, int(order[(i // H) % nb])
        i += 1
        if h not in cache:
            if len(cache) >= 4:
                cache.pop(next(iter(cache)))
            cache[h] = tuple(x[0, h].float().double().cpu().numpy() for x in (q, k, v))
        qh, kh, vh = cache[h]
        row = h * nb + p
        kept = {p: ci[rp[row]:rp[row + 1]].tolist()}
        t0 = time.perf_counter()
        oracle.masked_attention(qh, kh, vh, blocks, kept, scale, q_block_ids=[p])
        dt += time.perf_counter() - t0
        flops += 4.0 * lay.head_dim * blocks[p].length * sum(blocks[j].length for j in kept[p])
        done += 1
        heads_seen.add(h)
    return {"value": round(flops / dt / 1e12, 6), "unit": UNIT, "cores": int(cores), "kind": "oracle",
            "sample": f"oracle masked attention (fp64 numpy) with the GPU's CSR on {done} q-blocks "
                      f"(round-robin over {len(heads_seen)} heads, seeded block order) of {lay.name}, "
                      f"{dt:.1f} s of oracle time (fp64 upcasts excluded)"}


def stats(xs):
    """median and p90 (nearest rank) of a list of per-step times."""
    ys = sorted(xs)
    if not ys:
        return None, None
    return ys[len(ys) // 2] if len(ys) % 2 else 0.5 * (ys[len(ys) // 2 - 1] + ys[len(ys) // 2]), \
        ys[min(len(ys) - 1, int(math.ceil(0.9 * len(ys))) - 1)]


class _Csr:
    def __init__(self, row_ptr, col_idx):
        self.row_ptr, self.col_idx = row_ptr, col_idx


def local_device(local):
    """The rank's GPU.  ADASPA_BENCH_BACKEND=gloo (a plumbing check of the multi-rank code paths on a
    box with fewer GPUs than ranks; its timings mean nothing) lets ranks share devices."""
    return local % max(1, torch.cuda.device_count())


def init_dist(ws, local):
    if ws > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local_device(local))
        backend = os.environ.get("ADASPA_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    else:
        torch.cuda.set_device(0)


def l2_flush_buffer(dev):
    return torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)   # 512 MB > 126 MB L2


def time_k3_cold(hp, flush, reps=5):
    """K3 alone right after an L2 flush (M read from HBM), median ms."""
    import paper_2502_21079_b200 as ada
    out = []
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        ada.select_blocks(hp.mass, heads_desc=hp.desc, mode=hp.mode, target=hp.targets, flags=hp.flags,
                          tier_tau=hp.tier_tau, out=hp.csr)
        b.record()
        torch.cuda.synchronize()
        out.append(a.elapsed_time(b))
    return stats(out)[0]


def kernel_entries(lay, nb, nnz, kfl, med, peaks, traffic, p90=None, heads=None, sm_mhz=None):
    """Roofline entries of the path's kernels from per-kernel median ms.  med / p90:
    dicts with keys K1, FS (fused search, optional), K2, K3, K4."""
    tens_peak = peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"])
    sm_max = peaks.get("sm_max_mhz", 1965.0)
    exp_peak = 16.0 * 148 * sm_max * 1e6 / 1e12      # MUFU.EX2 16/clk/SM (T exp/s)
    H = lay.heads if heads is None else heads
    N, d = lay.n, lay.head_dim
    dense_fl = 4.0 * N * N * d * H
    k3_bytes = 4.0 * nb * nb * H + 4.0 * (H * nb + 1) + 4.0 * nnz + 4.0 * H * nb
    p90 = p90 or {}
    rnd = (lambda x, n=3: None if x is None else round(x, n))  # noqa: E731
    out = {
        "K1_dense_attn_lse": roofline_entry("tensor", dense_fl / (med["K1"] / 1e3) / 1e12, tens_peak, "TFLOP/s",
                                            traffic.get("K1"), ms=rnd(med["K1"]), ms_p90=rnd(p90.get("K1")),
                                            exp_frac=round(N * N * H / (med["K1"] / 1e3) / 1e12 / exp_peak, 4),
                                            exp_frac_at_clock=round(N * N * H / (med["K1"] / 1e3) / 1e12 /
                                                                    (16.0 * 148 * (sm_mhz or sm_max) * 1e6 / 1e12), 4)),
    }
    if med.get("FS"):
        # algorithmic work of the fused search = the dense pass's 4N^2dH: the block masses reuse its
        # exponentials (no second QK^T); plus the block-LSE bytes written and read (4*(nb+1)*N per head)
        out["K1K2K3_search_step"] = roofline_entry(
            "tensor", dense_fl / (med["FS"] / 1e3) / 1e12, tens_peak, "TFLOP/s", traffic.get("FS"),
            ms=rnd(med["FS"]), ms_p90=rnd(p90.get("FS")),
            blse_gb=round(2 * 4.0 * (nb + 1) * N * H / 1e9, 3),
            note="the whole search step t_w in one C-ABI call (adaspa_search_select): dense pass + block "
                 "LSEs (attn_fwd_kernel kModeBlse), block_mass_kernel with the per-row RECALL selection "
                 "epilogue, CSR assembly (head / scan / write)")
    k2_rate = N * N * H / (med["K2"] / 1e3) / 1e12
    # K2 sends 1 exponential pair in 8 to an FMA-pipe polynomial (search.cu kSearchPolyMask): the MUFU pipe
    # itself carries 7/8 of the rate; against its rate at the measured median SM clock of the run
    mufu_clk = 16.0 * 148 * (sm_mhz or sm_max) * 1e6 / 1e12
    out["K2_lse_cached_search"] = roofline_entry("alu", k2_rate, exp_peak, "Texp/s",
                                                 traffic.get("K2"), ms=rnd(med["K2"]), ms_p90=rnd(p90.get("K2")),
                                                 tensor_tflops=round(dense_fl / 2 / (med["K2"] / 1e3) / 1e12, 1),
                                                 mufu_share=0.875, mufu_frac_at_clock=round(0.875 * k2_rate / mufu_clk, 4),
                                                 peak_note="MUFU.EX2 16/clk/SM x 148 at sm_max_mhz; frac counts the "
                                                           "FMA-pipe exponentials too")
    out["K3_select_blocks"] = roofline_entry("hbm", k3_bytes / (med["K3"] / 1e3) / 1e9, peaks["hbm_gbs"], "GB/s",
                                             traffic.get("K3"), ms=rnd(med["K3"], 4), ms_p90=rnd(p90.get("K3"), 4))
    # one exponential per kept (q, k) pair, 4d FLOPs each: at d = 64 the MUFU.EX2 rate (16/clk/SM) bounds
    # the kept-block rate below the tensor peak -- 4 * 64 * 16 * 148 * clock = 1190 TFLOP/s at 1965 MHz,
    # 982 at 1620 -- so the entry also reports the exponential rate against MUFU at the run's clock
    k4_exp = kfl / (4.0 * d) / (med["K4"] / 1e3) / 1e12
    out["K4_block_sparse_attn"] = roofline_entry("tensor", kfl / (med["K4"] / 1e3) / 1e12, tens_peak, "TFLOP/s",
                                                 traffic.get("K4"), ms=rnd(med["K4"]), ms_p90=rnd(p90.get("K4")),
                                                 exp_frac=round(k4_exp / exp_peak, 4),
                                                 exp_frac_at_clock=round(k4_exp / mufu_clk, 4),
                                                 mufu_bound_tflops_at_clock=round(4.0 * d * mufu_clk, 1))
    return out


def variant_tiers(hp, q, k, v, lay, peaks, reps=5):
    """The paper's default selection on the same layer: SPARSITY 0.8 with
    head-adaptive tiers and the text sink, on the block masses of the main run's last search (exact
    LSE); K3 (tiers: two selection passes) and K4 on its CSR, median ms over `reps`."""
    import paper_2502_21079_b200 as ada
    H, nb = lay.heads, hp.nb
    rows = H * nb
    e = lambda n, dt: torch.empty(n, dtype=dt, device=q.device)  # noqa: E731
    csr = ada.Csr(e(rows + 1, torch.int32), e(rows * nb, torch.int32), e(rows, torch.int32),
                  torch.empty(1, H, dtype=torch.float32, device=q.device),
                  torch.empty(1, H, dtype=torch.int64, device=q.device))
    o = torch.empty_like(q)
    t3, t4 = [], []
    for i in range(reps + 1):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        ev[0].record()
        ada.select_blocks(hp.mass, heads_desc=hp.desc, mode=ada.SELECT_SPARSITY, target=[0.8] * H,
                          flags=ada.FLAG_TEXT_SINK | ada.FLAG_HEAD_TIERS, tier_tau=0.8, out=csr)
        ev[1].record()
        ada.block_sparse_attn(q, k, v, csr.row_ptr, csr.col_idx, block_size=lay.block, n_text=lay.n_text,
                              text_first=lay.text_first, o=o, workspace=hp.ws)
        ev[2].record()
        torch.cuda.synchronize()
        if i:
            t3.append(ev[0].elapsed_time(ev[1]))
            t4.append(ev[1].elapsed_time(ev[2]))
    kfl, nnz = kept_flops(lay, csr, lay.head_dim)
    tens_peak = peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"])
    m3, m4 = stats(t3)[0], stats(t4)[0]
    tf = kfl / (m4 / 1e3) / 1e12
    return {"selection": "sparsity 0.8 + head tiers (tau 0.8) + text sink, row-wise (paper default, "
                         "PAPER.md:527-533, 547, 549-550)",
            "K3_ms": round(m3, 4), "K4_ms": round(m4, 3), "K4_tflops": round(tf, 3),
            "K4_frac": round(tf / tens_peak, 4), "kept_density": round(nnz / (H * nb * nb), 4),
            "head_nnz": [int(x) for x in csr.head_nnz[0].tolist()]}


def variant_schedule_and_sweep(args):
    """BASELINE configs[4] (one HYV-110K layer through the 50-step schedule, T_s = {10, 30}, drifting
    inputs) and the length sweep of SURVEY.md f2 (HunyuanVideo 720p 5-24 s,
    block 128, sparsity 0.9), from tools/schedule_bench.py, so the driver's run
    measures them too."""
    import argparse as _ap
    import importlib.util
    spec = importlib.util.spec_from_file_location("_schedule_bench", os.path.join(ROOT, "tools", "schedule_bench.py"))
    sb = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(sb)
    ns = _ap.Namespace(key_steps=["10,30"], recall=args.recall)
    sched = sb.run_schedule(ns, emit=False)[0]
    sweep = sb.run_sweep(ns, blocks=(128,), seconds=(5, 8, 16, 24), emit=False)
    torch.cuda.empty_cache()
    return {"schedule_hyv110k_50steps": sched,
            "length_sweep_block128": [{k: r[k] for k in ("video_s", "seq_len", "nb", "K1_tflops", "K4_tflops_kept",
                                                         "kept_density", "fused_search_ms", "K1_ms",
                                                         "schedule_ms_per_layer", "speedup_vs_dense")}
                                      for r in sweep]}


def variant_config(name, args, peaks, traffic, reps=5, sm_mhz=None):
    """Another BASELINE config (CogVideoX-shaped layer, configs[1]) through the whole hot path:
    per-kernel median ms and roofline."""
    import paper_2502_21079_b200 as ada
    import workloads
    from paper_2502_21079_b200.hotpath import HotPath
    lay = workloads.layout_for(name)
    dev = torch.device("cuda", torch.cuda.current_device())
    q, k, v = workloads.generate_qkv(lay, device=dev)
    hp = HotPath(1, lay.heads, lay.n, lay.head_dim, lay.block, lay.n_text, lay.text_first,
                 mode=ada.SELECT_RECALL, targets=args.recall, flags=ada.FLAG_TEXT_SINK)
    o_warm = torch.empty_like(q)

    def one(ev=None):
        rec = (lambda i: ev[i].record()) if ev else (lambda i: None)  # noqa: E731
        rec(0)
        hp.dense(q, k, v, o=o_warm)
        rec(1)
        hp.search(q, k, v, fused=True)
        rec(2)
        hp.sparse(q, k, v)
        rec(3)
        m2 = hp.cached_search(q, k)
        rec(4)
        hp.select(m2)
        rec(5)

    for _ in range(2):
        one()
    per = []
    for _ in range(reps):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(7)]
        one(ev)
        torch.cuda.synchronize()
        per.append({"K1": ev[0].elapsed_time(ev[1]), "FS": ev[1].elapsed_time(ev[2]), "K4": ev[2].elapsed_time(ev[3]),
                    "K2": ev[3].elapsed_time(ev[4]), "K3": ev[4].elapsed_time(ev[5])})
    med = {n: stats([p[n] for p in per])[0] for n in per[0]}
    kfl, nnz = kept_flops(lay, hp.csr, lay.head_dim)
    kern = kernel_entries(lay, hp.nb, nnz, kfl, med, peaks, traffic.get(name, {}), sm_mhz=sm_mhz)
    out = {"seq_len": lay.n, "heads": lay.heads, "head_dim": lay.head_dim, "block": lay.block,
           "selection": f"recall {args.recall} per head, text sink",
           "K4_tflops": kern["K4_block_sparse_attn"]["achieved"], "ms_per_layer_sparse": round(med["K4"], 3),
           "search_overhead_ms": round(med["FS"] - med["K1"], 3),
           "search_overhead_vs_dense": round((med["FS"] - med["K1"]) / med["K1"], 4),
           "search_overhead_cached_vs_dense": round((med["K2"] + med["K3"]) / med["K1"], 4),
           "t_w_step_ms": {"fused_one_call": round(med["FS"], 3),
                           "two_pass_k1_k2_k3": round(med["K1"] + med["K2"] + med["K3"], 3)},
           "dense_ms": round(med["K1"], 3),
           "kept_density": round(nnz / (lay.heads * hp.nb * hp.nb), 4), "kernels": kern}
    del q, k, v, hp
    torch.cuda.empty_cache()
    return out


def run_ours(args):
    """One layer per job; rank p runs the search on its contiguous head group and K4 on its K4 head
    set (the same group, or the LPT set with --lpt).  value = the layer's kept FLOPs / the slowest
    rank's K4 time (strong scaling; at N=1 the whole layer on one GPU)."""
    ws, rank, local = dist_env()
    init_dist(ws, local)
    import workloads
    import paper_2502_21079_b200 as ada
    from paper_2502_21079_b200 import dist as D
    from paper_2502_21079_b200.hotpath import HotPath

    lay = workloads.layout_for(args.config)
    dev = torch.device("cuda", torch.cuda.current_device())
    H, N, d = lay.heads, lay.n, lay.head_dim
    if H < ws:
        raise SystemExit(f"{H} heads cannot be sharded over {ws} ranks")
    h0, h1 = D.head_range(H, ws, rank)
    Hl = h1 - h0
    full = workloads.generate_qkv(lay, device=dev)          # the same layer on every rank (same seed)
    if ws == 1:
        q, k, v = full
    else:
        q, k, v = (x[:, h0:h1].contiguous() for x in full)
    if not args.lpt:
        del full
        torch.cuda.empty_cache()
    if args.mode == "recall":
        hp = HotPath(1, Hl, N, d, lay.block, lay.n_text, lay.text_first,
                     mode=ada.SELECT_RECALL, targets=args.recall, flags=ada.FLAG_TEXT_SINK)
    else:
        hp = HotPath(1, Hl, N, d, lay.block, lay.n_text, lay.text_first,
                     mode=ada.SELECT_SPARSITY, targets=0.8, flags=ada.FLAG_TEXT_SINK | ada.FLAG_HEAD_TIERS)
    nb = hp.nb

    # K4 head set: the search group, or (--lpt) an LPT set by kept tiles from the first search
    hp.search(q, k, v)
    grp, gci = D.gather_csr(hp.csr.row_ptr, hp.csr.col_idx)
    costs = D.head_nnz(grp, nb)                              # kept tiles per head, whole layer
    contig = D.contiguous_assign(H, ws)
    assign = D.lpt_assign(costs, ws) if args.lpt else contig
    mine = assign[rank]
    if args.lpt:
        idx = torch.tensor(mine, device=dev)
        q4, k4, v4 = (x.index_select(1, idx).contiguous() for x in full)
        del full
        torch.cuda.empty_cache()
        o4 = torch.empty_like(q4)
        ws4 = torch.empty(max(ada.sparse_workspace_bytes(ada.make_desc(q4, lay.block, lay.n_text,
                                                                        lay.text_first)), 1),
                          dtype=torch.uint8, device=dev)

    o_warm = torch.empty_like(q)
    lse_warm = torch.empty(1, Hl, N, dtype=torch.float32, device=dev)

    # One step exercises every row of the path, in schedule order:
    #   K1 (a warm-up step: dense attention + LSE) | the search step t_w in one C-ABI call
    #   (adaspa_search_select: the dense pass with block LSEs, the block masses with the fresh LSE and,
    #   per q-block row in the same CTA, the RECALL selection; then the CSR) | [--lpt: CSR exchange] |
    #   K4 (a sparse step on the cached CSR) | K2 + K3 (a later key step: block masses with the cached
    #   t_w LSE, Alg. 2, then the selection on them)
    # events: 0 K1 1 t_w 2 exchange 3 K4 4 K2 5 K3 6
    def step(ev=None):
        rec = (lambda i: ev[i].record()) if ev else (lambda i: None)  # noqa: E731
        rec(0)
        hp.dense(q, k, v, o=o_warm, lse=lse_warm)
        rec(1)
        hp.search(q, k, v, fused=True)
        rec(2)
        if args.lpt:
            rp, ci = D.gather_csr(hp.csr.row_ptr, hp.csr.col_idx)
            prp, pci = D.pack_heads_csr(rp, ci, mine, nb)
            rec(3)
            ada.block_sparse_attn(q4, k4, v4, prp, pci, block_size=lay.block, n_text=lay.n_text,
                                  text_first=lay.text_first, o=o4, workspace=ws4)
            step.csr = _Csr(prp, pci)
        else:
            rec(3)
            hp.sparse(q, k, v)
            step.csr = hp.csr
        rec(4)
        m2 = hp.cached_search(q, k)
        rec(5)
        hp.select(m2)
        rec(6)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    K = args.steps
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(7)] for _ in range(K)]
    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    clk = ClockSampler(dev.index)
    t_wall = time.perf_counter()
    for s in range(K):
        step(ev[s])
    torch.cuda.synchronize()
    wall = time.perf_counter() - t_wall
    if ws > 1:
        torch.distributed.barrier()
    clocks = clk.stop()
    # per step: K1, t_w search step, exchange, K4, K2 (cached LSE), K3, total -- each the max over ranks
    NP = 7
    per = [[e[0].elapsed_time(e[1]), e[1].elapsed_time(e[2]), e[2].elapsed_time(e[3]), e[3].elapsed_time(e[4]),
            e[4].elapsed_time(e[5]), e[5].elapsed_time(e[6]), e[0].elapsed_time(e[6])] for e in ev]
    flat = D.reduce_max([x for p in per for x in p])
    per = [flat[NP * s:NP * s + NP] for s in range(K)]
    tot = [sum(p[i] for p in per) for i in range(NP)]
    med = [stats([p[i] for p in per])[0] for i in range(NP)]
    p90 = [stats([p[i] for p in per])[1] for i in range(NP)]
    I_K1, I_FS, I_X, I_K4, I_K2, I_K3, I_TOT = range(NP)
    kfl, nnz = kept_flops(lay, step.csr, d)
    kfl_all, nnz_all = D.reduce_sum([kfl, nnz])
    value = kfl_all * K / (tot[I_K4] / 1e3) / 1e12
    loads = [x[0] for x in D.all_gather_floats([nnz])]
    imb_contig = D.imbalance(costs, contig)[0]
    flush = l2_flush_buffer(dev)
    k3_cold = D.reduce_max([time_k3_cold(hp, flush)])[0]
    del flush

    # e2e: the same metric (K4 TFLOP/s on kept blocks) for a sparse step end to end through the public
    # API from pinned host buffers: H2D of Q,K,V, the block-sparse forward on the cached CSR, D2H of O,
    # pipelined over head groups (HotPath.run_sparse_host), on this rank's search head group
    e2e = None
    if not args.no_e2e:
        qh, kh, vh = (x.cpu().pin_memory() for x in (q, k, v))
        oh = torch.empty_like(qh).pin_memory()
        from paper_2502_21079_b200.hotpath import tapered_groups
        groups = tapered_groups(Hl)
        for _ in range(2):
            hp.run_sparse_host(qh, kh, vh, oh, groups=groups)
        torch.cuda.synchronize()
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if ws > 1:
            torch.distributed.barrier()
        s0.record()
        for _ in range(K):
            hp.run_sparse_host(qh, kh, vh, oh, groups=groups)
        s1.record()
        torch.cuda.synchronize()
        te = D.reduce_max([s0.elapsed_time(s1)])[0]
        kfl_c = D.reduce_sum([kept_flops(lay, hp.csr, d)[0]])[0]
        e2e = {"value": round(kfl_c * K / (te / 1e3) / 1e12, 3), "unit": UNIT,
               "h2d_bytes_per_step": 3 * q.numel() * q.element_size() * ws,
               "d2h_bytes_per_step": q.numel() * q.element_size() * ws,
               "ms_per_step": round(te / K, 3),
               "note": f"sparse step from pinned host memory: H2D Q,K,V + K4 (cached CSR) + D2H O per rank "
                       f"(its search head group), overlapped over {len(groups)} head groups of {groups} heads, K4 "
                       "launches alternating between two compute streams; PCIe-bound (2.06 GB of pinned H2D "
                       "and 0.69 GB of D2H per HYV-110K layer: 38.9 ms for both at once on the box, "
                       "tools/pcie_probe.py); TFLOP/s on kept blocks, whole job"}
        del qh, kh, vh, oh

    peaks, src = load_peaks()
    # ncu DRAM bytes per launch were captured on the HYV-110K step (profiles/ncu_traffic.json top
    # level); other configs report them only if captured for that config (a sub-dict by name)
    traffic = load_traffic()
    if args.config != "hyv110k":
        traffic = traffic.get(args.config, {}) if isinstance(traffic.get(args.config), dict) else {}
    launches = (hp.kernels_per_run() + 2 + 4) * K   # + K1 alone, K2 (cached LSE) and K3 (4) per step
    variants = None
    if ws == 1 and not args.no_variants and args.config == "hyv110k":
        variants = {"hyv110k_sparsity0.8_tiers": variant_tiers(hp, q, k, v, lay, peaks)}
        del q, k, v, hp
        torch.cuda.empty_cache()
        variants["cogx45k_recall0.9"] = variant_config("cogx45k", args, peaks, traffic,
                                                       sm_mhz=(clocks or {}).get("sm_mhz"))
        variants.update(variant_schedule_and_sweep(args))
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        qc, kc, vc = workloads.generate_qkv(lay, device=dev)
        cpu = cpu_baseline_sample(lay, qc, kc, vc, step.csr, args.cpu_seconds)

    if rank != 0:
        if ws > 1:
            torch.distributed.destroy_process_group()
        return
    ms = [x / K for x in tot]
    h_max = -(-H // ws)            # K1-K3 times are the slowest rank's, i.e. one with ceil(H/N) heads
    keys = {"K1": I_K1, "FS": I_FS, "K2": I_K2, "K3": I_K3, "K4": I_K4}
    kern = kernel_entries(lay, nb, nnz_all * h_max / H, kfl_all, {n: med[i] for n, i in keys.items()}, peaks,
                          traffic, p90={n: p90[i] for n, i in keys.items()}, heads=h_max,
                          sm_mhz=(clocks or {}).get("sm_mhz"))
    if ws > 1:   # K1-K3 achieved rates per rank's head group; K4 on the whole layer's kept FLOPs
        kern["K4_block_sparse_attn"] = roofline_entry("tensor", value, kern["K4_block_sparse_attn"]["peak"] * ws,
                                                      "TFLOP/s", None, ms=round(med[I_K4], 3),
                                                      ms_p90=round(p90[I_K4], 3), note=f"whole job, {ws} GPUs")
    kern["K3_select_blocks"]["ms_cold"] = round(k3_cold, 4)
    kern["K3_select_blocks"]["ms_warm"] = kern["K3_select_blocks"]["ms"]
    k3 = kern["K3_select_blocks"]
    k3["achieved_cold"] = round(k3["achieved"] * k3["ms"] / k3_cold, 3)
    dom_name = max(kern, key=lambda n: kern[n]["ms"])
    roof = dict(kern[dom_name])
    roof["kernel"] = dom_name
    roof["peak_source"] = f"{src} ({'bf16_tflops_sustained' if roof['bound'] == 'tensor' else 'see kernels'})"
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": ws, "steps": K, "warmup": args.warmup,
        "ms_per_step": round(ms[I_TOT], 3), "higher_is_better": True, "scaling": "strong" if ws > 1 else "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic (workloads/synth.py, seeded; DESIGN.md §5)",
        "config": {"workload": lay.name, "seq_len": N, "heads": H, "head_dim": d, "block": lay.block,
                   "n_text": lay.n_text, "selection": (f"recall {args.recall} per head, text sink"
                                                       if args.mode == "recall" else "sparsity 0.8 + head tiers"),
                   "parallelism": (f"head-sharded x{ws}" + (" + LPT K4 head sets" if args.lpt else "")
                                   if ws > 1 else "1 GPU, whole layer"),
                   "l2": "inputs larger than L2 (Q,K,V = %.2f GB per layer)" % (3 * N * H * d * 2 / 1e9)},
        "ms_per_layer_sparse": round(ms[I_K4], 3),
        # search overhead at t_w: what the whole search step (one call, selection included) adds to a
        # dense pass
        "search_overhead_ms": round(ms[I_FS] - ms[I_K1], 3),
        "search_overhead_vs_dense": round((tot[I_FS] - tot[I_K1]) / tot[I_K1], 4),
        # at a later key step (Alg. 2: no dense pass runs; K2 with the cached LSE, then K3)
        "search_overhead_cached_ms": round(ms[I_K2] + ms[I_K3], 3),
        "search_overhead_cached_vs_dense": round((tot[I_K2] + tot[I_K3]) / tot[I_K1], 4),
        "t_w_step_ms": {"fused_one_call": round(ms[I_FS], 3),
                        "two_pass_k1_k2_k3": round(ms[I_K1] + ms[I_K2] + ms[I_K3], 3)},
        "dense_ms": round(ms[I_K1], 3),
        "kept_density": round(nnz_all / (H * nb * nb), 4),
        "roofline": roof, "kernels": kern,
        "multi_gpu": {"k4_heads_per_rank": [len(a) for a in assign], "kept_tiles_per_rank": loads,
                      "kept_tile_imbalance": round(max(loads) / (sum(loads) / len(loads)), 4),
                      "contiguous_imbalance": round(imb_contig, 4),
                      "exchange_ms": round(ms[I_X], 3) if args.lpt else 0.0},
        "cpu_baseline": cpu, "e2e": e2e, "variants": variants,
        "gpu_launches": launches, "clocks": clocks,
        "wall_s_timed_region": round(wall, 3),
    }
    print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()


def run_ulysses(args):
    """configs[3]: ONE HunyuanVideo-shaped layer whose activations arrive sequence-sharded ([N/P, H, d]
    per rank, as a sequence-parallel DiT holds them).  A step = the search step t_w (NCCL all_to_all of
    Q, K, V to head shards [N, H_r, d] -> K1 -> K2 -> K3 on the local heads, read token-major through the
    descriptor strides with no unpack; all_to_all of O back) followed by a sparse step (all_to_all in,
    K4, all_to_all of O back).  --lpt: the sparse step's head sets are LPT by kept tiles (the a2a send
    order carries the permutation; the CSRs are all-gathered after the search).  value = kept FLOPs of
    the whole layer / max over ranks of the K4 time (strong scaling)."""
    ws, rank, local = dist_env()
    import torch.distributed as dist
    local = local_device(local)
    torch.cuda.set_device(local)
    if ws > 1:
        if os.environ.get("ADASPA_BENCH_BACKEND", "nccl") == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:   # plumbing check with ranks sharing a GPU (needs --p2p: gloo has no CUDA all_to_all)
            dist.init_process_group(os.environ["ADASPA_BENCH_BACKEND"])
    else:
        import socket
        so = socket.socket()
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
        so.close()
        dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                                device_id=torch.device("cuda", local))
    import workloads
    import paper_2502_21079_b200 as ada
    from paper_2502_21079_b200 import dist as D
    from paper_2502_21079_b200.hotpath import HotPath
    lay = workloads.layout_for(args.config)
    dev = torch.device("cuda", local)
    H, N, d = lay.heads, lay.n, lay.head_dim
    if H % ws:
        raise SystemExit(f"--ulysses needs heads ({H}) divisible by the world size ({ws})")
    Hp = H // ws
    sizes = D.seq_splits(N, ws)
    off = sum(sizes[:rank])
    q, k, v = workloads.generate_qkv(lay, device=dev)            # the global layer (same seed on every rank)
    loc = [x[0].transpose(0, 1)[off:off + sizes[rank]].contiguous() for x in (q, k, v)]   # [N_p, H, d]
    del q, k, v
    torch.cuda.empty_cache()
    hp = HotPath(1, Hp, N, d, lay.block, lay.n_text, lay.text_first, mode=ada.SELECT_RECALL,
                 targets=args.recall, flags=ada.FLAG_TEXT_SINK, token_major=True)
    nb = hp.nb
    kw = dict(block_size=lay.block, n_text=lay.n_text, text_first=lay.text_first)

    # the sparse step's head sets (LPT from a first search, or the contiguous groups)
    sh = [D.as_bhnd(D.ulysses_in(x, sizes=sizes)) for x in loc]
    hp.search(*sh)
    grp, gci = D.gather_csr(hp.csr.row_ptr, hp.csr.col_idx)
    costs = D.head_nnz(grp, nb)
    contig = D.contiguous_assign(H, ws)
    assign = D.lpt_assign(costs, ws) if args.lpt else contig
    mine = assign[rank]
    del sh
    ws4 = None
    ex_s = ex_4 = None
    if args.p2p:   # peer-memory exchange: one for the search step's head groups, one for the sparse step's
        ex_s = D.PeerExchange(N, H, d, sizes, contig, dev)
        ex_4 = D.PeerExchange(N, H, d, sizes, assign, dev)

    def a2a_in(ex, asg):
        if ex is None:
            return [D.as_bhnd(D.ulysses_in(x, sizes=sizes, assign=asg)) for x in loc]
        ex.push_in(loc)
        return [D.as_bhnd(x) for x in ex.wait_in()]

    def a2a_out(ex, o_tok, asg):
        if ex is None:
            return D.ulysses_out(o_tok, sizes, assign=asg)
        ex.push_out(o_tok)
        out = ex.wait_out()
        ex.release_out()
        return out

    def step(ev=None):
        rec = (lambda i: ev[i].record()) if ev else (lambda i: None)  # noqa: E731
        nonlocal ws4
        rec(0)
        sh = a2a_in(ex_s, contig)                                               # [1, Hp, N, d] token-major views
        rec(1)
        hp.search(*sh, events=ev[1:5] if ev else None)
        if ex_s is not None:
            ex_s.release_in()
        o_d = a2a_out(ex_s, hp.o_dense[0].transpose(0, 1), contig)              # O of the search step back
        rec(5)
        if args.lpt:
            rp, ci = D.gather_csr(hp.csr.row_ptr, hp.csr.col_idx)
            csr = _Csr(*D.pack_heads_csr(rp, ci, mine, nb))
        else:
            csr = hp.csr
        rec(6)
        s4 = a2a_in(ex_4, assign)                                               # sparse step's a2a in
        rec(7)
        if ws4 is None:
            ws4 = torch.empty(max(ada.sparse_workspace_bytes(ada.make_desc(s4[0], **kw)), 1), dtype=torch.uint8,
                              device=dev)
        o4 = torch.empty(1, N, len(mine), d, dtype=s4[0].dtype, device=dev).transpose(1, 2)   # token-major
        ada.block_sparse_attn(*s4, csr.row_ptr, csr.col_idx, o=o4, workspace=ws4, **kw)
        if ex_4 is not None:
            ex_4.release_in()
        rec(8)
        o_s = a2a_out(ex_4, o4[0].transpose(0, 1), assign)
        rec(9)
        step.csr = csr
        return o_d, o_s

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    K = args.steps
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(10)] for _ in range(K)]
    dist.barrier()
    torch.cuda.synchronize()
    clk = ClockSampler(dev.index)
    for i in range(K):
        step(evs[i])
    torch.cuda.synchronize()
    dist.barrier()
    clocks = clk.stop()
    # phases: a2a in (search), the search step (one call: dense pass, block masses + selection, CSR;
    # phases 2-3 are empty then), a2a out (search O), exchange, a2a in (sparse), K4, a2a out
    per = [[e[i].elapsed_time(e[i + 1]) for i in range(9)] for e in evs]
    flat = D.reduce_max([x for p in per for x in p])
    per = [flat[9 * s:9 * s + 9] for s in range(K)]
    tot = [sum(p[i] for p in per) for i in range(9)]
    kfl, nnz = kept_flops(workloads.layout_for(args.config, heads=len(mine)), step.csr, d)
    kfl_all, nnz_all = D.reduce_sum([kfl, nnz])
    loads = [x[0] for x in D.all_gather_floats([nnz])]
    if rank == 0:
        ms = [x / K for x in tot]
        line = {
            "metric": METRIC, "value": round(kfl_all * K / (tot[7] / 1e3) / 1e12, 3), "unit": UNIT,
            "n_gpus": ws, "steps": K, "warmup": args.warmup, "ms_per_step": round(sum(ms), 3),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (workloads/synth.py, seeded; DESIGN.md §5)",
            "config": {"workload": lay.name + "-ulysses", "seq_len": N, "heads": H, "heads_per_rank": Hp,
                       "head_dim": d, "block": lay.block,
                       "parallelism": f"ulysses a2a x{ws} " + ("(peer memory: IPC + copy engines)" if args.p2p else "(NCCL)")
                                      + (" + LPT sparse-step head sets" if args.lpt else ""),
                       "l2": "inputs larger than L2"},
            "ms_per_layer_sparse": round(ms[7], 3), "t_w_search_step_ms": round(ms[1] + ms[2] + ms[3], 3),
            "a2a_ms": {"search_in": round(ms[0], 3), "search_out": round(ms[4], 3), "sparse_in": round(ms[6], 3),
                       "sparse_out": round(ms[8], 3)},
            "exchange_ms": round(ms[5], 3),
            "kept_density": round(nnz_all / (H * nb * nb), 4),
            "multi_gpu": {"k4_heads_per_rank": [len(a) for a in assign], "kept_tiles_per_rank": loads,
                          "kept_tile_imbalance": round(max(loads) / (sum(loads) / len(loads)), 4),
                          "contiguous_imbalance": round(D.imbalance(costs, contig)[0], 4)},
            "gpu_launches": (hp.kernels_per_run()) * K, "clocks": clocks,
            "note": "times are max over ranks per phase; value uses the max-over-ranks K4 time",
        }
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()


def run_reference(args):
    """The oracle as the reference arm: each step runs the fp64 oracle hot path (dense attention ->
    block mass -> recall selection -> masked attention) for a bounded sample of q-blocks of head 0."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    import numpy as np
    import oracle
    import workloads
    lay = workloads.layout_for(args.config)
    dev = "cuda" if torch.cuda.is_available() else "cpu"
    q, k, v = workloads.generate_qkv(lay, device=dev)
    qh, kh, vh = (x[0, 0].float().double().cpu().numpy() for x in (q, k, v))
    del q, k, v
    blocks = oracle.block_map(lay.n_video, lay.n_text, lay.block, lay.text_first)
    nb = len(blocks)
    scale = 1.0 / math.sqrt(lay.head_dim)
    try:
        from threadpoolctl import threadpool_info
        cores = max((i.get("num_threads", 1) for i in threadpool_info()), default=os.cpu_count())
    except Exception:  # noqa: BLE001
        cores = os.cpu_count()
    per_step = 3
    stride = max(1, nb // 97)

    def step(i):
        ids = [((i * per_step + j) * stride) % nb for j in range(per_step)]
        fl, t_sparse = 0.0, 0.0
        for p in ids:
            b = blocks[p]
            rows = slice(b.start, b.start + b.length)
            _, lse = oracle.dense_attention(qh[rows], kh, vh, scale)
            lse_full = np.zeros(lay.n)
            lse_full[rows] = lse
            M = oracle.block_mass(qh, kh, lse_full, blocks, scale, q_block_ids=[p])[0]
            forced, cands = oracle.row_forced_and_candidates(blocks, p, True)
            kept = oracle.select_row_recall(M, forced, cands, args.recall)
            t0 = time.perf_counter()
            oracle.masked_attention(qh, kh, vh, blocks, {p: kept}, scale, q_block_ids=[p])
            t_sparse += time.perf_counter() - t0
            fl += 4.0 * lay.head_dim * b.length * sum(blocks[j].length for j in kept)
        return fl, t_sparse

    for i in range(args.warmup):
        step(i)
    fl, ts, t0 = 0.0, 0.0, time.perf_counter()
    for i in range(args.steps):
        a, b = step(args.warmup + i)
        fl += a
        ts += b
    wall = time.perf_counter() - t0
    val = fl / ts / 1e12
    sample = (f"oracle hot path (fp64 numpy: dense+LSE, block mass, recall {args.recall} selection, masked "
              f"attention) on {per_step} q-blocks of head 0 per step at {lay.name}; value = masked-attention "
              f"TFLOP/s on kept blocks")
    line = {
        "impl": "reference", "metric": METRIC, "value": round(val, 6), "unit": UNIT, "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(wall / args.steps * 1e3, 1),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (workloads/synth.py, seeded)",
        "config": {"workload": lay.name, "seq_len": lay.n, "heads": lay.heads, "head_dim": lay.head_dim,
                   "block": lay.block, "selection": f"recall {args.recall} per head, text sink"},
        "cpu_baseline": {"value": round(val, 6), "unit": UNIT, "cores": int(cores), "kind": "oracle",
                         "sample": sample},
        "e2e": {"value": round(val, 6), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    rc = maybe_spawn(args)
    if rc is not None:
        sys.exit(rc)
    if args.impl == "reference":
        run_reference(args)
    elif args.ulysses:
        run_ulysses(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
