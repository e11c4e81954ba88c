"""Synthetic Q/K/V shaped like the paper's workloads.

Geometry (eq:seqlen, L = f*h*w + t):
  tiny      f=7,  h=8,  w=8  (448 video) + 64 text,  H=2,  d=64,  B=64
  cogx45k   f=11, h=48, w=85 (44,880)    + 226 text, H=48, d=64,  B=64,  text first
  hyv110k   f=31, h=45, w=80 (111,600)   + 256 text, H=24, d=128, B=128, text last
  hyv129f   f=33, h=45, w=80 (118,800)   + 256 text, H=24, d=128, B=128, text last

Value structure mirrors what PAPER.md:253 and 295-334 (Obs. 1) describe --
frame-region hierarchy, a text sink and per-head variable concentration:
  z_video = normalize(0.8 U_frame[t] + 1.0 U_tile[y//4, x//8] + 0.6 e)
  q_h = A_h d^(1/4) z R_h + 0.5 eps + 0.5 d^(1/4) u_sink
  k_h = A_h d^(1/4) normalize(z + 0.3 eps'/sqrt(d)) R_h + 0.5 eps  (+ 2 d^(1/4) u_sink on text keys)
  v   = N(0,1) clipped to +-4
with R_h a seeded random rotation and A_h a seeded permutation of
linspace(sharp_lo, sharp_hi, H).  Everything is rounded to bf16.  Drift for the
multi-step schedule: x_t = sqrt(1-sigma^2) x_base + sigma * rms(x_base) * noise_t,
noise seeded with step_seed(t).

None of the method's arithmetic (softmax, LSE, block mass, selection) is here.
"""

import math
from dataclasses import dataclass

import torch

BASE_SEED = 21079


@dataclass(frozen=True)
class Layout:
    name: str
    f: int
    h: int
    w: int
    n_text: int
    text_first: bool
    heads: int
    head_dim: int
    block: int

    @property
    def n_video(self):
        return self.f * self.h * self.w

    @property
    def n(self):
        return self.n_video + self.n_text


# per-head sharpness range A_h (calibrated so that recall 0.9 keeps a mean block density
# near the paper's default 1 - sparsity = 0.2 with a >= 5x spread across heads)
SHARP = {"hyv110k": (2.75, 5.5), "hyv129f": (2.75, 5.5), "cogx45k": (2.75, 5.5)}

CONFIGS = {
    "tiny": Layout("tiny", 7, 8, 8, 64, False, 2, 64, 64),
    "tiny_tf": Layout("tiny_tf", 7, 8, 8, 64, True, 2, 64, 64),
    "cogx45k": Layout("cogx45k", 11, 48, 85, 226, True, 48, 64, 64),
    "hyv110k": Layout("hyv110k", 31, 45, 80, 256, False, 24, 128, 128),
    "hyv129f": Layout("hyv129f", 33, 45, 80, 256, False, 24, 128, 128),
}


def layout_for(name, **over):
    lay = CONFIGS[name]
    if over:
        d = dict(lay.__dict__)
        d.update(over)
        lay = Layout(**d)
    return lay


def step_seed(step, base=BASE_SEED):
    return base + 1000 * int(step)


def sharpness(heads, seed=BASE_SEED, lo=1.5, hi=4.0):
    g = torch.Generator().manual_seed(seed + 17)
    vals = torch.linspace(lo, hi, heads, dtype=torch.float64)
    return vals[torch.randperm(heads, generator=g)].tolist()


def _unit(x):
    return x / x.norm(dim=-1, keepdim=True).clamp_min(1e-12)


def _video_latent(lay, d, g, device):
    f, h, w = lay.f, lay.h, lay.w
    u_frame = _unit(torch.randn(f, d, generator=g, device=device))
    th, tw = -(-h // 4), -(-w // 8)
    u_tile = _unit(torch.randn(th * tw, d, generator=g, device=device))
    t_idx = torch.arange(f, device=device).repeat_interleave(h * w)
    y_idx = torch.arange(h, device=device).repeat_interleave(w).repeat(f)
    x_idx = torch.arange(w, device=device).repeat(f * h)
    tile = (y_idx // 4) * tw + (x_idx // 8)
    e = torch.randn(f * h * w, d, generator=g, device=device) / math.sqrt(d)
    return _unit(0.8 * u_frame[t_idx] + 1.0 * u_tile[tile] + 0.6 * e)


def generate_qkv(lay, batch=1, seed=BASE_SEED, device="cpu", sharp=None, sigma=0.0,
                 step=0, heads=None, dtype=torch.bfloat16):
    """Q, K, V as bf16 [batch, H, N, d] (contiguous).  `heads` overrides lay.heads
    (e.g. a head shard).  Deterministic for a given (device type, arguments)."""
    H = lay.heads if heads is None else heads
    d = lay.head_dim
    N = lay.n
    c = d ** 0.25
    out = [torch.empty(batch, H, N, d, dtype=dtype, device=device) for _ in range(3)]
    if sharp is None:
        sharp = SHARP.get(lay.name.split("_")[0], (1.5, 4.0))
    amps = sharpness(H, seed, *sharp)
    for b in range(batch):
        g = torch.Generator(device=device)
        g.manual_seed(seed + 7919 * b)
        zv = _video_latent(lay, d, g, device)
        zt = _unit(torch.randn(lay.n_text, d, generator=g, device=device))
        z = torch.cat([zt, zv]) if lay.text_first else torch.cat([zv, zt])
        is_text = torch.zeros(N, dtype=torch.bool, device=device)
        if lay.text_first:
            is_text[: lay.n_text] = True
        else:
            is_text[lay.n_video:] = True
        u_sink = _unit(torch.randn(d, generator=g, device=device))
        for h in range(H):
            rot, _ = torch.linalg.qr(torch.randn(d, d, generator=g, device=device))
            a = amps[h]
            zk = _unit(z + 0.3 * torch.randn(N, d, generator=g, device=device) / math.sqrt(d))
            q = a * c * (z @ rot) + 0.5 * torch.randn(N, d, generator=g, device=device) + 0.5 * c * u_sink
            k = a * c * (zk @ rot) + 0.5 * torch.randn(N, d, generator=g, device=device)
            k[is_text] += 2.0 * c * u_sink
            v = torch.randn(N, d, generator=g, device=device).clamp_(-4.0, 4.0)
            if sigma > 0.0:
                gs = torch.Generator(device=device)
                gs.manual_seed(step_seed(step, seed) + 31 * (b * H + h))
                keep = math.sqrt(1.0 - sigma * sigma)
                q = keep * q + sigma * q.pow(2).mean().sqrt() * torch.randn(N, d, generator=gs, device=device)
                k = keep * k + sigma * k.pow(2).mean().sqrt() * torch.randn(N, d, generator=gs, device=device)
                v = (keep * v + sigma * torch.randn(N, d, generator=gs, device=device)).clamp_(-4.0, 4.0)
            out[0][b, h] = q.to(dtype)
            out[1][b, h] = k.to(dtype)
            out[2][b, h] = v.to(dtype)
    return tuple(out)


def random_masses(rows, nb, seed=BASE_SEED, ties=True, dtype=torch.float32):
    """Block-mass-like rows for selection-only tests: heavy-tailed positive
    values (a few dominant blocks per row, like a concentrated head), with
    optional exact ties so the (mass desc, index asc) rule is exercised."""
    g = torch.Generator().manual_seed(seed)
    u = torch.rand(rows, nb, generator=g, dtype=torch.float64).clamp_min(1e-300)
    conc = torch.rand(rows, 1, generator=g, dtype=torch.float64) * 6.0 + 0.5
    x = (-torch.log(u)) ** conc
    if ties and nb >= 4:
        j = torch.randint(0, nb, (rows, 3), generator=g)
        x[torch.arange(rows)[:, None], j] = x[torch.arange(rows)[:, None], j[:, :1]]
    return x.to(dtype)
