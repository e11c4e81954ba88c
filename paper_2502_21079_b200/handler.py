"""Plug-and-play attention handler: the paper's `adaspa_attention_handler` (PAPER.md:126, 545-546:
"users can enable AdaSpa with only a one-line change").

    attn = adaspa_attention_handler(num_layers=L, n_text=256)   # once per generation
    ...
    o = attn(q, k, v)                                           # in each attention layer

Defaults are the paper's: sparsity 0.8, block 64, T_s = {10, 30}, the first 10
steps dense (t_w = 10), Text Sink and Row Wise on, head-adaptive sparsity tiers
(PAPER.md:527-533); `mode="recall"` selects the north_star's per-head recall target instead.

The c-th call is layer c % L of step (c // L) % n_steps + 1 unless the caller passes step/layer; a
new generation starts after n_steps * L calls (the caches are rebuilt at its t_w).  Q/K/V are
[B, H, N, d] (layout="bhnd") or [B, N, H, d] (layout="bnhd", the usual DiT layout; read through
strides, no copy); O comes back in the same layout.  Everything is the C ABI through
schedule.AdaSpaSchedule; nothing here computes.
"""

import torch

from . import _lib as L
from . import schedule as S


class AdaSpaAttentionHandler:
    def __init__(self, num_layers, *, n_text, text_first=False, block_size=64, mode="sparsity", sparsity=0.8,
                 recall=0.9, head_adaptive=True, text_sink=True, n_steps=50, warmup=10, key_steps=(10, 30),
                 tier_tau=0.8, softmax_scale=0.0, layout="bhnd"):
        if num_layers < 1:
            raise ValueError("num_layers must be >= 1")
        if layout not in ("bhnd", "bnhd"):
            raise ValueError("layout is 'bhnd' ([B,H,N,d]) or 'bnhd' ([B,N,H,d])")
        if mode not in ("sparsity", "recall"):
            raise ValueError("mode is 'sparsity' (paper) or 'recall' (north_star)")
        key_steps = sorted(set(int(x) for x in key_steps))
        if not key_steps or key_steps[0] != warmup:
            raise ValueError("the first key step is the end of the warm-up (t_key^1 = t_w, PAPER.md:400)")
        flags = L.FLAG_TEXT_SINK if text_sink else 0
        if mode == "sparsity" and head_adaptive:
            flags |= L.FLAG_HEAD_TIERS
        self.num_layers = int(num_layers)
        self.layout = layout
        self.schedule = S.AdaSpaSchedule(
            block_size=block_size, n_text=n_text, text_first=text_first, n_steps=n_steps, t_w=warmup,
            key_steps=key_steps, mode=L.SELECT_SPARSITY if mode == "sparsity" else L.SELECT_RECALL,
            targets=sparsity if mode == "sparsity" else recall, flags=flags, tier_tau=tier_tau,
            softmax_scale=softmax_scale)
        self.calls = 0

    def position(self, call=None):
        """(step, layer) of call number `call` (default: the next call), 1-indexed step."""
        c = self.calls if call is None else int(call)
        return (c // self.num_layers) % self.schedule.n_steps + 1, c % self.num_layers

    def mode_of(self, step):
        return S.step_mode(step, self.schedule.t_w, self.schedule.key_steps)

    def __call__(self, q, k, v, *, step=None, layer=None):
        if (step is None) != (layer is None):
            raise ValueError("pass both step and layer, or neither")
        if step is None:
            step, layer = self.position()
        self.calls += 1
        if self.layout == "bnhd":
            q, k, v = (x.transpose(1, 2) for x in (q, k, v))
        o = self.schedule.attention(layer, step, q, k, v, o=torch.empty_like(q))
        return o.transpose(1, 2) if self.layout == "bnhd" else o


adaspa_attention_handler = AdaSpaAttentionHandler  # the paper's name
