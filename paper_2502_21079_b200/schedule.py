"""Host schedule and per-layer caches of AdaSpa.

PAPER.md:397-405 (fig:overview caption): warm-up steps run full attention; the first key step
t_key^1 = t_w runs the Fused Online Search (Alg. 1: dense attention that also emits the LSE, then
the block mass with that fresh LSE, PAPER.md:459-497 -- here ONE C-ABI call, adaspa_search_select:
one dense pass that also emits the per-(row, kv block) log-sum-exps, the block masses whose CTAs
select their q-block row (RECALL), the CSR; SPARSITY / tiers: adaspa_dense_attn_lse_search then K3;
fused_search=False: K1, K2, K3); every later key step runs the LSE-Cached
Online Search (Alg. 2) with the LSE cached at t_w; all other steps after t_w run
the head-adaptive block-sparse attention with the cached index lists.
Defaults: T_s = {10, 30}, 10 warm-up steps, 50 steps.
Readings R18 (a later key step uses its new mask on the same step) and R19 (the t_w LSE is never
refreshed) of DESIGN.md §3.

Nothing here computes: every step is one or more C-ABI calls (K1..K4) on the caller's stream,
and the caches are device tensors owned by this object (the library allocates nothing).
"""

from . import _lib as L

FULL = "full"
FULL_SEARCH = "full+search"
SPARSE = "sparse"
CACHED_SEARCH_SPARSE = "cached-search+sparse"


def step_mode(t, t_w, key_steps):
    """Mode of 1-indexed step t."""
    ks = sorted(set(int(x) for x in key_steps))
    if not ks or ks[0] != t_w:
        raise ValueError("the first key step must equal t_w (PAPER.md:400, t_key^1 = t_w)")
    if t < t_w:
        return FULL
    if t == t_w:
        return FULL_SEARCH
    if t in ks:
        return CACHED_SEARCH_SPARSE
    return SPARSE


def trace(n_steps, t_w, key_steps):
    if max(key_steps) > n_steps or t_w < 1:
        raise ValueError("key steps out of range")
    return [step_mode(t, t_w, key_steps) for t in range(1, n_steps + 1)]


class LayerCache:
    """Per-layer state kept across denoising steps: the t_w LSE and the current CSR."""

    def __init__(self, desc, device, torch):
        B, H, N = desc.batch, desc.heads, desc.seq_len
        nb = L.num_blocks(desc)
        e = lambda *s, dt: torch.empty(*s, dtype=dt, device=device)  # noqa: E731
        self.lse = e(B, H, N, dt=torch.float32)
        self.mass = e(B, H, nb, nb, dt=torch.float32)
        rows = B * H * nb
        self.csr = L.Csr(e(rows + 1, dt=torch.int32), e(rows * nb, dt=torch.int32), e(rows, dt=torch.int32),
                         e(B, H, dt=torch.float32), e(B, H, dt=torch.int64))
        self.ws = e(max(L.sparse_workspace_bytes(desc), 1), dt=torch.uint8)
        self.have_lse = False
        self.have_mask = False


class AdaSpaSchedule:
    """Drives one or more attention layers through the AdaSpa step schedule.

    attention(layer, t, q, k, v) returns O for 1-indexed step t.  q/k/v are bf16 CUDA tensors
    viewed as [B, H, N, d] (any strides with a contiguous head dim; the same layout for all three).
    `targets` is one value or one per head: a recall r_h (RECALL mode, the north_star's primary
    mode) or a sparsity s_h (SPARSITY mode, optionally with FLAG_HEAD_TIERS).
    """

    def __init__(self, *, block_size, n_text, text_first=False, n_steps=50, t_w=10, key_steps=(10, 30),
                 mode=L.SELECT_RECALL, targets=0.9, flags=L.FLAG_TEXT_SINK, tier_tau=0.8, softmax_scale=0.0,
                 fused_search=True, fused_heads_per_pass=0):
        self.kw = dict(block_size=block_size, n_text=n_text, text_first=text_first, softmax_scale=softmax_scale)
        self.n_steps, self.t_w = int(n_steps), int(t_w)
        self.key_steps = sorted(set(int(x) for x in key_steps))
        trace(self.n_steps, self.t_w, self.key_steps)  # validates
        self.mode, self.flags, self.tier_tau = mode, flags, tier_tau
        self.targets = targets
        self.layers = {}
        self.calls = []  # (t, layer, mode) log, for tests and reports
        self.fused_search = fused_search
        self.fused_heads_per_pass = fused_heads_per_pass   # 0: all heads in one pass
        self._fws = None   # fused-search scratch, shared by all layers (the library allocates nothing)

    def _targets(self, H):
        if isinstance(self.targets, (int, float)):
            return [float(self.targets)] * H
        t = [float(x) for x in self.targets]
        if len(t) != H:
            raise ValueError(f"need {H} per-head targets")
        return t

    def cache(self, layer):
        return self.layers.get(layer)

    def _search(self, c, desc, q, k):
        L.lse_cached_search(q, k, c.lse, block_mass=c.mass, **self.kw)
        L.select_blocks(c.mass, heads_desc=desc, mode=self.mode, target=self._targets(desc.heads), flags=self.flags,
                        tier_tau=self.tier_tau, out=c.csr)
        c.have_mask = True

    def attention(self, layer, t, q, k, v, o=None):
        import torch
        mode = step_mode(t, self.t_w, self.key_steps)
        desc = L.make_desc(q, self.kw["block_size"], self.kw["n_text"], self.kw["text_first"],
                           self.kw["softmax_scale"])
        c = self.layers.get(layer)
        if c is None:
            c = self.layers[layer] = LayerCache(desc, q.device, torch)
        if o is None:
            o = torch.empty_like(q)
        self.calls.append((t, layer, mode))
        if mode == FULL:
            L.dense_attn_lse(q, k, v, o=o, want_lse=False, **self.kw)
        elif mode == FULL_SEARCH:
            if self.fused_search:                                    # Alg. 1 in one dense pass
                need = L.search_select_workspace_bytes(desc, self.fused_heads_per_pass)
                if self._fws is None or self._fws.numel() < need:
                    self._fws = torch.empty(need, dtype=torch.uint8, device=q.device)
                if self.mode == L.SELECT_RECALL and not (self.flags & L.FLAG_HEAD_TIERS):
                    # the whole search step, selection epilogue included; λ from t_w becomes the cache (R19)
                    L.search_select(q, k, v, target=self._targets(desc.heads), flags=self.flags, o=o, lse=c.lse,
                                    block_mass=c.mass, out=c.csr, workspace=self._fws, **self.kw)
                else:
                    L.dense_attn_lse_search(q, k, v, o=o, lse=c.lse, block_mass=c.mass, workspace=self._fws,
                                            **self.kw)               # λ from t_w becomes the cache (R19)
                    L.select_blocks(c.mass, heads_desc=desc, mode=self.mode, target=self._targets(desc.heads),
                                    flags=self.flags, tier_tau=self.tier_tau, out=c.csr)
                c.have_lse = True
                c.have_mask = True
            else:
                L.dense_attn_lse(q, k, v, o=o, lse=c.lse, **self.kw)   # λ from t_w becomes the cache (R19)
                c.have_lse = True
                self._search(c, desc, q, k)                              # Alg. 1 second pass, fresh λ
        else:
            if not c.have_mask:
                raise RuntimeError(f"layer {layer}: step {t} needs the mask of step t_w={self.t_w}")
            if mode == CACHED_SEARCH_SPARSE:
                self._search(c, desc, q, k)                          # Alg. 2 with the t_w λ (R19)
            L.block_sparse_attn(q, k, v, c.csr.row_ptr, c.csr.col_idx, o=o, workspace=c.ws, **self.kw)  # R18
        return o
