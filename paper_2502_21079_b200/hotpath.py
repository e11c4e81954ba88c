"""One pass of the AdaSpa hot path on fixed shapes:

    search step t_w (Alg. 1):  K1 dense attention + LSE + block mass with that LSE  ->  K3 selection
    every later step:          K4 block-sparse forward on the cached CSR
    later key steps (Alg. 2):  K2 block mass with the cached LSE  ->  K3

`search(fused=True)` runs the whole search step t_w in ONE C-ABI call (adaspa_search_select): one
dense pass that also emits per-(row, kv block) log-sum-exps, then an HBM-bound block-mass reduction
whose CTAs select their q-block row (RECALL) before the CSR is assembled; `search(fused="mass")` runs
the fused dense pass + block masses (adaspa_dense_attn_lse_search) then K3; `search(fused=False)`
runs K1, K2 with the fresh LSE, K3.  Buffers are allocated once;
`run()` accepts device tensors or (pinned) host tensors, in which case it stages them to the
device on the same stream; `run_sparse_host()` is a sparse step end to end from host memory.
Everything runs through the C ABI; nothing here computes.
"""

import torch

from . import _lib as L


def tapered_groups(heads):
    """Head-group sizes for run_sparse_host: one-head groups at both ends (K4 starts after one head's
    copy and the copy-out ends one head after the last K4), two-head groups in the middle (fewer K4
    launches).  Measured on two boxes against 24 one-head groups: 42.5 vs 43.1 and 43.5 vs 44.1 ms
    (tools/e2e_groups.py)."""
    if heads < 12:
        return [1] * heads
    mid = heads - 8
    return [1] * 4 + [2] * (mid // 2) + [1] * (mid % 2) + [1] * 4


class HotPath:
    def __init__(self, batch, heads, seq_len, head_dim, block_size, n_text, text_first=False,
                 mode=L.SELECT_RECALL, targets=0.9, flags=L.FLAG_TEXT_SINK, tier_tau=0.8,
                 softmax_scale=0.0, device="cuda", token_major=False):
        """token_major: Q/K/V/O stored [B, N, H, d] (the layout a Ulysses exchange delivers) and
        viewed as [B, H, N, d]; the kernels read it through the descriptor strides."""
        self.shape = (batch, heads, seq_len, head_dim)
        self.token_major = token_major
        self.kw = dict(block_size=block_size, n_text=n_text, text_first=text_first, softmax_scale=softmax_scale)
        self.mode, self.flags, self.tier_tau = mode, flags, tier_tau
        self.targets = [float(targets)] * heads if isinstance(targets, (int, float)) else [float(t) for t in targets]
        dev = torch.device(device)
        if dev.type == "cuda" and dev.index is None:
            dev = torch.device("cuda", torch.cuda.current_device())
        self.device = dev
        e = lambda *s, dt=torch.bfloat16: torch.empty(*s, dtype=dt, device=dev)  # noqa: E731
        if token_major:
            act = lambda: e(batch, seq_len, heads, head_dim).transpose(1, 2)  # noqa: E731
        else:
            act = lambda: e(*self.shape)  # noqa: E731
        self.q, self.k, self.v = act(), act(), act()
        self.desc = L.make_desc(self.q, block_size, n_text, text_first, softmax_scale)
        self.nb = L.num_blocks(self.desc)
        self.o_dense = act()
        self.o_sparse = act()
        self.lse = e(batch, heads, seq_len, dt=torch.float32)
        self.mass = e(batch, heads, self.nb, self.nb, dt=torch.float32)
        rows = batch * heads * self.nb
        self.csr = L.Csr(e(rows + 1, dt=torch.int32), e(rows * self.nb, dt=torch.int32), e(rows, dt=torch.int32),
                         e(batch, heads, dt=torch.float32), e(batch, heads, dt=torch.int64))
        self.ws = e(max(L.sparse_workspace_bytes(self.desc), 1), dt=torch.uint8)
        self.fws = None     # fused-search scratch (K3 workspace + 4*(nb+1)*N bytes per head), on first use
        self.heads_per_pass = 0   # fused search: heads per dense pass (0: all; fewer bound the scratch)
        self.mass2 = None   # block masses of a later key step (K2 with the cached LSE)

    def _stage(self, q, k, v):
        """Device tensors are used in place (any layout the descriptor strides can express, e.g. the
        token-major views a Ulysses exchange delivers); host tensors are copied into the buffers."""
        if all(x.device == self.device for x in (q, k, v)):
            return q, k, v
        if any(x.is_cuda and x.device != self.device for x in (q, k, v)):
            raise ValueError(f"inputs on {q.device}, HotPath on {self.device}")
        self.q.copy_(q, non_blocking=True)
        self.k.copy_(k, non_blocking=True)
        self.v.copy_(v, non_blocking=True)
        return self.q, self.k, self.v

    def search(self, q, k, v, events=None, fused=True):
        """The search step t_w (Alg. 1) into self.o_dense, self.lse (the LSE cache), self.mass and
        self.csr.  fused=True: one call, adaspa_search_select (RECALL without tiers; otherwise as "mass");
        fused="mass": adaspa_dense_attn_lse_search then K3; fused=False: K1, K2, K3.  events: optional
        list of 4 CUDA events recorded around K1, K2, K3 (a fused call lies between events 0 and 1)."""
        q, k, v = self._stage(q, k, v)
        rec = (lambda i: events[i].record()) if events else (lambda i: None)  # noqa: E731
        if fused is True and not self.select_fusable():
            fused = "mass"
        rec(0)
        if fused is True:
            if self.fws is None:
                self.fws = torch.empty(L.search_select_workspace_bytes(self.desc, self.heads_per_pass),
                                       dtype=torch.uint8, device=self.device)
            L.search_select(q, k, v, target=self.targets, flags=self.flags, o=self.o_dense, lse=self.lse,
                            block_mass=self.mass, out=self.csr, workspace=self.fws, **self.kw)
            rec(1)
            rec(2)
            rec(3)
            return self.csr
        if fused:
            if self.fws is None:
                self.fws = torch.empty(L.search_select_workspace_bytes(self.desc, self.heads_per_pass),
                                       dtype=torch.uint8, device=self.device)
            L.dense_attn_lse_search(q, k, v, o=self.o_dense, lse=self.lse, block_mass=self.mass,
                                    workspace=self.fws, **self.kw)
            rec(1)
        else:
            L.dense_attn_lse(q, k, v, o=self.o_dense, lse=self.lse, **self.kw)
            rec(1)
            L.lse_cached_search(q, k, self.lse, block_mass=self.mass, **self.kw)
        rec(2)
        self.select(self.mass)
        rec(3)
        return self.csr

    def select_fusable(self):
        """The selection epilogue of adaspa_search_select covers RECALL mode without head tiers."""
        return self.mode == L.SELECT_RECALL and not (self.flags & L.FLAG_HEAD_TIERS)

    def select(self, mass):
        """K3 on the given block masses into self.csr (a later key step selects on K2's masses)."""
        L.select_blocks(mass, heads_desc=self.desc, mode=self.mode, target=self.targets, flags=self.flags,
                        tier_tau=self.tier_tau, out=self.csr)
        return self.csr

    def dense(self, q, k, v, o=None, lse=None):
        """K1 alone (a warm-up step before t_w): O (and the LSE if `lse` is given)."""
        q, k, v = self._stage(q, k, v)
        o = self.o_dense if o is None else o
        L.dense_attn_lse(q, k, v, o=o, lse=lse, want_lse=lse is not None, **self.kw)
        return o

    def cached_search(self, q, k):
        """K2 of a later key step (Alg. 2): block masses with the CACHED t_w LSE
        (self.lse, reading R19) into self.mass2."""
        if self.mass2 is None:
            self.mass2 = torch.empty_like(self.mass)
        L.lse_cached_search(q, k, self.lse, block_mass=self.mass2, **self.kw)
        return self.mass2

    def sparse(self, q, k, v, csr=None, o=None):
        """K4 on the cached index lists (self.csr unless given): the step every later denoising step runs."""
        q, k, v = self._stage(q, k, v)
        csr = self.csr if csr is None else csr
        o = self.o_sparse if o is None else o
        L.block_sparse_attn(q, k, v, csr.row_ptr, csr.col_idx, o=o, workspace=self.ws, **self.kw)
        return o

    def run(self, q, k, v, events=None, fused=True):
        """search() then sparse(); events: optional list of 5 CUDA events recorded around K1..K4."""
        q, k, v = self._stage(q, k, v)
        self.search(q, k, v, events=events[:4] if events else None, fused=fused)
        self.sparse(q, k, v)
        if events:
            events[4].record()
        return self.o_sparse

    # launches of our kernels per run(): search step 5 (dense pass, block mass + selection epilogue, head,
    # scan, write; RECALL) or 6 (dense pass, block mass, K3's rows, head, scan, write; +2 with tiers), K4 3
    # (stream + order + attention)
    def kernels_per_run(self):
        if self.select_fusable() and L.num_blocks(self.desc) <= 2048:
            return 8
        return 9 + (2 if self.flags & L.FLAG_HEAD_TIERS else 0)

    def run_sparse_host(self, q_host, k_host, v_host, o_host, groups=24):
        """A sparse denoising step end to end from host memory (the steps between
        key steps only run the block-sparse forward on the cached index lists): per head group, the
        H2D copy of Q,K,V on a copy stream overlaps K4 of the previous group, and O goes back per
        group.  The groups' K4 launches alternate between the current stream and a second compute
        stream (each with its own workspace), so one launch's tail overlaps the next launch's start:
        twelve back-to-back launches on one stream take 37.5 ms against 31.2 ms for one launch
        (tools/e2e_parts.py).  groups: a number of equal head groups, or a list of head counts per group.
        q/k/v/o_host: pinned [B, H, N, d] host tensors.  Uses the CSR of the
        last run() (the cache).  Everything on the device path is the C-ABI's K4."""
        B, H, N, d = self.shape
        if B != 1:
            raise ValueError("run_sparse_host stages head groups of batch 1")
        cur = torch.cuda.current_stream(self.device)
        if not hasattr(self, "_copy_stream"):
            self._copy_stream = torch.cuda.Stream(self.device)
            self._out_stream = torch.cuda.Stream(self.device)
        if not hasattr(self, "_compute_stream2"):
            self._compute_stream2 = torch.cuda.Stream(self.device)
            self._ws2 = torch.empty_like(self.ws)
        cs, os_ = self._copy_stream, self._out_stream
        ks = (cur, self._compute_stream2)
        wss = (self.ws, self._ws2)
        ks[1].wait_stream(cur)
        cs.wait_stream(cur)
        if isinstance(groups, (list, tuple)):  # explicit head counts per group (e.g. tapered ends)
            if sum(groups) != H or min(groups) < 1:
                raise ValueError(f"group sizes {groups} must be >= 1 and sum to {H} heads")
            bounds = [0]
            for n in groups:
                bounds.append(bounds[-1] + int(n))
            groups = len(bounds) - 1
        else:
            groups = max(1, min(int(groups), H))  # at least one head per group
            bounds = [H * g // groups for g in range(groups + 1)]
        done_in, done_k4 = [], []
        for g in range(groups):
            h0, h1 = bounds[g], bounds[g + 1]
            with torch.cuda.stream(cs):
                for dev, host in ((self.q, q_host), (self.k, k_host), (self.v, v_host)):
                    dev[:, h0:h1].copy_(host[:, h0:h1], non_blocking=True)
                e = torch.cuda.Event()
                e.record(cs)
            done_in.append(e)
        for g in range(groups):
            h0, h1 = bounds[g], bounds[g + 1]
            st = ks[g & 1]
            st.wait_event(done_in[g])
            rp = self.csr.row_ptr[h0 * self.nb: h1 * self.nb + 1]
            with torch.cuda.stream(st):
                L.block_sparse_attn(self.q[:, h0:h1], self.k[:, h0:h1], self.v[:, h0:h1], rp, self.csr.col_idx,
                                    o=self.o_sparse[:, h0:h1], workspace=wss[g & 1], **self.kw)
            e = torch.cuda.Event()
            e.record(st)
            done_k4.append(e)
        for g in range(groups):
            h0, h1 = bounds[g], bounds[g + 1]
            os_.wait_event(done_k4[g])
            with torch.cuda.stream(os_):
                o_host[:, h0:h1].copy_(self.o_sparse[:, h0:h1], non_blocking=True)
        cur.wait_stream(ks[1])
        cur.wait_stream(os_)
        return o_host
