"""Multi-GPU plumbing of the hot path.

The method is independent per (batch, head): the LSE, the block masses and the CSR are per head,
so K1..K4 need no communication (the method is "orthogonal to ... parallelization").
What moves between GPUs is plumbing, done here with torch.distributed (NCCL on the GPUs, gloo in
the CPU tests):

* head sharding (`head_range`): rank p owns a contiguous group of heads -- the search step's
  (K1, K2, K3) assignment, equal head counts because dense work is the same for every head;
* LPT rebalancing of the sparse pass (`lpt_assign`, `gather_csr`, `pack_heads_csr`): per-head kept
  tiles differ by >20x under head-adaptive recall ("severe kernel load imbalance"),
  so after a search the CSRs are all-gathered (one NCCL exchange per key step, ~MBs) and each rank
  runs K4 on an LPT head set (heads by kept tiles, descending, each to the least-loaded rank);
* Ulysses exchange for activations that arrive sequence-sharded (a sequence-parallel DiT):
  `ulysses_in` turns each rank's token chunk of all heads, [N_p, H, d], into all tokens of its head
  set, [N, H_r, d], with one NCCL all_to_all per tensor (any head set per rank: an LPT assignment
  is just another send order); `ulysses_out` sends O back.  The received buffer is token-major
  [N, H_r, d] as it lands (chunks arrive in rank order), so the kernels read it through the
  descriptor strides (stride_n = H_r*d, stride_h = d) with no unpack copy (`as_bhnd`).

No arithmetic of the method happens here: tensors are moved, concatenated and re-indexed.
"""

import torch
import torch.distributed as dist


def head_range(H, world, rank):
    """Contiguous head group of `rank`: sizes differ by at most one."""
    base, extra = divmod(H, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def contiguous_assign(H, world):
    """head_range as a list of head lists (the search step's assignment)."""
    return [list(range(*head_range(H, world, r))) for r in range(world)]


def seq_splits(N, world):
    """Token chunk sizes of a sequence-sharded activation (rank order)."""
    base, extra = divmod(N, world)
    return [base + (1 if r < extra else 0) for r in range(world)]


def lpt_assign(costs, world):
    """Longest-processing-time head -> rank assignment: heads by cost descending (ties by index),
    each to the currently least-loaded rank (ties by rank).  Returns a list of head lists."""
    order = sorted(range(len(costs)), key=lambda h: (-float(costs[h]), h))
    load = [0.0] * world
    out = [[] for _ in range(world)]
    for h in order:
        r = min(range(world), key=lambda i: (load[i], i))
        out[r].append(h)
        load[r] += float(costs[h])
    return [sorted(x) for x in out]


def imbalance(costs, assign):
    """max-rank / mean-rank load of an assignment (1.0 = perfect), and the per-rank loads."""
    loads = [float(sum(costs[h] for h in hs)) for hs in assign]
    mean = sum(loads) / len(loads)
    return (max(loads) / mean if mean > 0 else 1.0), loads


def _world(group):
    return dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1


def gather_csr(row_ptr, col_idx, group=None):
    """All-gather the CSRs of every rank's head group (contiguous `head_range` groups, rank order)
    into one CSR of the whole layer: row_ptr [H*nb + 1] (rank r's rows re-based by the kept count of
    ranks < r), col_idx [total nnz].  row_ptr/col_idx: this rank's CSR (row_ptr [H_r*nb + 1], as
    adaspa_select_blocks writes it).  Two all_gathers (counts, then padded payloads); one host read
    of the counts.  Single process: returned as is."""
    world = _world(group)
    nnz = row_ptr[-1:].to(torch.int64)
    if world == 1:
        return row_ptr, col_idx[: int(nnz.item())]
    dev = row_ptr.device
    meta = torch.stack([nnz[0], torch.tensor(row_ptr.numel() - 1, dtype=torch.int64, device=dev)])
    metas = [torch.empty_like(meta) for _ in range(world)]
    dist.all_gather(metas, meta, group=group)
    metas = [m.tolist() for m in metas]
    max_nnz = max(max(m[0] for m in metas), 1)
    max_rows = max(m[1] for m in metas)
    rp_pad = torch.zeros(max_rows + 1, dtype=row_ptr.dtype, device=dev)
    rp_pad[: row_ptr.numel()] = row_ptr
    ci_pad = torch.zeros(max_nnz, dtype=col_idx.dtype, device=dev)
    n_loc = int(metas[dist.get_rank(group)][0])
    ci_pad[:n_loc] = col_idx[:n_loc]
    rps = [torch.empty_like(rp_pad) for _ in range(world)]
    cis = [torch.empty_like(ci_pad) for _ in range(world)]
    dist.all_gather(rps, rp_pad, group=group)
    dist.all_gather(cis, ci_pad, group=group)
    out_rp, out_ci, base = [], [], 0
    for r in range(world):
        n_r, rows_r = metas[r]
        out_rp.append(rps[r][:rows_r] + base)
        out_ci.append(cis[r][:n_r])
        base += n_r
    out_rp.append(torch.tensor([base], dtype=row_ptr.dtype, device=dev))
    return torch.cat(out_rp), torch.cat(out_ci)


def head_nnz(row_ptr, nb):
    """Kept blocks per head of a whole-layer CSR (the LPT cost), as a host list."""
    rp = row_ptr.to(torch.int64).cpu()
    return (rp[nb::nb] - rp[0:-1:nb]).tolist()


def pack_heads_csr(row_ptr, col_idx, heads, nb):
    """The CSR of `heads` (in that order) cut out of a whole-layer CSR: row_ptr [len(heads)*nb + 1],
    col_idx [their nnz] -- what K4 reads for a [1, len(heads), N, d] Q/K/V of those heads."""
    rp = row_ptr.to(torch.int64)
    bounds = rp[[h * nb for h in heads] + [(h + 1) * nb for h in heads]].cpu().tolist()
    starts, stops = bounds[: len(heads)], bounds[len(heads):]
    out_rp, out_ci, base = [], [], 0
    for h, a, b in zip(heads, starts, stops):
        out_rp.append(rp[h * nb:(h + 1) * nb] - a + base)
        out_ci.append(col_idx[a:b])
        base += b - a
    out_rp.append(torch.tensor([base], dtype=torch.int64, device=row_ptr.device))
    ci = torch.cat(out_ci) if out_ci else col_idx[:0]
    return torch.cat(out_rp).to(row_ptr.dtype), ci


def ulysses_in(x_local, group=None, sizes=None, assign=None):
    """Sequence-sharded [N_p, H, d] (this rank's token chunk, all heads) -> head-sharded
    [N, H_r, d] (all tokens, this rank's head set).  assign: the head list of every rank (default:
    contiguous groups, H divisible by the world size).  sizes: every rank's token count
    (seq_splits); gathered with one small all_gather if None.  Returns a contiguous tensor; view it
    as [1, H_r, N, d] with `as_bhnd` for the kernels."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    Np, H, d = x_local.shape
    if assign is None:
        if H % world:
            raise ValueError("Ulysses needs H divisible by the world size")
        assign = contiguous_assign(H, world)
    if sorted(h for a in assign for h in a) != list(range(H)):
        raise ValueError("assign must partition the heads")
    # send chunk r = heads assign[r] of my tokens, [N_p, |assign[r]|, d] each, rank order
    flat = [h for a in assign for h in a]
    if flat == list(range(H)):
        send = torch.cat([x_local[:, a[0]:a[-1] + 1].reshape(-1) if a else x_local[:0, 0].reshape(-1)
                          for a in assign]) if world > 1 else x_local.reshape(-1)
    else:
        idx = torch.tensor(flat, device=x_local.device)
        perm = x_local.index_select(1, idx)                      # [N_p, H, d] in assign order
        offs = [0]
        for a in assign:
            offs.append(offs[-1] + len(a))
        send = torch.cat([perm[:, offs[r]:offs[r + 1]].reshape(-1) for r in range(world)])
    if sizes is None:
        all_np = [torch.zeros(1, dtype=torch.int64, device=x_local.device) for _ in range(world)]
        dist.all_gather(all_np, torch.tensor([Np], dtype=torch.int64, device=x_local.device), group=group)
        sizes = [int(t.item()) for t in all_np]
    N = sum(sizes)
    Hr = len(assign[rank])
    recv = torch.empty(N, Hr, d, dtype=x_local.dtype, device=x_local.device)
    dist.all_to_all_single(recv.view(-1), send.contiguous(),
                           output_split_sizes=[s * Hr * d for s in sizes],
                           input_split_sizes=[Np * len(a) * d for a in assign], group=group)
    return recv


def ulysses_out(o_heads, n_local_sizes, group=None, assign=None):
    """Head-sharded O [N, H_r, d] (token-major, this rank's head set) -> sequence-sharded
    [N_p, H, d] for this rank, heads back in their global order.  n_local_sizes: the token chunk
    sizes of every rank (seq_splits); assign: as in ulysses_in."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    N, Hr, d = o_heads.shape
    Np = n_local_sizes[rank]
    if assign is None:
        assign = [list(range(r * Hr, (r + 1) * Hr)) for r in range(world)]
    H = sum(len(a) for a in assign)
    # my token chunk of every rank's head set arrives rank by rank: [N_p, |assign[r]|, d] each
    recv = torch.empty(Np * H * d, dtype=o_heads.dtype, device=o_heads.device)
    dist.all_to_all_single(recv, o_heads.contiguous().view(-1),
                           output_split_sizes=[Np * len(a) * d for a in assign],
                           input_split_sizes=[s * Hr * d for s in n_local_sizes], group=group)
    parts, off = [], 0
    for a in assign:
        n = Np * len(a) * d
        parts.append(recv[off:off + n].view(Np, len(a), d))
        off += n
    got = torch.cat(parts, dim=1)                               # [N_p, H, d] in assign order
    flat = [h for a in assign for h in a]
    if flat == list(range(H)):
        return got
    inv = torch.empty(H, dtype=torch.long)
    inv[torch.tensor(flat)] = torch.arange(H)
    return got.index_select(1, inv.to(got.device))


def as_bhnd(x_nhd):
    """[N, H_r, d] token-major -> a [1, H_r, N, d] strided view (stride_n = H_r*d, stride_h = d)."""
    return x_nhd.permute(1, 0, 2).unsqueeze(0)


def reduce_max(values, group=None):
    """Element-wise max over ranks of a list of floats (per-step, per-kernel times).  Single
    process: returned as is."""
    t = torch.tensor([float(x) for x in values], dtype=torch.float64)
    if _world(group) > 1:
        dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl" else t.device
        t = t.to(dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return [float(x) for x in t.cpu()]


def reduce_sum(values, group=None):
    """Element-wise sum over ranks (work: kept FLOPs, kept tiles)."""
    t = torch.tensor([float(x) for x in values], dtype=torch.float64)
    if _world(group) > 1:
        dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl" else t.device
        t = t.to(dev)
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return [float(x) for x in t.cpu()]


def all_gather_floats(values, group=None):
    """Every rank's list of floats (same length on every rank), rank order."""
    t = torch.tensor([float(x) for x in values], dtype=torch.float64)
    world = _world(group)
    if world == 1:
        return [[float(x) for x in t]]
    dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl" else t.device
    t = t.to(dev)
    out = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(out, t, group=group)
    return [[float(x) for x in o.cpu()] for o in out]


def reduce_step_timings(kernel_ms, kept_flops, steps, group=None):
    """Whole-job numbers of a bench run (bench.py): every rank timed `steps` steps
    of its share; kernel_ms = [total, K1, K2, K3, K4] summed over the steps (ms).  Returns
    (value TFLOP/s = sum over ranks of kept FLOPs x steps / the slowest rank's K4 time,
    per-kernel max-over-ranks ms)."""
    t = reduce_max(kernel_ms, group)
    w = reduce_sum([kept_flops], group)[0]
    value = w * steps / (t[4] / 1e3) / 1e12
    return value, t


def _runs(heads):
    """Maximal runs of consecutive head ids in a head list: (first head, count, position in the list)."""
    out, i = [], 0
    while i < len(heads):
        j = i
        while j + 1 < len(heads) and heads[j + 1] == heads[j] + 1:
            j += 1
        out.append((heads[i], j - i + 1, i))
        i = j + 1
    return out


class PeerExchange:
    """The Ulysses exchange over peer memory instead of NCCL.

    Every rank owns receive buffers -- `n_in` head-sharded tensors [N, H_r, d] (Q, K, V of its head
    set, token-major as the kernels read them) and one sequence-sharded [N_p, H, d] (O of its token
    chunk) -- plus a flag block [4, world] (in-ready, in-released, out-ready, out-released; slot p is
    written by rank p).  The buffers are CUDA IPC-mapped into every other rank once (handles
    exchanged with one all_gather_object).  A push is copy-engine 2-D copies straight into the
    destinations' buffers (each contiguous run of a destination's head list is one copy per tensor:
    rows = this rank's tokens, pitches H*d and H_r*d) followed by one 32-bit flag write per
    destination, all stream-ordered on the caller's stream; `wait_*` makes the caller's stream wait
    until every peer's flag reaches the exchange's epoch.  Before overwriting a destination's buffer
    a push waits for that destination's release of the previous epoch (`release_*`, recorded after
    the kernels that read the buffer), so exchanges can be issued ahead of compute.  No NCCL and no
    SMs on the data path; nothing of the method's arithmetic.  At world size 1 the "peer" is this
    process (local pointers, no IPC)."""

    IN_READY, IN_REL, OUT_READY, OUT_REL = range(4)

    def __init__(self, N, H, d, sizes, assign, device, group=None, n_in=3, dtype=torch.bfloat16):
        from . import _lib as L
        self._L = L
        self.world = _world(group)
        self.rank = dist.get_rank(group) if self.world > 1 else 0
        if sorted(h for a in assign for h in a) != list(range(H)) or len(assign) != self.world:
            raise ValueError("assign must partition the heads over the ranks")
        if len(sizes) != self.world or sum(sizes) != N:
            raise ValueError("sizes must give every rank's token count")
        self.N, self.H, self.d, self.sizes, self.assign = N, H, d, list(sizes), [list(a) for a in assign]
        self.offs = [sum(sizes[:r]) for r in range(self.world)]
        self.es = torch.empty(0, dtype=dtype).element_size()
        Hr = len(assign[self.rank])
        self.recv_in = [torch.empty(N, Hr, d, dtype=dtype, device=device) for _ in range(n_in)]
        self.recv_out = torch.empty(sizes[self.rank], H, d, dtype=dtype, device=device)
        self.flags = torch.zeros(4, self.world, dtype=torch.int32, device=device)
        self.n_in = n_in
        mine = [t.data_ptr() for t in self.recv_in] + [self.recv_out.data_ptr(), self.flags.data_ptr()]
        self._bases = []
        if self.world == 1:
            ptrs = [mine]
        else:
            torch.cuda.synchronize(device)
            blobs = [L.peer_export(p) for p in mine]
            every = [None] * self.world
            dist.all_gather_object(every, blobs, group=group)
            ptrs = []
            for r in range(self.world):
                if r == self.rank:
                    ptrs.append(mine)
                    continue
                row = []
                for b in every[r]:
                    p, base = L.peer_import(b)
                    row.append(p)
                    self._bases.append(base)
                ptrs.append(row)
        self.peer_in = [row[:n_in] for row in ptrs]
        self.peer_out = [row[n_in] for row in ptrs]
        self.peer_flags = [row[n_in + 1] for row in ptrs]
        self.epoch_in = 0
        self.epoch_out = 0

    def close(self):
        for b in self._bases:
            self._L.peer_close(b)
        self._bases = []

    def _flag(self, r, kind, slot):
        return self.peer_flags[r] + 4 * (kind * self.world + slot)

    def _own_flags(self, kind):
        return self.flags.data_ptr() + 4 * kind * self.world

    def push_in(self, xs, stream=None):
        """This rank's token chunks [N_p, H, d] (one per input tensor, contiguous) into every rank's
        head-sharded receive buffers; raises IN_READY on each destination."""
        L, es, d, H = self._L, self.es, self.d, self.H
        Np = self.sizes[self.rank]
        if len(xs) != self.n_in or any(tuple(x.shape) != (Np, H, d) or not x.is_contiguous() for x in xs):
            raise ValueError(f"push_in needs {self.n_in} contiguous [{Np}, {H}, {d}] tensors")
        e = self.epoch_in + 1
        # the destinations must have released epoch e-1 of their buffers
        L.peer_wait(self._own_flags(self.IN_REL), self.world, e - 1, stream)
        for r in range(self.world):
            Hr = len(self.assign[r])
            for h0, n, pos in _runs(self.assign[r]):
                for i, x in enumerate(xs):
                    L.peer_copy2d(self.peer_in[r][i] + (self.offs[self.rank] * Hr + pos) * d * es, Hr * d * es,
                                  x.data_ptr() + h0 * d * es, H * d * es, n * d * es, Np, stream)
            L.peer_signal(self._flag(r, self.IN_READY, self.rank), e, stream)
        self.epoch_in = e

    def wait_in(self, stream=None):
        """Later work on `stream` waits until every rank's push of this epoch has landed; returns
        the receive buffers [N, H_r, d]."""
        self._L.peer_wait(self._own_flags(self.IN_READY), self.world, self.epoch_in, stream)
        return self.recv_in

    def release_in(self, stream=None):
        """After the kernels that read recv_in (stream-ordered): lets the next push overwrite them."""
        for r in range(self.world):
            self._L.peer_signal(self._flag(r, self.IN_REL, self.rank), self.epoch_in, stream)

    def push_out(self, o_heads, stream=None):
        """O of this rank's head set [N, H_r, d] (token-major) back to every rank's [N_p, H, d] buffer
        (heads in their global order); raises OUT_READY on each destination."""
        L, es, d, H = self._L, self.es, self.d, self.H
        mine = self.assign[self.rank]
        Hr = len(mine)
        if tuple(o_heads.shape) != (self.N, Hr, d) or o_heads.stride() != (Hr * d, d, 1):
            raise ValueError(f"push_out needs a [{self.N}, {Hr}, {d}] token-major tensor")
        e = self.epoch_out + 1
        L.peer_wait(self._own_flags(self.OUT_REL), self.world, e - 1, stream)
        for p in range(self.world):
            for h0, n, pos in _runs(mine):
                L.peer_copy2d(self.peer_out[p] + h0 * d * es, H * d * es,
                              o_heads.data_ptr() + (self.offs[p] * Hr + pos) * d * es, Hr * d * es, n * d * es,
                              self.sizes[p], stream)
            L.peer_signal(self._flag(p, self.OUT_READY, self.rank), e, stream)
        self.epoch_out = e

    def wait_out(self, stream=None):
        self._L.peer_wait(self._own_flags(self.OUT_READY), self.world, self.epoch_out, stream)
        return self.recv_out

    def release_out(self, stream=None):
        for r in range(self.world):
            self._L.peer_signal(self._flag(r, self.OUT_REL, self.rank), self.epoch_out, stream)
