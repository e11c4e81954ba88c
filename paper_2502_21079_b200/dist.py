"""Multi-GPU plumbing of the hot path.

The method is independent per (batch, head): the LSE, the block masses and the CSR are per head,
so K1..K4 need no communication.  Two ways to spread it over GPUs:

* head sharding (`head_range`): rank p owns a contiguous group of heads;
* Ulysses exchange, for activations that arrive sequence-sharded (a sequence-parallel DiT):
  `ulysses_in` turns each rank's token chunk of all heads, [N_p, H, d], into all tokens of its
  head group, [N, H/P, d], with one NCCL all_to_all per tensor; `ulysses_out` sends O back.
  The received buffer is token-major [N, H/P, d] as it lands (chunks arrive in rank order), so
  the kernels read it through the descriptor strides (stride_n = H/P*d, stride_h = d) with no
  unpack copy.

torch.distributed is the plumbing (process group, all_to_all_single); no arithmetic of the method
happens here.  The optional LPT head -> rank assignment (`lpt_assign`) balances per-head kept-tile
counts, which differ by >20x under head-adaptive recall.
"""

import torch
import torch.distributed as dist


def head_range(H, world, rank):
    """Contiguous head group of `rank`: sizes differ by at most one."""
    base, extra = divmod(H, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


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


def ulysses_in(x_local, group=None, sizes=None):
    """Sequence-sharded [N_p, H, d] (this rank's token chunk, all heads) -> head-sharded
    [N, Hp, d] (all tokens, this rank's contiguous head group).  H must divide by the world size.
    sizes: every rank's token count (seq_splits); gathered with one small all_gather if None.
    Returns a contiguous tensor; view it as [1, Hp, N, d] with `as_bhnd` for the kernels."""
    world = dist.get_world_size(group)
    Np, H, d = x_local.shape
    if H % world:
        raise ValueError("Ulysses needs H divisible by the world size")
    Hp = H // world
    # send chunk r = heads [r*Hp, (r+1)*Hp) of my tokens: [world, Np, Hp, d] contiguous
    send = x_local.view(Np, world, Hp, d).permute(1, 0, 2, 3).contiguous()
    if sizes is None:
        all_np = [torch.zeros(1, dtype=torch.int64, device=x_local.device) for _ in range(world)]
        dist.all_gather(all_np, torch.tensor([Np], dtype=torch.int64, device=x_local.device), group=group)
        sizes = [int(t.item()) for t in all_np]
    N = sum(sizes)
    recv = torch.empty(N, Hp, d, dtype=x_local.dtype, device=x_local.device)
    dist.all_to_all_single(recv.view(-1), send.view(-1),
                           output_split_sizes=[s * Hp * d for s in sizes],
                           input_split_sizes=[Np * Hp * d] * world, group=group)
    return recv


def ulysses_out(o_heads, n_local_sizes, group=None):
    """Head-sharded O [N, Hp, d] (token-major) -> sequence-sharded [N_p, H, d] for this rank.
    n_local_sizes: the token chunk sizes of every rank (seq_splits)."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    N, Hp, d = o_heads.shape
    Np = n_local_sizes[rank]
    # my token chunk of every rank's head group arrives as [world, Np, Hp, d]
    recv = torch.empty(world, Np, Hp, d, dtype=o_heads.dtype, device=o_heads.device)
    dist.all_to_all_single(recv.view(-1), o_heads.contiguous().view(-1),
                           output_split_sizes=[Np * Hp * d] * world,
                           input_split_sizes=[s * Hp * d for s in n_local_sizes], group=group)
    return recv.permute(1, 0, 2, 3).reshape(Np, world * Hp, d)


def as_bhnd(x_nhd):
    """[N, Hp, d] token-major -> a [1, Hp, N, d] strided view (stride_n = Hp*d, stride_h = d)."""
    return x_nhd.permute(1, 0, 2).unsqueeze(0)


def reduce_step_timings(kernel_ms, kept_flops, steps, group=None):
    """Whole-job numbers of a weak-scaling bench run (bench.py): every rank timed
    `steps` steps of its own layer; kernel_ms = [total, K1, K2, K3, K4] summed over the steps (ms).
    Returns (value TFLOP/s = sum over ranks of kept FLOPs x steps / the slowest rank's K4 time,
    per-kernel max-over-ranks ms).  Single process: no collective."""
    t = torch.tensor([float(x) for x in kernel_ms], dtype=torch.float64)
    w = torch.tensor([float(kept_flops)], dtype=torch.float64)
    if dist.is_available() and dist.is_initialized():
        dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl" else t.device
        t, w = t.to(dev), w.to(dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
        dist.all_reduce(w, op=dist.ReduceOp.SUM, group=group)
    t = t.cpu()
    value = float(w.item()) * steps / (float(t[4]) / 1e3) / 1e12
    return value, [float(x) for x in t]
