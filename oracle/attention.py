"""Dense attention, block mass and masked attention in fp64 (oracle; test
infrastructure only).  All functions take ONE head: q [Nq,d], k/v [N,d] as
float64 numpy arrays (the caller upcasts the same bf16 tensors the GPU reads,
which is exact).
"""

import numpy as np


def dense_attention(q, k, v, scale):
    """PAPER.md:166-191 (subsec:flash, W_attn, LSE and safe softmax):
    Z = scale * Q K^T;  LSE(z) = max_j z_j + log sum_j exp(z_j - max_k z_k);
    W = exp(Z - LSE);  O = W V.   Reading R5: scale = 1/sqrt(d) in every pass.

    Returns (O [Nq,d], lse [Nq]) with lse the natural-log LSE of the scaled
    logits (the quantity Alg. 1 line 11 caches)."""
    q = np.asarray(q, dtype=np.float64)
    k = np.asarray(k, dtype=np.float64)
    v = np.asarray(v, dtype=np.float64)
    z = scale * (q @ k.T)
    m = z.max(axis=1)
    lse = m + np.log(np.exp(z - m[:, None]).sum(axis=1))
    w = np.exp(z - lse[:, None])
    return w @ v, lse


def block_mass(q, k, lse, blocks, scale, q_block_ids=None):
    """W_sum_attn: the sum of the attention weights inside
    each (q-block, kv-block) tile, with the weights taken as
    exp(scale * q_i . k_j - lse_i)  (Alg. 1 lines 17-21 / Alg. 2 lines 4-8,
    PAPER.md:486-491, 509-515, reading R4: "Log(qk - LSE)" is exp(qk*scale - LSE)).

    `lse` is whatever LSE the caller supplies: the exact one of the same (Q,K)
    at the fused search step, or the cached one from step t_w at later key
    steps (Alg. 2).  The matrix is built explicitly, one q-block
    row at a time.  Returns M [len(q_block_ids), nb] (fp64)."""
    q = np.asarray(q, dtype=np.float64)
    k = np.asarray(k, dtype=np.float64)
    lse = np.asarray(lse, dtype=np.float64)
    nb = len(blocks)
    if q_block_ids is None:
        q_block_ids = range(nb)
    q_block_ids = list(q_block_ids)
    out = np.zeros((len(q_block_ids), nb), dtype=np.float64)
    for r, p in enumerate(q_block_ids):
        bp = blocks[p]
        rows = slice(bp.start, bp.start + bp.length)
        w = np.exp(scale * (q[rows] @ k.T) - lse[rows][:, None])
        for j, bj in enumerate(blocks):
            out[r, j] = w[:, bj.start:bj.start + bj.length].sum()
    return out


def masked_attention(q, k, v, blocks, kept, scale, q_block_ids=None):
    """Blockified sparse attention, PAPER.md:415-427 (the -c(1 - M~_S) bias)
    taken with c = +inf (exact exclusion, SPEC.md:140 reading): for query i in
    q-block p, J = union of the tokens of the kv-blocks kept in row p, and
        lse'_i = log sum_{j in J} exp(z_ij),   O_i = sum_{j in J} exp(z_ij - lse'_i) v_j.
    `kept[p]` is the iterable of kept kv-block indices of row p (any order).
    Returns (O [rows,d], lse' [rows]) for the q-blocks in q_block_ids, rows in
    q-block order then token order."""
    q = np.asarray(q, dtype=np.float64)
    k = np.asarray(k, dtype=np.float64)
    v = np.asarray(v, dtype=np.float64)
    nb = len(blocks)
    if q_block_ids is None:
        q_block_ids = range(nb)
    outs, lses = [], []
    for p in q_block_ids:
        bp = blocks[p]
        cols = np.concatenate([np.arange(blocks[j].start, blocks[j].start + blocks[j].length)
                               for j in sorted(set(int(x) for x in kept[p]))])
        z = scale * (q[bp.start:bp.start + bp.length] @ k[cols].T)
        m = z.max(axis=1)
        l = m + np.log(np.exp(z - m[:, None]).sum(axis=1))
        outs.append(np.exp(z - l[:, None]) @ v[cols])
        lses.append(l)
    return np.concatenate(outs, axis=0), np.concatenate(lses)


def expand_block_mask(keep, blocks):
    """M_S in {0,1}^{nb x nb}  ->  M~_S in {0,1}^{L x L}."""
    n = sum(b.length for b in blocks)
    out = np.zeros((n, n), dtype=bool)
    for p, bp in enumerate(blocks):
        for j, bj in enumerate(blocks):
            if keep[p][j]:
                out[bp.start:bp.start + bp.length, bj.start:bj.start + bj.length] = True
    return out
