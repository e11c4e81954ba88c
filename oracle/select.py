"""Head-adaptive hierarchical block selection (oracle; test infrastructure only).

Plain Python over fp64 masses.  Order of every sort is the key
(mass descending, kv-block index ascending) -- reading R10.
"""

import itertools
import math

import numpy as np


def k_from_sparsity(s, n_candidates):
    """Row-wise top-k budget ("k in {1..(1-sparsity)(L/B)^2}" taken
    per q-block row because of Row Wise; readings R6, R11):
        k = max(1, floor((1 - s) * n + 0.5 + 1e-9)),  capped at n.
    The 1e-9 makes (3*0.8-1)/2 = 0.7000000000000002 round like 0.7."""
    if n_candidates <= 0:
        return 0
    k = int(math.floor((1.0 - float(s)) * n_candidates + 0.5 + 1e-9))
    return min(max(1, k), n_candidates)


def row_forced_and_candidates(blocks, p, text_sink):
    """Text Sink (reading R13): every text kv-block is forced for
    every row, and a text q-block row keeps every kv-block (the vt, tv and tt
    parts).  Returns (forced, candidates) as ascending index lists.  Without
    the text sink nothing is forced and every block is a candidate."""
    nb = len(blocks)
    if not text_sink:
        return [], list(range(nb))
    if blocks[p].modality == "text":
        return list(range(nb)), []
    forced = [j for j in range(nb) if blocks[j].modality == "text"]
    cands = [j for j in range(nb) if blocks[j].modality == "video"]
    return forced, cands


def _sorted_candidates(masses, candidates):
    return sorted(candidates, key=lambda j: (-masses[j], j))


def select_row_recall(masses, forced, candidates, r):
    """RECALL mode for one q-block row (north_star; Recall is PAPER.md:228-232
    evaluated per row, readings R7, R8, R9, R12, R25).

    T = sum of the row's masses (all kv-blocks).  Keep `forced`, then add
    candidates in (mass desc, idx asc) order until the kept mass reaches r*T
    ("reaches" = acc >= r*T in fp64).  r >= 1 keeps everything.  If the forced
    set alone already reaches r*T (or r <= 0) only it is kept, and if it is
    empty the single top candidate is kept so that no row is empty."""
    masses = [float(x) for x in masses]
    T = 0.0
    for x in masses:
        T += x
    kept = list(forced)
    if r >= 1.0:
        return sorted(set(kept) | set(candidates))
    target = r * T
    acc = 0.0
    for j in forced:
        acc += masses[j]
    order = _sorted_candidates(masses, candidates)
    if acc >= target or r <= 0.0:
        if not kept and order:
            kept.append(order[0])
        return sorted(kept)
    for j in order:
        kept.append(j)
        acc += masses[j]
        if acc >= target:
            break
    return sorted(kept)


def select_row_sparsity(masses, forced, candidates, k):
    """SPARSITY mode for one row: S* of PAPER.md:436-448 with Row Wise
    (PAPER.md:550): `forced` plus the k best candidates by (mass desc, idx asc).
    Forced blocks are extras outside k (reading R12)."""
    masses = [float(x) for x in masses]
    order = _sorted_candidates(masses, candidates)
    return sorted(set(forced) | set(order[:k]))


def head_tiers(recalls, s_base, tau=0.8):
    """Head-adaptive hierarchical sparsity: sort heads by
    Recall; n = #heads with Recall > tau (tau = 0.8); the n
    highest-Recall heads get (1+s)/2, the n lowest get (3s-1)/2.
    Readings R16/R17: strict '>' , n capped at floor(H/2), ties by head index
    ascending, s < 1/3 rejected.  `s_base` is one value or one per head; the
    formula is applied to each head's own base."""
    H = len(recalls)
    s = [float(x) for x in (s_base if np.ndim(s_base) else [s_base] * H)]
    if any(x < 1.0 / 3.0 for x in s):
        raise ValueError("head tiers need sparsity >= 1/3 (PAPER.md:532, (3s-1)/2 >= 0)")
    n = min(sum(1 for x in recalls if float(x) > tau), H // 2)
    order = sorted(range(H), key=lambda h: (-float(recalls[h]), h))
    out = list(s)
    for h in order[:n]:
        out[h] = (1.0 + s[h]) / 2.0
    for h in order[H - n:] if n > 0 else []:
        out[h] = (3.0 * s[h] - 1.0) / 2.0
    return out


def _select_head(Mh, blocks, mode, target, text_sink):
    nb = len(blocks)
    keep = np.zeros((nb, nb), dtype=bool)
    for p in range(nb):
        forced, cands = row_forced_and_candidates(blocks, p, text_sink)
        if mode == "recall":
            kept = select_row_recall(Mh[p], forced, cands, target)
        else:
            kept = select_row_sparsity(Mh[p], forced, cands, k_from_sparsity(target, len(cands)))
        keep[p, kept] = True
    return keep


def _head_recall(Mh, keep):
    """Whole-matrix Recall of PAPER.md:230 at block granularity: kept mass over
    total mass, all rows (reading R16)."""
    num = 0.0
    den = 0.0
    for p in range(Mh.shape[0]):
        for j in range(Mh.shape[1]):
            den += float(Mh[p, j])
            if keep[p, j]:
                num += float(Mh[p, j])
    return num / den if den > 0 else 0.0


def select_blocks(M, blocks, mode, targets, text_sink=True, tiers=False, tau=0.8):
    """Selection for all heads of one batch element.  M: [H, nb, nb] fp64.
    mode: "recall" (targets = per-head r_h) or "sparsity" (targets = s_h).
    tiers (SPARSITY mode only): select at the base targets, compute each head's
    Recall, re-target with head_tiers, select again.
    Returns (keep [H,nb,nb] bool, head_recall [H], head_nnz [H], final_targets [H])."""
    M = np.asarray(M, dtype=np.float64)
    H = M.shape[0]
    targets = [float(x) for x in targets]
    if tiers:
        if mode != "sparsity":
            raise ValueError("tiers apply to SPARSITY mode")
        base = [_select_head(M[h], blocks, mode, targets[h], text_sink) for h in range(H)]
        rec = [_head_recall(M[h], base[h]) for h in range(H)]
        targets = head_tiers(rec, targets, tau)
    keep = np.stack([_select_head(M[h], blocks, mode, targets[h], text_sink) for h in range(H)])
    recall = np.array([_head_recall(M[h], keep[h]) for h in range(H)])
    nnz = keep.reshape(H, -1).sum(axis=1)
    return keep, recall, nnz, targets


def to_csr(keep):
    """keep [R, nb] bool (rows in (b,h,qb) order) -> (row_ptr [R+1], col_idx [nnz])
    with ascending kv-block ids per row."""
    keep = np.asarray(keep, dtype=bool).reshape(-1, np.asarray(keep).shape[-1])
    row_ptr = [0]
    cols = []
    for r in range(keep.shape[0]):
        ids = [j for j in range(keep.shape[1]) if keep[r, j]]
        cols.extend(ids)
        row_ptr.append(len(cols))
    return np.array(row_ptr, dtype=np.int64), np.array(cols, dtype=np.int64)


def brute_force_min_set(masses, forced, candidates, r):
    """Enumerate every subset S of the candidates; among those with
    mass(forced u S) >= r*T return (min |S|, max mass over sets of that size).
    Tiny rows only (2^|candidates| subsets).  Pins select_row_recall's
    minimality: the greedy over sorted masses is optimal for min cardinality."""
    masses = [float(x) for x in masses]
    T = math.fsum(masses)
    base = math.fsum(masses[j] for j in forced)
    target = r * T
    for size in range(0, len(candidates) + 1):
        best = None
        for S in itertools.combinations(candidates, size):
            m = base + math.fsum(masses[j] for j in S)
            if m >= target - 1e-12 * T:
                best = m if best is None else max(best, m)
        if best is not None:
            return size, best
    return None, None
