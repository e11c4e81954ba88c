"""Shared helpers of the -m gpu parity tests: run the oracle on the same seeded tensors and
compare with the tolerances of DESIGN.md §6 (north_star: O max-abs 2e-2 / mean-abs 2e-3,
LSE 1e-3, selection exact outside the 1e-6 tie zone)."""

import math

import numpy as np
import torch

import oracle

O_MAX_ABS = 2e-2
O_MEAN_ABS = 2e-3
LSE_ABS = 1e-3
TIE = 1e-6
# K2 block mass, |dM| / |q-block|.  Per element p = 2^x with x = fma(S, c, -lse*log2e):
# fp32 S = q.k carries |S_raw| * 2^-24 rounding, i.e. |S_scaled| * 2^-24 in the exponent (natural units),
# plus 2^-22 from ex2.approx and 2^-24 from the fma: at |S_scaled| <= 32 the relative error per element is
# <= 32 * 2^-24 + 2^-22 + 2^-24 ~= 2.2e-6, and a block sum inherits it (all terms positive).  2.5x margin.
MASS_REL = 5e-6


def np64(t):
    return t.detach().float().cpu().double().numpy()


def blocks_of(lay_or_desc, B):
    if hasattr(lay_or_desc, "n_video"):
        return oracle.block_map(lay_or_desc.n_video, lay_or_desc.n_text, B, lay_or_desc.text_first)
    raise TypeError


def csr_rows(row_ptr, col_idx):
    rp = row_ptr.cpu().numpy().astype(np.int64)
    ci = col_idx.cpu().numpy()
    return [ci[rp[r]:rp[r + 1]].tolist() for r in range(len(rp) - 1)]


def compare_out(o_gpu, o_ref, lse_gpu=None, lse_ref=None, what=""):
    d = np.abs(np64(o_gpu) - o_ref)
    assert d.max() <= O_MAX_ABS, f"{what}: O max-abs {d.max():.3e}"
    assert d.mean() <= O_MEAN_ABS, f"{what}: O mean-abs {d.mean():.3e}"
    if lse_gpu is not None:
        dl = np.abs(lse_gpu.detach().cpu().double().numpy() - lse_ref)
        assert dl.max() <= LSE_ABS, f"{what}: LSE max-abs {dl.max():.3e}"
    return d.max(), d.mean()


def selection_ok_topk(masses, forced, candidates, k, gpu_kept, oracle_kept):
    """The tie-zone rule for SPARSITY mode (row-wise top-k; R6/R10-R12): the
    GPU keeps the forced set plus exactly k candidates, and (G xor O) lies among candidates whose
    normalised mass is within 1e-6 of the k-th largest (the cut), where several top-k sets exist."""
    m = np.asarray(masses, dtype=np.float64)
    T = m.sum()
    G, O = set(gpu_kept), set(oracle_kept)
    if not set(forced) <= G:
        return False, "forced blocks missing"
    kk = min(k, len(candidates))
    if len(G - set(forced)) != kk:
        return False, f"{len(G - set(forced))} candidates kept, want {kk}"
    if G == O:
        return True, ""
    mh = m / T if T > 0 else m
    order = sorted(candidates, key=lambda j: (-m[j], j))
    c = mh[order[kk - 1]] if kk > 0 else 0.0
    A = {j for j in candidates if abs(mh[j] - c) <= TIE}
    diff = G ^ O
    if not diff <= A:
        return False, f"diff {sorted(diff)} not in tie zone {sorted(A)}"
    return True, ""


def selection_ok(masses, forced, candidates, r, gpu_kept, oracle_kept):
    """north_star tie-zone rule: (G xor O) must lie in the ambiguity set A,
    and G must still reach the recall target (within 1e-6)."""
    m = np.asarray(masses, dtype=np.float64)
    T = m.sum()
    G, O = set(gpu_kept), set(oracle_kept)
    if G == O:
        return True, ""
    mh = m / T if T > 0 else m
    order = sorted(candidates, key=lambda j: (-m[j], j))
    chosen = [j for j in order if j in O]
    kstar = len(chosen)
    c = mh[chosen[-1]] if chosen else 0.0
    A = {j for j in candidates if abs(mh[j] - c) <= TIE}
    P = np.cumsum([mh[j] for j in order]) + sum(mh[j] for j in forced)
    pk1 = P[kstar - 2] if kstar >= 2 else sum(mh[j] for j in forced)
    pk = P[kstar - 1] if kstar >= 1 else pk1
    if pk1 >= r - TIE or pk <= r + TIE:
        for idx in (kstar - 1, kstar):
            if 0 <= idx < len(order):
                A.add(order[idx])
    diff = G ^ O
    if not diff <= A:
        return False, f"diff {sorted(diff)} not in tie zone {sorted(A)}"
    if sum(mh[j] for j in G) < r - TIE:
        return False, "GPU selection misses the recall target"
    return True, ""
