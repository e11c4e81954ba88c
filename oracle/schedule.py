"""AdaSpa step schedule (oracle; test infrastructure only).

PAPER.md:397-405 (fig:overview caption): warm-up steps T_w = {1..t_w}, key steps
T_s = {t_s^1..t_s^k} with t_key^1 = t_w.  Steps 1..t_w-1 run full attention;
step t_w runs the Fused Online Search (full attention + block mass, Alg. 1);
steps t_w+1..t_key^2-1 run block-sparse attention with that mask; each later
key step t_key^i runs the LSE-Cached Online Search (Alg. 2) with the LSE cached
at t_w and uses the new mask from t_key^i itself onward (readings R18, R19).
"""


def schedule_trace(n_steps, t_w, key_steps):
    """Mode of each step 1..n_steps: "full", "full+search", "sparse",
    "cached-search+sparse"."""
    ks = sorted(set(int(x) for x in key_steps))
    if not ks or ks[0] != t_w:
        raise ValueError("first key step must equal t_w (PAPER.md:400, t_key^1 = t_w)")
    if ks[-1] > n_steps or t_w < 1:
        raise ValueError("key steps out of range")
    out = []
    for t in range(1, n_steps + 1):
        if t < t_w:
            out.append("full")
        elif t == t_w:
            out.append("full+search")
        elif t in ks:
            out.append("cached-search+sparse")
        else:
            out.append("sparse")
    return out
