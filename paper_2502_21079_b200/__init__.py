"""B200-native AdaSpa hot path (arXiv 2502.21079).

The four C-ABI entry points of include/adaspa.h, bound through ctypes:

    dense_attn_lse     K1  dense attention forward + LSE           (Alg. 1 pass 1)
    lse_cached_search  K2  block mass sum exp(S - LSE_cached)      (Alg. 2 / Alg. 1 pass 2)
    select_blocks      K3  head-adaptive hierarchical selection -> CSR
    block_sparse_attn  K4  block-sparse attention forward
    dense_attn_lse_search  K1+K2 fused: the search step t_w in one dense pass (Alg. 1)
    search_select      K1+K2+K3 fused: the RECALL-mode search step t_w with the selection epilogue

plus the host schedule (schedule.py), the paper's plug-and-play `adaspa_attention_handler`
(handler.py) and head sharding / Ulysses exchange (dist.py).
Importing fails loudly if libadaspa.so was not built: there is no CPU fallback.
"""

from ._lib import (  # noqa: F401
    AttnDesc, AdaSpaError, Csr, abi_version, make_desc, num_blocks, dense_attn_lse, lse_cached_search,
    dense_attn_lse_search, fused_search_workspace_bytes, search_select, search_select_workspace_bytes,
    select_blocks, block_sparse_attn, sparse_workspace_bytes, SELECT_RECALL, SELECT_SPARSITY,
    FLAG_TEXT_SINK, FLAG_HEAD_TIERS, LIB_PATH,
)
from .handler import AdaSpaAttentionHandler, adaspa_attention_handler  # noqa: F401,E402
