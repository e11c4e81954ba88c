"""fp64 CPU oracle for the AdaSpa hot path (arXiv 2502.21079).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py`` (its ``cpu_baseline`` leg and ``--impl reference`` arm) may import
this package.  The product path (``paper_2502_21079_b200``) never imports it and
shares no code with it: the oracle has its own block map, its own sort and its
own arithmetic, written from PAPER.md in plain numpy / Python.

Every function cites the PAPER.md passage (line + label) it restates.  Where the
paper is silent, garbled or self-contradictory the oracle takes the reading
numbered in DESIGN.md §3 ("Readings"); those numbers are quoted as ``R#``.

Parity status: every function below is pinned by ``tests/test_oracle_*.py``
against something other than itself (library routines, closed forms, brute
force, paper-printed values).  Pins are listed per function in DESIGN.md §4.
No function is "parity unpinned".
"""

from .blocks import Block, block_map, num_blocks, token_block_of
from .attention import dense_attention, block_mass, masked_attention, expand_block_mask
from .select import (
    k_from_sparsity,
    select_row_recall,
    select_row_sparsity,
    head_tiers,
    select_blocks,
    to_csr,
    brute_force_min_set,
    row_forced_and_candidates,
)
from .schedule import schedule_trace

__all__ = [
    "Block", "block_map", "num_blocks", "token_block_of",
    "dense_attention", "block_mass", "masked_attention", "expand_block_mask",
    "k_from_sparsity", "select_row_recall", "select_row_sparsity", "head_tiers",
    "select_blocks", "to_csr", "brute_force_min_set", "row_forced_and_candidates",
    "schedule_trace",
]
