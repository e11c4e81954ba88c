"""Modality-aware block map (oracle; test infrastructure only).

PAPER.md:152-157 (eq:seqlen): the 3D-full-attention sequence is
L = f*h*w + t, video and text tokens in one sequence.
PAPER.md:415-416 (Definition of Blockified Sparse Attention): the length
dimension is partitioned into chunks of B tokens.
PAPER.md:300-310 (Obs. 1) and the north_star's "text/video hierarchical
blockification": readings R14/R15 in DESIGN.md -- each modality segment is
blockified on its own, so no block straddles the text/video boundary, and the
last block of each segment may be partial.
"""

from dataclasses import dataclass
from typing import List


@dataclass(frozen=True)
class Block:
    start: int      # first token index in the sequence
    length: int     # valid tokens (<= B; the segment's last block may be short)
    modality: str   # "video" or "text"


def _segment_blocks(seg_start: int, seg_len: int, B: int, modality: str) -> List[Block]:
    out = []
    pos = 0
    while pos < seg_len:
        out.append(Block(seg_start + pos, min(B, seg_len - pos), modality))
        pos += B
    return out


def block_map(n_video: int, n_text: int, B: int, text_first: bool) -> List[Block]:
    """Blocks in sequence order.  R14: text_first selects [text|video]
    (CogVideoX-shaped) versus [video|text] (HunyuanVideo-shaped)."""
    if B <= 0 or n_video < 0 or n_text < 0 or n_video + n_text <= 0:
        raise ValueError("bad layout")
    if text_first:
        return _segment_blocks(0, n_text, B, "text") + _segment_blocks(n_text, n_video, B, "video")
    return _segment_blocks(0, n_video, B, "video") + _segment_blocks(n_video, n_text, B, "text")


def num_blocks(n_video: int, n_text: int, B: int) -> int:
    return -(-n_video // B) + -(-n_text // B)


def token_block_of(blocks: List[Block]) -> List[int]:
    """token index -> block index, built by walking the blocks (used by the
    brute-force pins, independent of any arithmetic formula)."""
    out = []
    for bi, b in enumerate(blocks):
        out.extend([bi] * b.length)
    return out
