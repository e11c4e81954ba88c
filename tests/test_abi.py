"""CPU-side checks of the C ABI: the library loads, exports every symbol include/adaspa.h
declares, and rejects bad arguments before touching the GPU (no kernel launch here)."""

import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_functions():
    src = open(os.path.join(ROOT, "include", "adaspa.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(adaspa_[a-z_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    import paper_2502_21079_b200.build as b
    b.build()
    from paper_2502_21079_b200 import _lib
    return _lib


def test_exports_every_header_symbol(lib):
    names = _header_functions()
    assert len(names) == 20, names
    for n in names:
        assert hasattr(lib._lib, n), n
        assert n in lib.SYMBOLS, n


def test_abi_version(lib):
    assert lib.abi_version() == 1


def _desc(lib, **kw):
    d = dict(batch=1, heads=24, seq_len=111856, head_dim=128, block_size=128, n_text=256, text_first=0,
             softmax_scale=0.0, stride_b=24 * 111856 * 128, stride_h=111856 * 128, stride_n=128)
    d.update(kw)
    return lib.AttnDesc(**d)


def test_num_blocks_matches_paper_geometry(lib):
    # PAPER.md:152-157 / SURVEY 8(d): HYV-110K nb = 872 + 2, CogX-45K nb = 4 + 702, HYV-129f 929 + 2
    assert lib.num_blocks(_desc(lib)) == 874
    assert lib.num_blocks(_desc(lib, heads=48, seq_len=45106, head_dim=64, block_size=64, n_text=226,
                                text_first=1, stride_b=48 * 45106 * 64, stride_h=45106 * 64, stride_n=64)) == 706
    assert lib.num_blocks(_desc(lib, seq_len=119056)) == 931
    assert lib.num_blocks(_desc(lib, head_dim=96)) == -1


def _status(lib, fn, *args):
    return fn(*args)


def test_rejects_bad_arguments_without_launch(lib):
    L = lib._lib
    nul = ctypes.c_void_p(0)
    fake = ctypes.c_void_p(0x10000)   # aligned, never dereferenced: validation fails first
    d = _desc(lib, head_dim=96)
    assert L.adaspa_dense_attn_lse(ctypes.byref(d), fake, fake, fake, fake, nul, nul) == lib.ERR_UNSUPPORTED
    d = _desc(lib, block_size=32)
    assert L.adaspa_lse_cached_search(ctypes.byref(d), fake, fake, fake, fake, nul) == lib.ERR_UNSUPPORTED
    d = _desc(lib)
    assert L.adaspa_dense_attn_lse(ctypes.byref(d), nul, fake, fake, fake, nul, nul) == lib.ERR_INVALID_ARG
    assert b"q is NULL" in L.adaspa_last_error()
    mis = ctypes.c_void_p(0x10008)
    assert L.adaspa_dense_attn_lse(ctypes.byref(d), fake, mis, fake, fake, nul, nul) == lib.ERR_INVALID_ARG
    d = _desc(lib, n_text=200000)
    assert L.adaspa_dense_attn_lse(ctypes.byref(d), fake, fake, fake, fake, nul, nul) == lib.ERR_INVALID_ARG
    d = _desc(lib, stride_n=100)
    assert L.adaspa_dense_attn_lse(ctypes.byref(d), fake, fake, fake, fake, nul, nul) == lib.ERR_INVALID_ARG


def test_select_argument_rules(lib):
    L = lib._lib
    fake = ctypes.c_void_p(0x10000)
    nul = ctypes.c_void_p(0)
    d = _desc(lib, heads=2, seq_len=512, head_dim=64, block_size=64, n_text=64, stride_b=2 * 512 * 64,
              stride_h=512 * 64, stride_n=64)
    nb = lib.num_blocks(d)
    cap = 2 * nb * nb
    ws = int(L.adaspa_select_workspace_bytes(ctypes.byref(d)))
    assert ws > 0

    def call(mode, tgt, flags=1, capacity=cap, wsb=ws):
        arr = (ctypes.c_double * 2)(*tgt)
        return L.adaspa_select_blocks(ctypes.byref(d), fake, mode, arr, flags, 0.8, fake, fake, capacity, nul,
                                      nul, nul, fake, wsb, nul)
    assert call(lib.SELECT_SPARSITY, [1.0, 0.5]) == lib.ERR_INVALID_ARG          # s must be < 1
    assert call(lib.SELECT_SPARSITY, [0.2, 0.5], flags=3) == lib.ERR_INVALID_ARG  # tiers need s >= 1/3
    assert call(lib.SELECT_RECALL, [0.9, 0.9], flags=3) == lib.ERR_INVALID_ARG    # tiers: sparsity mode only
    assert call(lib.SELECT_RECALL, [float("nan"), 0.9]) == lib.ERR_INVALID_ARG
    assert call(lib.SELECT_RECALL, [0.9, 0.9], capacity=cap - 1) == lib.ERR_INVALID_ARG
    assert call(lib.SELECT_RECALL, [0.9, 0.9], wsb=ws - 1) == lib.ERR_WORKSPACE_TOO_SMALL
    assert call(lib.SELECT_RECALL, [0.9, 0.9], flags=8) == lib.ERR_INVALID_ARG


def test_sparse_workspace_and_errors(lib):
    L = lib._lib
    d = _desc(lib)
    assert lib.sparse_workspace_bytes(d) > 0
    fake = ctypes.c_void_p(0x10000)
    nul = ctypes.c_void_p(0)
    st = L.adaspa_block_sparse_attn(ctypes.byref(d), fake, fake, fake, nul, fake, fake, nul, fake, 1 << 40, nul)
    assert st == lib.ERR_INVALID_ARG
    st = L.adaspa_block_sparse_attn(ctypes.byref(d), fake, fake, fake, fake, fake, fake, nul, fake, 16, nul)
    assert st == lib.ERR_WORKSPACE_TOO_SMALL


def test_fused_search_workspace_and_errors(lib):
    """adaspa_dense_attn_lse_search: workspace sizing (4*(nb+1)*N bytes per head and batch element,
    passes of as many heads as fit) and argument errors rejected before any launch."""
    L = lib._lib
    d = _desc(lib)
    nb = lib.num_blocks(d)
    per = 4 * (nb + 1) * d.seq_len * d.batch
    assert lib.fused_search_workspace_bytes(d, 1) == per
    assert lib.fused_search_workspace_bytes(d, 0) == per * d.heads
    assert lib.fused_search_workspace_bytes(d, 99) == per * d.heads
    fake = ctypes.c_void_p(0x10000)
    nul = ctypes.c_void_p(0)
    st = L.adaspa_dense_attn_lse_search(ctypes.byref(d), fake, fake, fake, fake, fake, fake, fake, per - 1, nul)
    assert st == lib.ERR_WORKSPACE_TOO_SMALL
    st = L.adaspa_dense_attn_lse_search(ctypes.byref(d), fake, fake, fake, fake, fake, nul, fake, per, nul)
    assert st == lib.ERR_INVALID_ARG and b"block_mass" in L.adaspa_last_error()
    st = L.adaspa_dense_attn_lse_search(ctypes.byref(d), nul, fake, fake, fake, fake, fake, fake, per, nul)
    assert st == lib.ERR_INVALID_ARG


def test_search_select_workspace_and_errors(lib):
    """adaspa_search_select (the whole RECALL search step t_w): workspace = the K3 workspace (256-B
    aligned) + the fused-search scratch per head pass; argument errors rejected before any launch."""
    L = lib._lib
    d = _desc(lib)
    nb = lib.num_blocks(d)
    per = 4 * (nb + 1) * d.seq_len * d.batch
    sel = int(L.adaspa_select_workspace_bytes(ctypes.byref(d)))
    sel = (sel + 255) // 256 * 256
    assert lib.search_select_workspace_bytes(d, 1) == sel + per
    assert lib.search_select_workspace_bytes(d, 0) == sel + per * d.heads
    fake = ctypes.c_void_p(0x10000)
    nul = ctypes.c_void_p(0)
    H = d.heads
    ok = (ctypes.c_double * H)(*([0.9] * H))
    cap = d.batch * H * nb * nb

    def call(q=fake, mass=fake, tgt=ok, flags=1, rp=fake, cap=cap, ws=sel + per):
        return L.adaspa_search_select(ctypes.byref(d), q, fake, fake, fake, fake, mass, tgt, flags, rp, fake, cap,
                                      nul, nul, nul, fake, ws, nul)

    assert call(ws=sel + per - 1) == lib.ERR_WORKSPACE_TOO_SMALL
    assert call(q=nul) == lib.ERR_INVALID_ARG
    assert call(rp=nul) == lib.ERR_INVALID_ARG
    assert call(cap=cap - 1) == lib.ERR_INVALID_ARG
    assert call(flags=3) == lib.ERR_INVALID_ARG and b"TIERS" in L.adaspa_last_error()
    bad = (ctypes.c_double * H)(*([float("nan")] * H))
    assert call(tgt=bad) == lib.ERR_INVALID_ARG


def test_search_select_needs_block_mass_above_2048_blocks(lib):
    """nb > 2048: the selection runs on the written masses, so block_mass = NULL is an argument error."""
    L = lib._lib
    d = lib.AttnDesc(1, 1, 140000, 64, 64, 0, 0, 0.0, 140000 * 64, 140000 * 64, 64)
    assert lib.num_blocks(d) > 2048
    fake = ctypes.c_void_p(0x10000)
    nul = ctypes.c_void_p(0)
    nb = lib.num_blocks(d)
    ws = lib.search_select_workspace_bytes(d, 0)
    tg = (ctypes.c_double * 1)(0.9)
    st = L.adaspa_search_select(ctypes.byref(d), fake, fake, fake, fake, fake, nul, tg, 1, fake, fake, nb * nb,
                                nul, nul, nul, fake, ws, nul)
    assert st == lib.ERR_INVALID_ARG and b"2048" in L.adaspa_last_error()


def test_peer_plumbing_rejects_bad_arguments(lib):
    """The peer-memory exchange entries reject NULL / inconsistent arguments before touching CUDA."""
    L = lib._lib
    nul = ctypes.c_void_p(0)
    fake = ctypes.c_void_p(0x10000)
    assert L.adaspa_peer_export(nul, None) == lib.ERR_INVALID_ARG
    assert L.adaspa_peer_import(None, None, None) == lib.ERR_INVALID_ARG
    assert L.adaspa_peer_close(nul) == lib.ERR_INVALID_ARG
    assert L.adaspa_peer_copy2d(fake, 16, fake, 16, 32, 4, nul) == lib.ERR_INVALID_ARG   # pitch < width
    assert L.adaspa_peer_copy2d(fake, 64, fake, 64, 0, 4, nul) == lib.OK                  # empty copy: no-op
    assert L.adaspa_peer_signal(nul, 1, nul) == lib.ERR_INVALID_ARG
    assert L.adaspa_peer_wait(nul, 2, 1, nul) == lib.ERR_INVALID_ARG
    assert b"flags" in L.adaspa_peer_last_error()
