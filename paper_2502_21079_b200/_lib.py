"""Thin ctypes binding over libadaspa.so (include/adaspa.h).

Argument marshalling only: tensors -> (pointer, strides), host targets -> a double
array, the current torch stream -> cudaStream_t.  Every step of the hot path runs
in the CUDA kernels behind the C ABI; there is no Python or CPU fallback.  Importing
this module fails loudly if the library has not been built.
"""

import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ADASPA_LIB") or os.path.join(_HERE, "libadaspa.so")  # override: diagnostic builds

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `python paper_2502_21079_b200/build.py` "
        "(there is no CPU fallback for the AdaSpa kernels)")

_lib = ctypes.CDLL(LIB_PATH)

OK = 0
ERR_INVALID_ARG = 1
ERR_UNSUPPORTED = 2
ERR_CUDA = 3
ERR_WORKSPACE_TOO_SMALL = 4

SELECT_RECALL = 0
SELECT_SPARSITY = 1
FLAG_TEXT_SINK = 1
FLAG_HEAD_TIERS = 2


class AttnDesc(ctypes.Structure):
    _fields_ = [
        ("batch", ctypes.c_int32), ("heads", ctypes.c_int32), ("seq_len", ctypes.c_int32),
        ("head_dim", ctypes.c_int32), ("block_size", ctypes.c_int32), ("n_text", ctypes.c_int32),
        ("text_first", ctypes.c_int32), ("softmax_scale", ctypes.c_float),
        ("stride_b", ctypes.c_int64), ("stride_h", ctypes.c_int64), ("stride_n", ctypes.c_int64),
    ]


class PeerHandle(ctypes.Structure):
    """adaspa_peer_handle: CUDA IPC handle of an allocation + the pointer's byte offset in it."""
    _fields_ = [("handle", ctypes.c_uint8 * 64), ("offset", ctypes.c_int64)]


_P = ctypes.c_void_p
_D = ctypes.POINTER(AttnDesc)
_PH = ctypes.POINTER(PeerHandle)

SYMBOLS = {
    "adaspa_abi_version": (ctypes.c_int32, []),
    "adaspa_num_blocks": (ctypes.c_int32, [_D]),
    "adaspa_dense_attn_lse": (ctypes.c_int, [_D, _P, _P, _P, _P, _P, _P]),
    "adaspa_lse_cached_search": (ctypes.c_int, [_D, _P, _P, _P, _P, _P]),
    "adaspa_dense_attn_lse_search": (ctypes.c_int, [_D, _P, _P, _P, _P, _P, _P, _P, ctypes.c_size_t, _P]),
    "adaspa_fused_search_workspace_bytes": (ctypes.c_size_t, [_D, ctypes.c_int32]),
    "adaspa_search_select": (ctypes.c_int, [_D, _P, _P, _P, _P, _P, _P, ctypes.POINTER(ctypes.c_double),
                                             ctypes.c_uint32, _P, _P, ctypes.c_int64, _P, _P, _P, _P,
                                             ctypes.c_size_t, _P]),
    "adaspa_search_select_workspace_bytes": (ctypes.c_size_t, [_D, ctypes.c_int32]),
    "adaspa_select_workspace_bytes": (ctypes.c_size_t, [_D]),
    "adaspa_select_blocks": (ctypes.c_int, [_D, _P, ctypes.c_int, ctypes.POINTER(ctypes.c_double), ctypes.c_uint32,
                                             ctypes.c_double, _P, _P, ctypes.c_int64, _P, _P, _P, _P,
                                             ctypes.c_size_t, _P]),
    "adaspa_sparse_workspace_bytes": (ctypes.c_size_t, [_D]),
    "adaspa_block_sparse_attn": (ctypes.c_int, [_D, _P, _P, _P, _P, _P, _P, _P, _P, ctypes.c_size_t, _P]),
    "adaspa_peer_export": (ctypes.c_int, [_P, _PH]),
    "adaspa_peer_import": (ctypes.c_int, [_PH, ctypes.POINTER(_P), ctypes.POINTER(_P)]),
    "adaspa_peer_close": (ctypes.c_int, [_P]),
    "adaspa_peer_copy2d": (ctypes.c_int, [_P, ctypes.c_int64, _P, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, _P]),
    "adaspa_peer_signal": (ctypes.c_int, [_P, ctypes.c_uint32, _P]),
    "adaspa_peer_wait": (ctypes.c_int, [_P, ctypes.c_int32, ctypes.c_uint32, _P]),
    "adaspa_peer_last_error": (ctypes.c_char_p, []),
    "adaspa_status_string": (ctypes.c_char_p, [ctypes.c_int]),
    "adaspa_last_error": (ctypes.c_char_p, []),
}

for _name, (_res, _args) in SYMBOLS.items():
    _fn = getattr(_lib, _name)
    _fn.restype = _res
    _fn.argtypes = _args


class AdaSpaError(RuntimeError):
    def __init__(self, status, where):
        self.status = status
        msg = _lib.adaspa_last_error().decode()
        super().__init__(f"{where}: {_lib.adaspa_status_string(status).decode()}: {msg}")


def _check(status, where):
    if status != OK:
        raise AdaSpaError(status, where)


def abi_version():
    return int(_lib.adaspa_abi_version())


def make_desc(q, block_size, n_text, text_first=False, softmax_scale=0.0):
    """Descriptor for q viewed as [B, H, N, d] (any strides with stride(-1) == 1)."""
    if q.dim() != 4:
        raise ValueError("expected a 4-D [B, H, N, d] view")
    B, H, N, d = q.shape
    sb, sh, sn, sd = q.stride()
    if sd != 1:
        raise ValueError("head_dim must be contiguous (stride 1)")
    return AttnDesc(B, H, N, d, int(block_size), int(n_text), 1 if text_first else 0,
                    float(softmax_scale), sb, sh, sn)


def num_blocks(desc):
    return int(_lib.adaspa_num_blocks(ctypes.byref(desc)))


def _stream(stream):
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def _scratch(nbytes, device, stream):
    """Scratch owned by one call: if the call runs on a stream other than the current one, tell the
    caching allocator, so that the block is not handed out again before that stream is done."""
    t = torch.empty(nbytes, dtype=torch.uint8, device=device)
    if stream is not None and stream != torch.cuda.current_stream(device):
        t.record_stream(stream)
    return t


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else ctypes.c_void_p(0)


def _same_layout(desc, *ts):
    for t in ts:
        if t.dtype != torch.bfloat16 or not t.is_cuda:
            raise TypeError("Q/K/V/O must be bf16 CUDA tensors")
        if tuple(t.shape) != (desc.batch, desc.heads, desc.seq_len, desc.head_dim):
            raise ValueError("Q/K/V/O shapes differ")
        # a dimension of extent 1 is never stepped over, so its stride does not matter (a Ulysses
        # as_bhnd view [1, Hp, N, d] has stride_b = Hp*d, a [B, N, H, d] buffer N*H*d)
        want = (desc.stride_b, desc.stride_h, desc.stride_n, 1)
        if any(n > 1 and s != w for n, s, w in zip(t.shape, t.stride(), want)):
            raise ValueError("Q/K/V/O must share one layout (strides)")


def _check_f32(t, shape, name):
    if t.dtype != torch.float32 or not t.is_cuda or not t.is_contiguous() or tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name} must be a contiguous fp32 CUDA tensor of shape {tuple(shape)}")


def dense_attn_lse(q, k, v, *, block_size, n_text, text_first=False, softmax_scale=0.0, o=None, lse=None,
                   want_lse=True, stream=None):
    """K1: O = softmax(scale Q K^T) V and the per-row LSE.  Returns (o, lse)."""
    desc = make_desc(q, block_size, n_text, text_first, softmax_scale)
    if o is None:
        o = torch.empty_like(q)
    _same_layout(desc, q, k, v, o)
    if lse is None and want_lse:
        lse = torch.empty(desc.batch, desc.heads, desc.seq_len, dtype=torch.float32, device=q.device)
    if lse is not None:
        _check_f32(lse, (desc.batch, desc.heads, desc.seq_len), "lse")
    _check(_lib.adaspa_dense_attn_lse(ctypes.byref(desc), _ptr(q), _ptr(k), _ptr(v), _ptr(o), _ptr(lse),
                                      _stream(stream)), "adaspa_dense_attn_lse")
    return o, lse


def fused_search_workspace_bytes(desc, heads_per_pass=0):
    return int(_lib.adaspa_fused_search_workspace_bytes(ctypes.byref(desc), int(heads_per_pass)))


def dense_attn_lse_search(q, k, v, *, block_size, n_text, text_first=False, softmax_scale=0.0, o=None, lse=None,
                          block_mass=None, workspace=None, heads_per_pass=0, stream=None):
    """K1 + K2 fused (the search step t_w, Alg. 1 in one dense pass): O, the row LSE and the block
    masses with that LSE.  workspace: a uint8 CUDA tensor (allocated for `heads_per_pass` heads if
    None; 0 = all heads in one pass).  Returns (o, lse, block_mass)."""
    desc = make_desc(q, block_size, n_text, text_first, softmax_scale)
    if o is None:
        o = torch.empty_like(q)
    _same_layout(desc, q, k, v, o)
    nb = num_blocks(desc)
    if lse is None:
        lse = torch.empty(desc.batch, desc.heads, desc.seq_len, dtype=torch.float32, device=q.device)
    _check_f32(lse, (desc.batch, desc.heads, desc.seq_len), "lse")
    if block_mass is None:
        block_mass = torch.empty(desc.batch, desc.heads, nb, nb, dtype=torch.float32, device=q.device)
    _check_f32(block_mass, (desc.batch, desc.heads, nb, nb), "block_mass")
    if workspace is None:
        workspace = _scratch(fused_search_workspace_bytes(desc, heads_per_pass), q.device, stream)
    if workspace.dtype != torch.uint8 or not workspace.is_cuda:
        raise ValueError("workspace must be a uint8 CUDA tensor")
    _check(_lib.adaspa_dense_attn_lse_search(ctypes.byref(desc), _ptr(q), _ptr(k), _ptr(v), _ptr(o), _ptr(lse),
                                             _ptr(block_mass), _ptr(workspace), workspace.numel(),
                                             _stream(stream)), "adaspa_dense_attn_lse_search")
    return o, lse, block_mass


def lse_cached_search(q, k, lse, *, block_size, n_text, text_first=False, softmax_scale=0.0, block_mass=None,
                      stream=None):
    """K2: block_mass[b,h,p,j] = sum exp(scale q.k - lse).  Returns block_mass [B,H,nb,nb] fp32."""
    desc = make_desc(q, block_size, n_text, text_first, softmax_scale)
    _same_layout(desc, q, k)
    nb = num_blocks(desc)
    _check_f32(lse, (desc.batch, desc.heads, desc.seq_len), "lse")
    if block_mass is None:
        block_mass = torch.empty(desc.batch, desc.heads, nb, nb, dtype=torch.float32, device=q.device)
    _check_f32(block_mass, (desc.batch, desc.heads, nb, nb), "block_mass")
    _check(_lib.adaspa_lse_cached_search(ctypes.byref(desc), _ptr(q), _ptr(k), _ptr(lse), _ptr(block_mass),
                                         _stream(stream)), "adaspa_lse_cached_search")
    return block_mass


class Csr:
    """Selection result (device tensors) of adaspa_select_blocks."""

    def __init__(self, row_ptr, col_idx, row_order, head_recall, head_nnz):
        self.row_ptr = row_ptr
        self.col_idx = col_idx
        self.row_order = row_order
        self.head_recall = head_recall
        self.head_nnz = head_nnz


def select_blocks(block_mass, *, heads_desc, mode, target, flags=FLAG_TEXT_SINK, tier_tau=0.8, out=None,
                  want_row_order=True, stream=None):
    """K3: per-head selection to CSR.  heads_desc is an AttnDesc (from make_desc) giving the
    layout/modality split; target is a per-head sequence of recall or sparsity values."""
    desc = heads_desc
    nb = num_blocks(desc)
    B, H = desc.batch, desc.heads
    _check_f32(block_mass, (B, H, nb, nb), "block_mass")
    tgt = [float(x) for x in target]
    if len(tgt) != H:
        raise ValueError(f"need {H} per-head targets, got {len(tgt)}")
    tarr = (ctypes.c_double * H)(*tgt)
    dev = block_mass.device
    rows = B * H * nb
    if out is None:
        out = Csr(torch.empty(rows + 1, dtype=torch.int32, device=dev),
                  torch.empty(rows * nb, dtype=torch.int32, device=dev),
                  torch.empty(rows, dtype=torch.int32, device=dev) if want_row_order else None,
                  torch.empty(B, H, dtype=torch.float32, device=dev),
                  torch.empty(B, H, dtype=torch.int64, device=dev))
    wsb = int(_lib.adaspa_select_workspace_bytes(ctypes.byref(desc)))
    ws = _scratch(max(wsb, 1), dev, stream)
    _check(_lib.adaspa_select_blocks(ctypes.byref(desc), _ptr(block_mass), int(mode), tarr, int(flags),
                                     float(tier_tau), _ptr(out.row_ptr), _ptr(out.col_idx), out.col_idx.numel(),
                                     _ptr(out.row_order), _ptr(out.head_recall), _ptr(out.head_nnz), _ptr(ws),
                                     wsb, _stream(stream)), "adaspa_select_blocks")
    return out


def search_select_workspace_bytes(desc, heads_per_pass=0):
    return int(_lib.adaspa_search_select_workspace_bytes(ctypes.byref(desc), int(heads_per_pass)))


def search_select(q, k, v, *, block_size, n_text, target, text_first=False, softmax_scale=0.0,
                  flags=FLAG_TEXT_SINK, o=None, lse=None, block_mass=None, want_block_mass=True, out=None,
                  want_row_order=True, workspace=None, heads_per_pass=0, stream=None):
    """K1 + K2 + K3 fused: the whole RECALL-mode search step t_w (adaspa_search_select).  target: per-head
    recall r_h.  block_mass is written only if given or want_block_mass (required when nb > 2048).
    Returns (o, lse, block_mass or None, Csr)."""
    desc = make_desc(q, block_size, n_text, text_first, softmax_scale)
    if o is None:
        o = torch.empty_like(q)
    _same_layout(desc, q, k, v, o)
    nb = num_blocks(desc)
    B, H = desc.batch, desc.heads
    dev = q.device
    if lse is None:
        lse = torch.empty(B, H, desc.seq_len, dtype=torch.float32, device=dev)
    _check_f32(lse, (B, H, desc.seq_len), "lse")
    if block_mass is None and (want_block_mass or nb > 2048):
        block_mass = torch.empty(B, H, nb, nb, dtype=torch.float32, device=dev)
    if block_mass is not None:
        _check_f32(block_mass, (B, H, nb, nb), "block_mass")
    tgt = [float(x) for x in target]
    if len(tgt) != H:
        raise ValueError(f"need {H} per-head targets, got {len(tgt)}")
    tarr = (ctypes.c_double * H)(*tgt)
    rows = B * H * nb
    if out is None:
        out = Csr(torch.empty(rows + 1, dtype=torch.int32, device=dev),
                  torch.empty(rows * nb, dtype=torch.int32, device=dev),
                  torch.empty(rows, dtype=torch.int32, device=dev) if want_row_order else None,
                  torch.empty(B, H, dtype=torch.float32, device=dev),
                  torch.empty(B, H, dtype=torch.int64, device=dev))
    if workspace is None:
        workspace = _scratch(search_select_workspace_bytes(desc, heads_per_pass), dev, stream)
    if workspace.dtype != torch.uint8 or not workspace.is_cuda:
        raise ValueError("workspace must be a uint8 CUDA tensor")
    _check(_lib.adaspa_search_select(ctypes.byref(desc), _ptr(q), _ptr(k), _ptr(v), _ptr(o), _ptr(lse),
                                     _ptr(block_mass), tarr, int(flags), _ptr(out.row_ptr), _ptr(out.col_idx),
                                     out.col_idx.numel(), _ptr(out.row_order), _ptr(out.head_recall),
                                     _ptr(out.head_nnz), _ptr(workspace), workspace.numel(), _stream(stream)),
           "adaspa_search_select")
    return o, lse, block_mass, out


def sparse_workspace_bytes(desc):
    return int(_lib.adaspa_sparse_workspace_bytes(ctypes.byref(desc)))


def block_sparse_attn(q, k, v, row_ptr, col_idx, *, block_size, n_text, text_first=False, softmax_scale=0.0,
                      o=None, lse=None, want_lse=False, workspace=None, stream=None):
    """K4: block-sparse attention over the CSR.  Returns (o, lse or None)."""
    desc = make_desc(q, block_size, n_text, text_first, softmax_scale)
    if o is None:
        o = torch.empty_like(q)
    _same_layout(desc, q, k, v, o)
    if lse is None and want_lse:
        lse = torch.empty(desc.batch, desc.heads, desc.seq_len, dtype=torch.float32, device=q.device)
    if lse is not None:
        _check_f32(lse, (desc.batch, desc.heads, desc.seq_len), "lse")
    for t, nm in ((row_ptr, "row_ptr"), (col_idx, "col_idx")):
        if t.dtype != torch.int32 or not t.is_cuda or not t.is_contiguous():
            raise ValueError(f"{nm} must be a contiguous int32 CUDA tensor")
    rows = desc.batch * desc.heads * num_blocks(desc)
    if row_ptr.numel() < rows + 1:
        raise ValueError(f"row_ptr has {row_ptr.numel()} entries, the CSR needs B*H*nb+1 = {rows + 1}")
    wsb = sparse_workspace_bytes(desc)
    if workspace is None or workspace.numel() < wsb:
        workspace = _scratch(max(wsb, 1), q.device, stream)
    _check(_lib.adaspa_block_sparse_attn(ctypes.byref(desc), _ptr(q), _ptr(k), _ptr(v), _ptr(row_ptr),
                                         _ptr(col_idx), _ptr(o), _ptr(lse), _ptr(workspace), workspace.numel(),
                                         _stream(stream)), "adaspa_block_sparse_attn")
    return o, lse


# ---------------------------------------------------------------- peer-memory plumbing (multi-GPU)
def _peer_check(status, where):
    if status != OK:
        raise RuntimeError(f"{where}: {_lib.adaspa_status_string(status).decode()}: "
                           f"{_lib.adaspa_peer_last_error().decode()}")


def peer_export(ptr):
    """IPC handle (bytes) of a device pointer: CUDA IPC handle of its allocation + the byte offset."""
    h = PeerHandle()
    _peer_check(_lib.adaspa_peer_export(ctypes.c_void_p(ptr), ctypes.byref(h)), "adaspa_peer_export")
    return bytes(h.handle) + int(h.offset).to_bytes(8, "little", signed=True)


def peer_import(blob):
    """Map a peer process's exported pointer: returns (device pointer, base to close)."""
    h = PeerHandle()
    ctypes.memmove(h.handle, blob[:64], 64)
    h.offset = int.from_bytes(blob[64:72], "little", signed=True)
    ptr, base = ctypes.c_void_p(), ctypes.c_void_p()
    _peer_check(_lib.adaspa_peer_import(ctypes.byref(h), ctypes.byref(ptr), ctypes.byref(base)), "adaspa_peer_import")
    return ptr.value, base.value


def peer_close(base):
    _peer_check(_lib.adaspa_peer_close(ctypes.c_void_p(base)), "adaspa_peer_close")


def peer_copy2d(dst, dst_pitch, src, src_pitch, width, rows, stream=None):
    _peer_check(_lib.adaspa_peer_copy2d(ctypes.c_void_p(dst), dst_pitch, ctypes.c_void_p(src), src_pitch, width, rows,
                                        _stream(stream)), "adaspa_peer_copy2d")


def peer_signal(flag_ptr, value, stream=None):
    _peer_check(_lib.adaspa_peer_signal(ctypes.c_void_p(flag_ptr), value, _stream(stream)), "adaspa_peer_signal")


def peer_wait(flags_ptr, n, value, stream=None):
    _peer_check(_lib.adaspa_peer_wait(ctypes.c_void_p(flags_ptr), n, value, _stream(stream)), "adaspa_peer_wait")
