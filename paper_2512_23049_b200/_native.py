"""ctypes binding of the sm_100a C-ABI library (include/choreo_b200.h).

There is no fallback: if the in-tree ``_choreo_b200.so`` is missing or fails to
load, every engine entry point raises ``NativeError``.  Build it with
``python -m paper_2512_23049_b200.build`` (or ``__graft_entry__.build()``).
"""

from __future__ import annotations

import ctypes
import os

from .errors import NativeError

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_choreo_b200.so")

F32 = 0
BF16 = 1

_P = ctypes.c_void_p
_I = ctypes.c_int
_F = ctypes.c_float

# name -> argtypes (all functions return int status)
SIGNATURES: dict[str, list] = {
    "choreo_embed": [_P, _I, _I, _P, _I, _P, _P],
    "choreo_embed_select": [_P, _I, _I, _P, _P, _P, _I, _P, _P],
    "choreo_residual_rmsnorm": [_P, _P, _I, _I, _P, _I, _I, _I, _F, _P, _I, _I, _P, _I, _P],
    "choreo_silu_mul": [_P, _I, _I, _I, _I, _P, _I, _I, _P],
    "choreo_rope_append": [_P, _I, _I, _I, _I, _P, _P, _P, _P, _P, _P, _I, _I, _I, _I, _I, _I,
                           _I, _P, _P, _I, _P],
    "choreo_rerotate": [_P, _I, _I, _I, _I, _I, _I, _P, _P, _P, _I, _P, _P, _I, _P],
    "choreo_assemble": [_P, _P, _P, _P, _P, _I, _P, _I, _P, _I, _I, _I, _I, _P, _P, _P, _P, _P,
                        _P, _P, _P, _I, _I, _I, _I, _I, _P, _P],
    "choreo_attn_split": [_P, _P, _P, _I, _I, _I, _I, _I, _I, _I, _P, _P, _P, _P, _P, _P, _P,
                          _I, _P, _P, _I, _P],
    "choreo_prefill_attn": [_P, _P, _P, _I, _I, _I, _I, _I, _I, _I, _I, _P, _P, _P, _P, _P,
                            _P, _P, _I, _P, _P, _I, _P, _I, _I, _P],
    "choreo_attn_combine": [_P, _P, _P, _P, _I, _I, _I, _P, _I, _I, _P],
    "choreo_select_greedy": [_P, _I, _I, _I, _I, _P, _P],
    "choreo_selftest_umma": [_P, _P, _P, _P, _P, _P, _P],
    "choreo_linear_skinny": [_P, _I, _I, _P, _I, _I, _P, _P, _P, _I, _P],
    "choreo_decode_layers": [_P, _P],
    "choreo_linear_skinny_pieces": [_P, _I, _I, _P, _I, _I, _P, _P, _P, _I, _P, _P],
    "choreo_rope_append_pieces": [_P, _I, _P, _P, _P, _P, _P, _P, _I, _I, _I, _I, _I, _I, _I, _P,
                                  _P, _I, _P],
    "choreo_residual_rmsnorm_pieces": [_P, _P, _P, _I, _I, _I, _F, _P, _I, _I, _P],
    "choreo_linear_gate_up_silu": [_P, _I, _I, _P, _I, _I, _P, _P, _P, _P],
    "choreo_select_nucleus": [_P, _I, _I, _I, _P, _P, _P, _P],
    "choreo_decode_attn_v2": [_P, _P, _P, _I, _I, _I, _I, _I, _I, _I, _P, _P, _P, _P, _P, _P, _P,
                              _I, _P, _P, _P, _I, _P],
    "choreo_layer_chain": [_P, _P],
    "choreo_chain_prologue": [_P, _P, _I, _I, _P, _P, _I, _P, _P],
    "choreo_rope_append_pieces_ex": [_P, _I, _P, _P, _P, _P, _P, _P, _I, _I, _I, _I, _I, _I, _I,
                                     _P, _P, _I, _P, _F, _P],
    "choreo_decode_attn_v2_ex": [_P, _P, _P, _I, _I, _I, _I, _I, _I, _I, _P, _P, _P, _P, _P,
                                 _P, _P, _I, _P, _P, _P, _I, _P, _P, _I, _P],
    "choreo_assemble_ex": [_P, _P, _P, _P, _P, _I, _P, _I, _P, _I, _I, _I, _I, _P, _P, _P, _P,
                           _P, _P, _P, _P, _I, _I, _I, _I, _I, _P, _P, _I, _P],
    "choreo_events_create": [_P, _I],
    "choreo_events_elapsed": [_P, _I, _P],
    "choreo_events_destroy": [_P, _I],
}
EXTRA = ["choreo_abi_version", "choreo_last_error"]

_lib = None


def load() -> ctypes.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise NativeError(f"CUDA extension not built: {LIB_PATH} is missing "
                          "(run `python -m paper_2512_23049_b200.build`); there is no CPU fallback")
    try:
        lib = ctypes.CDLL(LIB_PATH)
    except OSError as exc:
        raise NativeError(f"cannot load {LIB_PATH}: {exc}") from exc
    for name, args in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = ctypes.c_int
    lib.choreo_abi_version.restype = ctypes.c_int
    lib.choreo_last_error.restype = ctypes.c_char_p
    _lib = lib
    return lib


class _Caller:
    def __init__(self, name: str) -> None:
        self.name = name
        self.fn = None

    def __call__(self, *args) -> None:
        if self.fn is None:
            self.fn = getattr(load(), self.name)
        rc = self.fn(*args)
        if rc != 0:
            msg = load().choreo_last_error().decode(errors="replace")
            raise NativeError(f"{self.name} failed with code {rc}: {msg}")


embed = _Caller("choreo_embed")
embed_select = _Caller("choreo_embed_select")
residual_rmsnorm = _Caller("choreo_residual_rmsnorm")
linear_skinny_pieces = _Caller("choreo_linear_skinny_pieces")
rope_append_pieces = _Caller("choreo_rope_append_pieces")
residual_rmsnorm_pieces = _Caller("choreo_residual_rmsnorm_pieces")


class K7Pieces(ctypes.Structure):
    """Mirror of ChoreoK7Pieces (include/choreo_b200.h): a deferred K7 output."""
    _fields_ = [("y", ctypes.c_void_p), ("ws", ctypes.c_void_p), ("n", ctypes.c_int),
                ("kb", ctypes.c_int), ("iters", ctypes.c_int), ("grid", ctypes.c_int),
                ("nx", ctypes.c_int), ("split", ctypes.c_int)]
silu_mul = _Caller("choreo_silu_mul")
rope_append = _Caller("choreo_rope_append")
rerotate = _Caller("choreo_rerotate")
assemble = _Caller("choreo_assemble")
assemble_ex = _Caller("choreo_assemble_ex")
attn_split = _Caller("choreo_attn_split")
attn_combine = _Caller("choreo_attn_combine")
prefill_attn = _Caller("choreo_prefill_attn")
select_greedy = _Caller("choreo_select_greedy")
selftest_umma = _Caller("choreo_selftest_umma")
linear_skinny = _Caller("choreo_linear_skinny")
decode_layers = _Caller("choreo_decode_layers")
linear_gate_up_silu = _Caller("choreo_linear_gate_up_silu")
select_nucleus = _Caller("choreo_select_nucleus")
decode_attn_v2 = _Caller("choreo_decode_attn_v2")
decode_attn_v2_ex = _Caller("choreo_decode_attn_v2_ex")
rope_append_pieces_ex = _Caller("choreo_rope_append_pieces_ex")
layer_chain = _Caller("choreo_layer_chain")
chain_prologue = _Caller("choreo_chain_prologue")
events_create = _Caller("choreo_events_create")
events_elapsed = _Caller("choreo_events_elapsed")
events_destroy = _Caller("choreo_events_destroy")


class DecodeStep(ctypes.Structure):
    """Mirror of ChoreoDecodeStep (include/choreo_b200.h)."""

    _fields_ = [(n, _I) for n in ("n_layers", "d", "n_heads", "n_kv", "head_dim", "ffn_dim")] + \
        [(n, _P) for n in ("attn_norm", "w_qkv", "wo", "ffn_norm", "w_gu", "w_down")] + \
        [("eps", _F), ("k_pool", _P), ("v_pool", _P), ("n_pages", _I), ("page_size", _I),
         ("cos_t", _P), ("sin_t", _P), ("max_delta", _I), ("n_rows", _I), ("split", _I),
         ("n_items", _I)] + \
        [(n, _P) for n in ("pos", "page", "slot", "fat", "counts", "row_part_off", "row_part",
                           "x", "delta_in", "h", "qkv", "q", "part_o", "part_lse", "attn", "ao",
                           "gu", "act", "delta", "k7_ws", "k7_cnt", "attn_events")] + \
        [(n, _P) for n in ("row_t", "vis_page", "vis_len", "vis_own", "blk_rows", "items",
                           "linear_events")] + \
        [(n, _I) for n in ("layer_begin", "layer_end", "part")] + \
        [(n, _P) for n in ("h_b", "ssq_a", "ssq_b", "chain_ws", "chain_counters",
                           "chain_done", "chain_events", "q_k5", "item_order")] + \
        [("k3_tag", _I)]


class LayerChain(ctypes.Structure):
    """Mirror of ChoreoLayerChain (include/choreo_b200.h)."""

    _fields_ = [(n, _I) for n in ("n_rows", "split", "d", "n_heads", "n_kv", "head_dim",
                                  "ffn_dim")] + \
        [("eps", _F), ("phases", _I)] + \
        [(n, _P) for n in ("wo", "ffn_norm", "w_gu", "w_down", "attn_norm_next", "w_qkv")] + \
        [("layer_qkv", _I)] + \
        [(n, _P) for n in ("x", "attn", "h_a", "act", "h_b", "ssq_a", "ssq_b", "q", "k_pool",
                           "v_pool")] + \
        [("n_pages", _I), ("page_size", _I)] + \
        [(n, _P) for n in ("pos", "page", "slot", "cos_t", "sin_t")] + \
        [("max_delta", _I)] + \
        [(n, _P) for n in ("ws", "counters", "done")]


def ptr(t) -> int | None:
    """Raw device pointer of a torch tensor (None for None)."""
    return None if t is None else t.data_ptr()


def dtype_code(dtype) -> int:
    import torch

    if dtype == torch.float32:
        return F32
    if dtype == torch.bfloat16:
        return BF16
    raise NativeError(f"unsupported dtype {dtype}")
