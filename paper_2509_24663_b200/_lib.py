"""ctypes binding of the C ABI (include/swattn_b200.h).

The shared library ``libswattn_b200.so`` is built in-tree by
``__graft_entry__.build()`` (``make -C paper_2509_24663_b200/csrc``).  There is
no fallback: if the library is missing, every entry point raises.
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# SWATTN_B200_LIB: an alternative in-tree build of the same library (kernel A/B
# experiments under tools/); never a different implementation.
LIB_PATH = os.environ.get("SWATTN_B200_LIB") or os.path.join(_HERE, "libswattn_b200.so")

SWATTN_OK = 0
SWATTN_EINVAL = 1
SWATTN_EUNSUPPORTED = 2
SWATTN_ECUDA = 3
SWATTN_EEMPTY = 4

SELECT_MODE = {"exact": 0, "fused-exact": 1, "approx": 2}
SELECT_PREPARED = 0x100  # compressed keys already in the workspace (swattn_b200.h)
FORCED_MODE = {None: 0, "dense": 1, "sparse": 2}


class CConfig(ctypes.Structure):
    _fields_ = [(name, ctypes.c_int32) for name in (
        "h_q", "h_kv", "d_h", "B", "l_C1", "s_C1", "l_C2", "s_C2", "l", "s",
        "N_init", "N_local", "k_top", "w", "scale_compressed_logits", "experimental")]


class CPagedKV(ctypes.Structure):
    _fields_ = [
        ("k_pages", ctypes.c_void_p),
        ("v_pages", ctypes.c_void_p),
        ("block_table", ctypes.c_void_p),
        ("seq_lens", ctypes.c_void_p),
        ("max_pages", ctypes.c_int32),
        ("kc1", ctypes.c_void_p),
        ("kc2", ctypes.c_void_p),
        ("max_m1", ctypes.c_int32),
        ("max_m2", ctypes.c_int32),
        ("num_pages", ctypes.c_int32),
    ]


_lib = None


class LibraryMissing(RuntimeError):
    pass


def lib():
    """Load (once) and return the ctypes library handle."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise LibraryMissing(
            f"{LIB_PATH} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    P = ctypes.c_void_p
    I32, I64, SZ = ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t
    cfgp = ctypes.POINTER(CConfig)
    sig = {
        "swattn_last_error": (ctypes.c_char_p, []),
        "swattn_version": (I32, []),
        "swattn_validate_config": (I32, [cfgp]),
        "swattn_profile_supported": (I32, [cfgp]),
        "swattn_num_pooled": (I64, [I64, I32, I32]),
        "swattn_workspace_bytes": (SZ, [cfgp, I64]),
        "swattn_compress_keys": (I32, [cfgp, P, I64, P, P, P]),
        "swattn_block_scores": (I32, [cfgp, P, P, P, I64, I32, P, I64, P, P]),
        "swattn_shared_scores": (I32, [cfgp, P, P, P, I64, I32, P, P, P]),
        "swattn_topk_blocks": (I32, [cfgp, P, I64, I64, P, P, P]),
        "swattn_select_blocks": (I32, [cfgp, P, P, I64, I32, P, P, P, P, SZ, P]),
        "swattn_sparse_fwd": (I32, [cfgp, P, P, P, I64, P, P, P, P, P, SZ, P]),
        "swattn_sparse_workspace_bytes": (SZ, [cfgp, I64]),
        "swattn_sparse_fwd_lists": (I32, [cfgp, P, P, P, I64, P, I64, P, P, P, P]),
        "swattn_sparse_bwd": (I32, [cfgp, P, P, P, I64, P, P, P, P, P, P, P, P, P, SZ, P]),
        "swattn_sparse_bwd_workspace_bytes": (SZ, [cfgp, I64]),
        "swattn_dense_bwd": (I32, [cfgp, P, P, P, I64, I32, P, P, P, P, P, P, P, SZ, P]),
        "swattn_dense_bwd_workspace_bytes": (SZ, [cfgp, I64, I32]),
        "swattn_dense_fwd": (I32, [cfgp, P, P, P, I64, I32, P, P, P]),
        "swattn_attend": (I32, [cfgp, P, P, P, I64, I64, I32, I32, P, P,
                                ctypes.POINTER(I32), P, SZ, P]),
        "swattn_select_blocks_rows": (I32, [cfgp, P, P, I64, I64, I64, I32, P, P, P, P, SZ, P]),
        "swattn_sparse_fwd_rows": (I32, [cfgp, P, P, P, I64, I64, I64, P, P, P, P, P, SZ, P]),
        "swattn_attend_rows": (I32, [cfgp, P, P, P, I64, I64, I64, I32, P, P, P, SZ, P]),
        "swattn_attend_prepare": (I32, [cfgp, P, I64, P, SZ, P]),
        "swattn_attend_groups": (I32, [cfgp, P, P, P, I64, I32, I32, I64, I32, I32, P, P,
                                       ctypes.POINTER(I32), P, SZ, P]),
        "swattn_attend_rows_groups": (I32, [cfgp, P, P, P, I64, I64, I64, I32, I32, I32, P, P, P,
                                            SZ, P]),
        "swattn_workspace_ckeys": (I32, [cfgp, I64, P, ctypes.POINTER(P), ctypes.POINTER(P)]),
        "swattn_kcache_append": (I32, [cfgp, ctypes.POINTER(CPagedKV), P, I32, P]),
        "swattn_kcache_append_tokens": (I32, [cfgp, ctypes.POINTER(CPagedKV), P, P, P, I32, P]),
        "swattn_decode_step": (I32, [cfgp, ctypes.POINTER(CPagedKV), P, I32, P, P, P, P, SZ, P]),
        "swattn_decode_workspace_bytes": (SZ, [cfgp, I32, I32]),
        "swattn_decode_reranked_offset": (I64, [cfgp, I32, I32]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


EXPORTED = (
    "swattn_last_error", "swattn_version", "swattn_validate_config", "swattn_profile_supported",
    "swattn_num_pooled", "swattn_workspace_bytes", "swattn_compress_keys", "swattn_block_scores",
    "swattn_shared_scores", "swattn_topk_blocks", "swattn_select_blocks", "swattn_sparse_fwd",
    "swattn_sparse_workspace_bytes", "swattn_sparse_fwd_lists", "swattn_sparse_bwd", "swattn_sparse_bwd_workspace_bytes",
    "swattn_dense_bwd", "swattn_dense_bwd_workspace_bytes",
    "swattn_dense_fwd", "swattn_attend", "swattn_select_blocks_rows", "swattn_sparse_fwd_rows",
    "swattn_attend_rows", "swattn_attend_prepare", "swattn_attend_groups", "swattn_attend_rows_groups", "swattn_workspace_ckeys", "swattn_kcache_append", "swattn_kcache_append_tokens", "swattn_decode_step",
    "swattn_decode_workspace_bytes", "swattn_decode_reranked_offset",
)


def last_error() -> str:
    msg = lib().swattn_last_error()
    return msg.decode() if msg else ""


def check(rc: int, what: str) -> None:
    """Map a C status to the reference's exception classes (core.py:36-45,
    sparse.py:75-76)."""
    if rc == SWATTN_OK:
        return
    from .core import ConfigError, SwattnError
    msg = last_error() or what
    if rc == SWATTN_EINVAL:
        if msg.split(":", 1)[0] in ("positivity", "head-divisibility", "group-size",
                                    "pooling-profile", "window-coverage"):
            raise ConfigError(msg)
        raise ValueError(msg)
    if rc == SWATTN_EEMPTY:
        raise RuntimeError(msg)
    if rc == SWATTN_EUNSUPPORTED:
        raise NotImplementedError(msg)
    raise SwattnError(f"{what}: {msg}")


_CFG_CACHE: dict = {}


def c_config(cfg) -> CConfig:
    """The C struct of an AttentionConfig (cached per config: the C side
    only reads it)."""
    try:
        hit = _CFG_CACHE.get(cfg)
    except TypeError:  # unhashable (a mutable stand-in): build it every time
        return _build_c_config(cfg)
    if hit is None:
        hit = _CFG_CACHE[cfg] = _build_c_config(cfg)
    return hit


def _build_c_config(cfg) -> CConfig:
    c = CConfig()
    for name, _ in CConfig._fields_:
        if name == "scale_compressed_logits":
            c.scale_compressed_logits = int(bool(cfg.scale_compressed_logits))
        elif name == "experimental":
            c.experimental = int(bool(cfg.experimental))
        else:
            setattr(c, name, int(getattr(cfg, name)))
    return c


def ptr(t) -> int | None:
    """Device pointer of a torch tensor (None passes NULL)."""
    return None if t is None else t.data_ptr()


def stream_handle(device=None) -> int:
    import torch
    return torch.cuda.current_stream(device).cuda_stream
