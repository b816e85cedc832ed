"""B200-native (sm_100a) InfLLM-V2 dense-sparse switchable attention.

Drop-in for the hot path of the reference package ``swattn`` 0.1.0: the
module layout and entry points mirror it (``switch.attend``,
``selection.select_blocks``, ``sparse.sparse_forward``,
``dense.tiled_gqa_forward``, ``compression.mean_pool_keys``).  Every stage
runs as a hand-written CUDA kernel in ``libswattn_b200.so`` behind the C ABI
of ``include/swattn_b200.h``; there is no CPU fallback.
"""

from .core import (AttentionConfig, ConfigError, OpCounter, SwattnError, TensorFormatError,
                   make_qkv, validate_config)

__all__ = ["AttentionConfig", "ConfigError", "OpCounter", "SwattnError", "TensorFormatError",
           "make_qkv", "validate_config"]
__version__ = "0.1.0"
