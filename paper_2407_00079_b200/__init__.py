"""B200-native (sm_100a) KVCache hot path of Mooncake (arXiv 2407.00079).

Stage 1a block hashing, 1b prefix matching, 2 gather, 3 layer-wise transfer,
4 scatter -- hand-written CUDA in ``csrc/`` behind the C ABI ``include/kvx.h``
(``libkvx.so``), mirrored for Python in :mod:`.kvx`.  Importing this package
without the compiled library raises ImportError: there is no CPU fallback.
"""
from . import kvx  # noqa: F401
from .kvx import (  # noqa: F401
    BlockIndex,
    KVPool,
    KvxError,
    LayerIO,
    TransferEngine,
    ValidationError,
    XMatch,
    chain_hash,
    chain_hash_batch,
    copy_check,
    launch_count,
    match_prefix_batch,
    set_copy_impl,
)

__version__ = "0.1.0"
