"""B200-native ACE Prove phase (arxiv 2603.10242).

The hot path lives in ``lib/libacegpu.so`` (sm_100a CUDA behind the C ABI in
``include/acegpu.h``). This package is the host-side mirror of the reference
prover API (``proj/include/ace/prover.hpp``): ``prover``, ``crypto``, ``wire``,
plus ``shard`` for multi-GPU chunk sharding. There is no CPU fallback.
"""
from . import _native  # noqa: F401  (fails loudly if libacegpu.so is missing)

__all__ = ["prover", "crypto", "wire", "shard"]
