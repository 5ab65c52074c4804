"""B200-native (sm_100a) scrambled distributed attention -- the FedRAG hot path.

The product is libsdattn_b200.so behind the C ABI in include/sdattn_b200.h; this package holds
its sources (csrc/), the ctypes binding (capi) and torch-facing plumbing (ops, protocol,
distributed). Importing it fails loudly if the library has not been built.
"""
from . import capi  # noqa: F401  (raises ImportError when libsdattn_b200.so is missing)

__all__ = ["capi"]
