"""B200-native Paillier plugin for secure vertical federated GBDT (arXiv 2504.03909).

The product is the C ABI library ``lib/libsfxb_cuda.so`` (include/sfxb_cuda.h)
and the C++ EncryptionPlugin adapter (``host/``); ``_lib`` is the ctypes
binding used by the tests and bench.py.
"""
from . import _lib  # noqa: F401
from ._lib import AuthorizationError, Context, SfxbError  # noqa: F401

__all__ = ["Context", "SfxbError", "AuthorizationError"]
