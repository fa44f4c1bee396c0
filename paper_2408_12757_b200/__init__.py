"""B200-native (sm_100a) implementation of NanoFlow's hot path (arXiv 2408.12757).

The product is libnf.so (C ABI in include/nf.h); ``nf`` is its ctypes
binding and ``runtime`` the PyTorch device-memory plumbing around it.
"""
import os

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG_DIR, "libnf.so")


def load():
    """Import the binding (raises if libnf.so is missing: no CPU fallback)."""
    from . import nf  # noqa: F401
    return nf
