"""B200-native (sm_100a) MEFT sparse Key-Experts adapter layer.

The product is ``libmeft_cuda.so`` (hand-written CUDA for sm_100a behind the C ABI in include/meft_cuda.h) and
the drop-in C++ shim ``libmeft_dropin.so`` (the reference's proj/include/meft API over that ABI). This Python
package is a thin ctypes mirror used by the tests and bench.py.
"""
from ._lib import LIB_PATH, MeftError, exported_symbols, lib  # noqa: F401

__all__ = ["LIB_PATH", "MeftError", "exported_symbols", "lib"]
