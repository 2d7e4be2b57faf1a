"""paper_2602_01053_b200 -- B200-native Flash-LoRA-Attention over a shared, paged KV + low-rank cache.

The product is ``lib/liblorakv_b200.so`` (hand-written CUDA for sm_100a behind the C ABI declared in
``include/lorakv_b200.h``) plus the source-compatible C++ headers in ``include/lorakv/``.  This Python
package is only the thin ctypes binding that the tests and ``bench.py`` drive the C ABI through; it
contains no compute and no fallback: every call fails loudly when the CUDA library or a B200 is missing.
"""
from .abi import (Adapters, Context, Gather, LorakvError, Pool, Projection, build, lib_path, load_library,  # noqa: F401
                  BF16, F32, HOST, DEVICE, SCHEMES)

__all__ = ["Adapters", "Context", "LorakvError", "Pool", "Projection", "build", "lib_path", "load_library",
           "BF16", "F32", "HOST", "DEVICE", "SCHEMES"]
