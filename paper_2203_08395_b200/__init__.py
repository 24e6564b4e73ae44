"""B200-native dependency-ordered DAG propagation (arXiv 2203.08395 hot path).

The product is libhf.so (C ABI in include/hf.h, CUDA sources in csrc/); this
package holds its build script and the thin ctypes binding ``hf``.  Importing
``paper_2203_08395_b200.hf`` loads libhf.so and raises if it is missing -- there
is no CPU fallback.
"""
__all__ = ["hf", "build"]
