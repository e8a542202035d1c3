"""B200-native multi-tenant stage-schedule executor (arXiv 2111.14255 hot path).

The product is libmt.so (include/mt.h); `mt` is its thin ctypes binding and `session` holds
the torch plumbing (device memory for weights, workspace, inputs, outputs).
"""
from . import mt  # noqa: F401  (raises ImportError if libmt.so is missing: no CPU fallback)
