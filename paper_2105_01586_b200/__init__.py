"""B200-native FEM harmonic inpainting with data optimisation (Chizhov & Weickert,
arXiv 2105.01586): the data-parallel hot path behind the C ABI of include/femi.h.

    femi      -- ctypes binding of libfemi.so (marshalling only)
    pipeline  -- host-side drivers built from the ABI calls (inpaint, densify, tonal)
    multi     -- multi-GPU plumbing (replicas, batch sharding, max-over-ranks timing)
"""
from . import femi  # noqa: F401
from .femi import FemiError, Mesh, System  # noqa: F401
