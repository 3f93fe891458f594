"""B200-native thresholded-Ax (arXiv 2105.05879): Kerdock-sketch preprocessing,
streaming median-of-means estimator and exact support refinement on sm_100a.

The product is the C-ABI library ``libfst_b200.so`` (include/fst_b200.h); this
package holds its sources (``csrc/``), the Python mirror of the reference API
(``fst``) and host-side synthetic input generators (``generators``).
"""
from . import fst  # noqa: F401

__all__ = ["fst"]
