"""B200-native (sm_100a) sample-based divide step (arXiv 1902.07554):
nearest-sample point assignment and border-simplex detection.

The product path is libsbdt_gpu.so (include/sbdt_gpu.h); `gpu` mirrors the
reference's SPEC interface over it, `host` produces the seeded inputs.
"""
from . import gpu, host  # noqa: F401
from .gpu import (BorderSet, Context, DegenerateSimplex, IntersectionPolicy, Partitioning,  # noqa: F401
                  assign_points, find_border)

__all__ = ["gpu", "host", "assign_points", "find_border", "IntersectionPolicy", "Partitioning", "BorderSet",
           "Context", "DegenerateSimplex"]
