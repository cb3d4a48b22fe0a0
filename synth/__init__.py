"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This package holds *no* arithmetic of the method (no kernels, no loads, no
expansions): only geometry generators, material/load parameter records and
seeded random vectors, exactly as described in SURVEY.md §8(d).1 and
DESIGN.md §3 ("input recipe").  Both `oracle/` and the product package may
import it; it imports neither.
"""
from .geometry import (  # noqa: F401
    Geometry,
    straight_crack,
    parallel_fractures,
    random_fractures,
    segments_intersect,
)
from .configs import CONFIGS, make_config, random_dd  # noqa: F401
