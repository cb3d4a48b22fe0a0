"""The five BASELINE.json configurations as plain parameter records.

Indices follow BASELINE.json list order, 1-based (cfg1 = configs[0]).  The
configs cross-reference each other 0-indexed;
the readings applied here are listed in DESIGN.md §2.

"p" is the stated expansion order (BASELINE.json: order 20); "p_star" the
smallest order meeting every tolerance on solution-like vectors (reading R7).

Only numbers and seeded geometry live here; every formula of the method
(loads resolved on faces, kernels, ...) is implemented separately by the
oracle and by the CUDA path.
"""
from __future__ import annotations

import numpy as np

from .geometry import Geometry, parallel_fractures, random_fractures, straight_crack

MPa = 1.0e6

# material: kind 0 = elastic, 1 = poroelastic.  G (Pa), nu, nu_u, alpha, kappa = k/mu
_ELASTIC_E20 = {"kind": 0, "G": 20e9 / (2 * 1.25), "nu": 0.25, "nu_u": 0.25, "alpha": 0.0,
                "kappa": 0.0}
_PORO_CFG3 = {"kind": 1, "G": 6e9, "nu": 0.2, "nu_u": 0.33, "alpha": 0.8,
              "kappa": 1e-18 / 1e-3}

CONFIGS = {
    1: {"name": "cfg1_sneddon", "material": _ELASTIC_E20, "leaf": 32, "p": 20, "p_star": 28,
        # uniform internal pressure, no far field (BASELINE configs[0])
        "load": {"p_f": 1.0 * MPa, "sH": 0.0, "sh": 0.0, "p0": 0.0, "mode": "absolute"},
        "tol": 1e-10},
    2: {"name": "cfg2_random_elastic", "material": _ELASTIC_E20, "leaf": 32, "p": 20, "p_star": 28,
        "load": {"p_f": 10.0 * MPa, "sH": 30.0 * MPa, "sh": 25.0 * MPa, "p0": 0.0,
                 "mode": "absolute"},
        "tol": 1e-10},
    3: {"name": "cfg3_well_poro", "material": _PORO_CFG3, "leaf": 32, "p": 20, "p_star": 30,
        # uniform NET pressure 5 MPa on the faces; pressure row (sh + 5) - p0 (P15)
        "load": {"p_f": 5.0 * MPa, "sH": 30.0 * MPa, "sh": 25.0 * MPa, "p0": 20.0 * MPa,
                 "mode": "net"},
        "dt": 100.0, "steps": 1, "tol": 1e-10},
    4: {"name": "cfg4_random_poro_march", "material": _PORO_CFG3, "leaf": 32, "p": 20, "p_star": 28,
        # injection pressure read as p_f - p0 = 10 MPa (P14)
        "load": {"p_f": 30.0 * MPa, "sH": 30.0 * MPa, "sh": 25.0 * MPa, "p0": 20.0 * MPa,
                 "mode": "absolute"},
        "dt": 60.0, "steps": 200, "tol": 1e-10},
    5: {"name": "cfg5_scaling_elastic", "material": _ELASTIC_E20, "leaf": 64, "p": 20, "p_star": 20,
        "load": None, "d_seed": 55, "reps": 100},
}


def make_config(cfg: int) -> Geometry:
    """Seeded geometry of config `cfg` (1..5), user element order."""
    if cfg == 1:
        return straight_crack(1.0, 200)
    if cfg == 2:
        return random_fractures(100, 20, 100.0, 2.0, 6.0, seed=2)
    if cfg == 3:
        return parallel_fractures(5, 100.0, 20.0, 4000)
    if cfg == 4:
        return random_fractures(40, 50, 100.0, 5.0, 15.0, seed=4)
    if cfg == 5:
        return random_fractures(10_000, 100, 2000.0, 2.0, 6.0, seed=5)
    raise ValueError(f"unknown config {cfg}")


def random_dd(n: int, ncomp: int, seed: int, lo: float = -1e-3, hi: float = 1e-3) -> np.ndarray:
    """Seeded DD vector, element-major interleaved [n, ncomp] (SURVEY.md §8c.1 DOF layout)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    return rng.uniform(lo, hi, size=(n, ncomp))
