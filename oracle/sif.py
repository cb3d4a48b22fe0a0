"""ORACLE (test infrastructure only) — stress intensity factors.

Olson's empirical relation, Eq.(SIF):
    K_I  = 0.806 E / (4 (1 - nu^2)) sqrt(pi / (2 a)) D_n
    K_II = 0.806 E / (4 (1 - nu^2)) sqrt(pi / (2 a)) D_s
with (reading R9) a = the tip element's half-length, E = 2 G (1 + nu) with
drained nu, D_n = opening (opening-positive), two tips per fracture.
Pins: S:469 value 1.010e6 Pa sqrt(m); Sneddon K_I / (p sqrt(pi a)) = 1.0095
at N = 200 (tests/test_oracle_elastic.py).
"""
from __future__ import annotations

import numpy as np


def sif(w_tip, ds_tip, a_tip, E, nu):
    f = 0.806 * E / (4.0 * (1.0 - nu * nu)) * np.sqrt(np.pi / (2.0 * np.asarray(a_tip)))
    return f * np.asarray(w_tip), f * np.asarray(ds_tip)
