"""Oracle pins for the propagation criterion (reading R23, oracle/propagation.py)."""
import math

import numpy as np
import pytest

from oracle import propagation as OPR


def test_mts_pure_mode_I():
    th, keq = OPR.mts(2.0e6, 0.0)
    assert th == 0.0 and keq == 2.0e6


def test_mts_pure_mode_II_textbook_angle():
    # Erdogan-Sih: pure mode II kinks at -arccos(1/3) = -70.53 deg with
    # K_eq = K_II * cos(th/2) * (-3/2 sin th) = (2/sqrt(3)) K_II
    th, keq = OPR.mts(0.0, 1.0e6)
    assert th == pytest.approx(-math.acos(1.0 / 3.0), rel=1e-13)
    assert keq == pytest.approx(2.0 / math.sqrt(3.0) * 1.0e6, rel=1e-13)


@pytest.mark.parametrize("KI,KII", [(1.0, 0.3), (1.0, -0.7), (0.2, 1.0), (3.0, 0.01)])
def test_mts_is_the_stationary_maximum_of_the_hoop_stress(KI, KII):
    th, keq = OPR.mts(KI, KII)
    # stationarity: K_I sin th + K_II (3 cos th - 1) = 0
    assert abs(KI * math.sin(th) + KII * (3 * math.cos(th) - 1)) <= 1e-12 * (KI + abs(KII))
    # maximum of sigma_thetatheta over (-pi, pi) at th, and K_eq = sqrt(2 pi r) sigma(th)
    grid = np.linspace(-math.pi + 1e-6, math.pi - 1e-6, 20001)
    s = np.array([OPR.sigma_thetatheta(KI, KII, t) for t in grid])
    assert OPR.sigma_thetatheta(KI, KII, th) >= s.max() * (1 - 1e-9)
    assert keq == pytest.approx(math.sqrt(2 * math.pi) * OPR.sigma_thetatheta(KI, KII, th), rel=1e-12)
    # mirror symmetry: K_II -> -K_II flips the kink angle, keeps K_eq
    th2, keq2 = OPR.mts(KI, -KII)
    assert th2 == pytest.approx(-th, abs=1e-15) and keq2 == pytest.approx(keq, rel=1e-14)


def test_grown_element_continues_a_mode_I_crack():
    # tip at the + end of an element at 30 deg: the new element lies on the
    # same line, beyond the tip, same length, outward end +
    b = math.radians(30)
    nx, ny, na, nb, ne = OPR.grow_tip(1.0, 2.0, 0.05, b, 1, 0.0)
    assert (nx, ny) == pytest.approx((1.0 + 0.1 * math.cos(b), 2.0 + 0.1 * math.sin(b)), abs=1e-15)
    assert na == 0.05 and nb == pytest.approx(b) and ne == 1
    # the - end: grows backwards along the line, outward end -
    nx, ny, na, nb, ne = OPR.grow_tip(1.0, 2.0, 0.05, b, 0, 0.0)
    assert (nx, ny) == pytest.approx((1.0 - 0.1 * math.cos(b), 2.0 - 0.1 * math.sin(b)), abs=1e-15)
    assert nb == pytest.approx(b) and ne == 0
