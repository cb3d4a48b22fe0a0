"""GPU propagation loop (Fig. 8 branch; reading R23)
vs the oracle's dense loop: same grow decisions, SIFs and new elements."""
import math

import numpy as np
import pytest

from oracle import propagation as OPR

from ._util import rel_l2

pytestmark = pytest.mark.gpu

G0, NU0 = 8e9, 0.25


@pytest.fixture(scope="module")
def ddm():
    import torch
    import paper_1812_05087_b200 as D
    ctx = D.Context(0)
    return D, ctx, torch


def _cracks():
    """Two inclined cracks (20 + 12 elements), tips = first/last elements."""
    xs, ys, hs, bs, tips = [], [], [], [], []
    for (cx, cy, L, ang, ne) in ((0.0, 0.0, 1.0, 30.0, 20), (3.0, 1.5, 0.6, 110.0, 12)):
        b = math.radians(ang)
        k = (np.arange(ne) + 0.5) / ne * 2 - 1
        n0 = len(xs)
        xs += list(cx + L * k * math.cos(b))
        ys += list(cy + L * k * math.sin(b))
        hs += [L / ne] * ne
        bs += [b] * ne
        tips += [(n0, 0), (n0 + ne - 1, 1)]
    return np.array(xs), np.array(ys), np.array(hs), np.array(bs), tips


@pytest.mark.parametrize("K_IC", [1.0e6, 2.2e7, 1.0e9])
def test_propagation_matches_oracle(ddm, K_IC):
    D, ctx, torch = ddm
    xc, yc, a, beta, tips = _cracks()
    load = {"p_f": 40e6, "sH": 30e6, "sh": 25e6}
    steps = 3
    ox, oy, oa, ob, otips, oh = OPR.propagate(xc, yc, a, beta, tips, G0, NU0, load, K_IC, steps)
    f = lambda v: torch.tensor(v, dtype=torch.float64, device="cuda")
    mat = D.material(0, G0, NU0)
    gx, gy, ga, gb, gt, gh = D.propagate(ctx, f(xc), f(yc), f(a), f(beta),
                                         torch.tensor(tips), mat, load, K_IC, steps,
                                         leaf_size=8, order_p=32)
    assert len(gh) == len(oh)
    for s_g, s_o in zip(gh, oh):
        assert s_g["n"] == s_o["n"]
        assert s_g["grow"] == s_o["grow"]
        assert rel_l2(np.array(s_g["KI"]), np.array(s_o["KI"])) <= 1e-6
        assert rel_l2(np.array(s_g["KII"]), np.array(s_o["KII"])) <= 1e-6
    assert gx.numel() == ox.size
    for gv, ov in ((gx, ox), (gy, oy), (ga, oa), (gb, ob)):
        assert np.allclose(gv.cpu().numpy(), ov, rtol=1e-6, atol=1e-9)
    assert [tuple(t) for t in gt.cpu().tolist()] == [tuple(t) for t in otips]
    if K_IC == 1.0e6:   # every tip grows every step
        assert all(all(s["grow"]) for s in oh) and ox.size == xc.size + 4 * steps


def test_tip_growth_arguments(ddm):
    D, ctx, torch = ddm
    z = torch.zeros(1, dtype=torch.float64, device="cuda")
    e = torch.ones(1, dtype=torch.int32, device="cuda")
    with pytest.raises(D.DDMError):
        D.tip_growth(ctx, z, z, z, z, z, z, e, -1.0)
    # K_I <= 0 never grows
    grow, *_ = D.tip_growth(ctx, z - 1.0, z, z, z, z + 0.1, z, e, 0.0)
    assert int(grow.item()) == 0
