"""Pins of the far-field log1p polynomials compiled into the grid kernel (green.cuh FarPoly, R25).

log x = L + log1p(r), r = x c - 1, with |r| <= 1 / (2^(FB+1) + 1) for the bin-midpoint c of an FB-bit table; the
kernel evaluates log1p(r) = r (1 + r (a2 + r a3 [+ r^2 a4])).  The constants are read from the CUDA header (so the
test pins what is compiled) and checked against log1p in 40-digit arithmetic over the whole reduced range: the
absolute error must stay within the bound DESIGN.md states for each variant, far below the 1e-9 hierarchical
precision.  A dropped term or a sign slip in a coefficient fails by orders of magnitude.
"""
import os
import re

import mpmath as mp
import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "paper_1906_04209_b200", "csrc", "green.cuh")


def _consts():
    src = open(HDR).read()
    out = {}
    for m in re.finditer(r"struct FarPoly<(\d+), (\d+)> \{\s*static constexpr double ([^;]+);", src):
        vals = dict((k.strip(), float(v)) for k, v in (kv.split("=") for kv in m.group(3).split(",")))
        out[(int(m.group(1)), int(m.group(2)))] = vals
    return out


@pytest.mark.parametrize("fb,deg,bound", [(7, 3, 1.2e-11), (7, 4, 1e-13)])
def test_far_log1p_polynomial(fb, deg, bound):
    c = _consts()[(fb, deg)]
    mp.mp.dps = 40
    h = 0.5 / (2 ** fb + 0.5) * (1 + 2.0 ** -20)   # bin half-width, plus the rcp.approx seed error of c
    err = 0.0
    for r in np.concatenate([np.linspace(-h, h, 2001), [-h, h, 0.0]]):
        poly = r * (1 + r * (c["a2"] + r * (c["a3"] + r * c["a4"])))
        err = max(err, abs(float(mp.log1p(mp.mpf(float(r)))) - poly))
    assert err <= bound, (fb, deg, err)
    # against the Taylor coefficients: the minimax set differs only in the last digits that buy the error bound
    assert abs(c["a2"] + 0.5) < 1e-5 and abs(c["a3"] - 1.0 / 3.0) < 1e-4


def test_far_log1p_quadratic_fb9():
    """The R32 default far form: log1p(r) = r (c1 + c2 r) on the FB = 9 bins, |r| <= 2^-10 (1 + 2^-20): minimax
    absolute error 7.7e-11 (the bound DESIGN.md R32 states), two orders below the 1e-9 precision it serves; the
    handle switches to the FB = 7 cubic below precision 1e-10 (kGridQuadMinPrecision)."""
    src = open(HDR).read()
    m = re.search(r"struct FarQuad<9> \{\s*static constexpr double c1 = ([-0-9.eE]+), c2 = ([-0-9.eE]+);", src)
    c1, c2 = float(m.group(1)), float(m.group(2))
    mp.mp.dps = 40
    h = 0.5 / (2 ** 9 + 0.5) * (1 + 2.0 ** -20)
    err = 0.0
    for r in np.concatenate([np.linspace(-h, h, 4001), [-h, h, 0.0]]):
        err = max(err, abs(float(mp.log1p(mp.mpf(float(r)))) - r * (c1 + c2 * r)))
    assert err <= 8e-11, err
    assert abs(c1 - 1.0) < 1e-6 and abs(c2 + 0.5) < 1e-6
