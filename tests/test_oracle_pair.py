"""Pins for the oracle's pair arithmetic (O1 wrap, O2 displacement, O5 LJ force/energy).

Each expected value below is fixed by the paper or by mathematics, not by the oracle:
closed-form LJ values at dyadic distances (Eq. eqn:LJpotential P:678-685, Eq. eqn:LJforce
P:969-978), the physical sign (repulsive core), F = -dV/dr by central differences,
SPEC's wrap examples and the golden 'tie and seam' fixture.
"""
import json
import os
from fractions import Fraction

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def two_body(orc, r, shift=0.0, rc=2.5, axis=0, box=20.0):
    pos = np.zeros((2, 3)) + 1.0
    pos[1, axis] += r
    f = orc.forces(pos, [box] * 3, orc.LJ(rc=rc, shift=shift))
    return pos, f


def exact_lj(r: Fraction, shift: Fraction):
    """V(r) and g(r) = 48 (r^-14 - r^-8 / 2) at sigma = eps = 1, exactly (closed form)."""
    inv = 1 / r
    v = 4 * (inv ** 12 - inv ** 6 + shift)
    g = 48 * (inv ** 14 - Fraction(1, 2) * inv ** 8)
    return v, g


@pytest.mark.parametrize("r,V0,g", [
    (1.0, 0.0, 24.0),                                   # r = sigma: V = 0, g = 24 (repulsive)
    (2.0, -63.0 / 1024.0, -93.0 / 1024.0),               # attractive tail, exact in binary
    (1.5, -170240.0 / 531441.0, -1230848.0 / 1594323.0),
])
def test_closed_form_pair(orc, r, V0, g):
    _, f = two_body(orc, r, shift=0.0)
    # PE = V(r) (two ordered pairs, each counting V/2 -- reading R2)
    assert f.pe == pytest.approx(V0, rel=1e-15, abs=1e-16)
    # F_0 = g * (r_0 - r_1) = -g r x_hat ; F_1 = -F_0
    assert f.F[0, 0] == pytest.approx(-g * r, rel=1e-15)
    assert f.F[1, 0] == pytest.approx(g * r, rel=1e-15)
    assert np.all(f.F[:, 1:] == 0.0)
    # the paper's +1/4 shift adds exactly 4 eps * 1/4 = 1 per interacting pair
    _, fq = two_body(orc, r, shift=0.25)
    assert fq.pe == pytest.approx(V0 + 1.0, rel=1e-15)


def test_repulsive_core_sign(orc):
    """Eq. eqn:LJforce: F_i = +48 eps/sigma^2 (r_i - r_j)[...] pushes i away from j at r < 2^(1/6)."""
    _, f = two_body(orc, 1.0)
    assert f.F[0, 0] < 0.0 and f.F[1, 0] > 0.0          # particle 0 sits at lower x
    _, f = two_body(orc, 2.0)
    assert f.F[0, 0] > 0.0 and f.F[1, 0] < 0.0          # attraction


def test_minimum_at_2_16(orc):
    r = 2.0 ** (1.0 / 6.0)
    _, f = two_body(orc, r, shift=0.0)
    assert abs(f.F[0, 0]) < 1e-13
    assert f.pe == pytest.approx(-1.0, rel=1e-14)        # V_min = -eps
    _, fq = two_body(orc, r, shift=0.25)
    assert abs(fq.pe) < 1e-14                             # WCA-shifted: V(2^(1/6)) = 0


def test_strict_cutoff(orc):
    """r = rc exactly contributes nothing (strict <, reading R4); beyond rc exactly 0."""
    for r in (2.5, 2.75, 3.0):
        _, f = two_body(orc, r, shift=0.25)
        assert f.pe == 0.0 and np.all(f.F == 0.0)
    _, f = two_body(orc, 2.5 - 2.0 ** -40, shift=0.0)
    assert f.pe != 0.0


@pytest.mark.parametrize("r", [0.95, 1.1, 1.3, 1.7, 2.2])
def test_central_difference(orc, r):
    """F = -dV/dr (Eq. eqn:LJforce first line) by a 4th-order central difference of V."""
    h = 1e-4
    vals = []
    for k in (-2, -1, 1, 2):
        _, f = two_body(orc, r + k * h, shift=0.0)
        vals.append(f.pe)
    dVdr = (vals[0] - 8 * vals[1] + 8 * vals[2] - vals[3]) / (12 * h)
    _, f = two_body(orc, r, shift=0.0)
    # force on particle 1 (at larger x) along +x equals -dV/dr
    assert f.F[1, 0] == pytest.approx(-dVdr, rel=1e-8)


def test_general_sigma_eps(orc):
    """Scaling: V(r; sigma, eps) = eps V(r/sigma; 1, 1); F scales as eps/sigma."""
    sig, eps, r = 1.3, 0.7, 1.6
    pos = np.array([[1.0, 1.0, 1.0], [1.0 + r, 1.0, 1.0]])
    f = orc.forces(pos, [30.0] * 3, orc.LJ(rc=2.5 * sig, eps=eps, sigma=sig, shift=0.0))
    f1 = orc.forces(pos / sig, [30.0 / sig] * 3, orc.LJ(rc=2.5, shift=0.0))
    assert f.pe == pytest.approx(eps * f1.pe, rel=1e-13)
    assert f.F[0, 0] == pytest.approx(eps / sig * f1.F[0, 0], rel=1e-13)


def test_wrap_examples(orc):
    """SPEC.md:96-99 wrap examples, half-open [0, L)."""
    box = [10.0, 10.0, 10.0]
    p = orc.wrap(np.array([[-0.25, 10.0, 23.5]]), box)
    assert p.tolist() == [[9.75, 0.0, 3.5]]
    # tiny negative rounds to L under x + L -> folded to 0 (half-open)
    p = orc.wrap(np.array([[-1e-18, 5.0, 5.0]]), box)
    assert p[0, 0] == 0.0
    # idempotent
    q = orc.wrap(np.random.default_rng(0).uniform(-30, 30, (100, 3)), box)
    assert np.array_equal(orc.wrap(q, box), q)
    assert np.all((q >= 0) & (q < 10.0))
    with pytest.raises(ValueError, match="particle 1"):
        orc.wrap(np.array([[1.0, 1.0, 1.0], [np.nan, 0.0, 0.0]]), box)


def test_displacement_minimum_image(orc):
    box = [9.0, 9.0, 9.0]
    d = orc.displacement([0.5, 0.5, 0.5], [8.0, 0.5, 4.0], box)
    assert d.tolist() == [1.5, 0.0, -3.5]
    d = orc.displacement([8.0, 0.5, 0.5], [0.5, 0.5, 0.5], box)
    assert d.tolist() == [-1.5, 0.0, 0.0]
    assert orc.r2([3.0, 4.0, 12.0]) == 169.0


def test_tie_and_seam_fixture(orc):
    g = json.load(open(os.path.join(GOLD, "tie_and_seam.json")))
    pos, box = np.array(g["pos"]), np.array(g["box"])
    rn = g["rc"] + g["delta"]
    for method in ("brute", "cells"):
        off, nbr = orc.neighbours(pos, box, rn, method)
        got = [nbr[off[i]:off[i + 1]].tolist() for i in range(len(pos))]
        assert got == g["nb_rbar"], method
    f = orc.forces(pos, box, orc.LJ(rc=g["rc"], shift=0.0))
    np.testing.assert_allclose(f.F, np.array(g["F"]), rtol=1e-15, atol=1e-15)
    np.testing.assert_allclose(f.e, np.array(g["e_shift0"]), rtol=1e-15, atol=0)
    assert f.pe == pytest.approx(g["pe_shift0"], rel=1e-15)
    assert np.all(f.F.sum(axis=0) == 0.0)
    fq = orc.forces(pos, box, orc.LJ(rc=g["rc"], shift=0.25))
    assert fq.pe == pytest.approx(g["pe_shift_quarter"], rel=1e-15)
    # independent closed-form re-derivation of the golden numbers (exact rationals)
    v15, g15 = exact_lj(Fraction(3, 2), Fraction(0))
    v2, g2 = exact_lj(Fraction(2), Fraction(0))
    assert float(g15 * Fraction(3, 2)) == pytest.approx(g["F"][0][0], rel=1e-15)  # F0 = g * (+1.5)
    assert float(-2 * g2) == pytest.approx(g["F"][0][2], rel=1e-15)
    assert float((v15 + v2) / 2) == pytest.approx(g["e_shift0"][0], rel=1e-15)
    # list-driven forces equal brute-force forces bitwise
    off, nbr = orc.neighbours(pos, box, rn, "brute")
    fl = orc.forces(pos, box, orc.LJ(rc=g["rc"], shift=0.0), nlist=(off, nbr))
    assert np.array_equal(fl.F, f.F) and np.array_equal(fl.e, f.e)
