"""Pins for the bond-order-analysis oracle (oracle/boa.py): Tab. tab:Q4Q6 of the paper
(values for perfect lattices quoted from Stukowski 2012 / Mickel 2013,
three decimals), the spherical-harmonic addition theorem and inversion symmetry."""
import numpy as np
import pytest

import ljinputs as li

TAB = {  # Tab. tab:Q4Q6: (Q4, Q5, Q6)
    "fcc": (0.191, 0.0, 0.575),
    "hcp": (0.097, 0.252, 0.485),
    "bcc": (0.036, 0.0, 0.511),
}


def lattice(kind):
    if kind == "fcc":
        pos, box = li.fcc(3, 3, 3, rho=4.0 / np.sqrt(2.0) ** 3)   # nearest neighbour at 1
        return pos, box, 1.2                                        # 12 neighbours
    if kind == "hcp":
        pos, box = li.hcp(4, 3, 3)
        return pos, box, 1.2                                        # 12 neighbours
    pos, box = li.bcc(4, 4, 4)
    return pos, box, 1.4                                            # 8 + 6 = 14 neighbours


@pytest.mark.parametrize("kind", ["fcc", "hcp", "bcc"])
def test_table_q4q6(kind):
    from oracle.boa import boa
    pos, box, rc = lattice(kind)
    for ell, ref in zip((4, 5, 6), TAB[kind]):
        Q, nnb = boa(pos, box, ell, rc)
        assert np.all(nnb == (14 if kind == "bcc" else 12))
        np.testing.assert_allclose(Q, ref, atol=5.5e-4)   # table gives three decimals


def test_single_neighbour_is_one():
    """Addition theorem: sum_m |Y_l^m|^2 = (2l+1)/4pi, so one neighbour gives Q_l = 1."""
    from oracle.boa import boa
    pos = np.array([[1.0, 1.0, 1.0], [1.3, 1.7, 1.55]])
    for ell in (0, 1, 2, 4, 6, 8):
        Q, nnb = boa(pos, [10.0] * 3, ell, 1.5)
        assert nnb.tolist() == [1, 1]
        np.testing.assert_allclose(Q, 1.0, rtol=1e-13)


def test_rotation_invariance_and_isolated():
    from oracle.boa import boa
    rng = np.random.default_rng(2)
    pos = rng.uniform(2, 8, (40, 3))
    Q, _ = boa(pos, [10.0] * 3, 6, 1.6)
    c, s = np.cos(0.7), np.sin(0.7)
    R = np.array([[c, -s, 0], [s, c, 0], [0, 0, 1]])
    Q2, _ = boa((pos - 5) @ R.T + 5, [10.0] * 3, 6, 1.6)
    np.testing.assert_allclose(Q, Q2, rtol=1e-10, atol=1e-12)
    Q0, n0 = boa(np.array([[1.0, 1, 1], [5.0, 5, 5]]), [10.0] * 3, 6, 1.0)
    assert np.all(Q0 == 0.0) and np.all(n0 == 0)
