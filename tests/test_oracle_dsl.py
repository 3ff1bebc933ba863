"""Pins for the DSL oracle (oracle/dsl.py): the sequential Particle / Pair Loop wrapper of
Listing lst:simplest_pairloop running the paper's own kernels."""
import numpy as np
import pytest

import ljinputs as li
from dsl_kernels import CNA_I, CNA_II, KINETIC, LJ, LJ_CONSTANTS, SIMPLE, VEL_UPDATE


def c1(cells=6, sigma_d=0.05):
    pos, box = li.fcc(cells, cells, cells)
    return li.perturb(pos, sigma_d), box


def test_lj_listing_equals_force_oracle():
    """Listing 9 through the pair loop equals O5 (Eq. eqn:LJforce, R1/R2): F within 1e-13 S_i,
    u = sum over ordered pairs = 2 PE."""
    import oracle
    from oracle import dsl
    pos, box = c1()
    n = len(pos)
    d, s = dsl.pair_loop(LJ, pos, box, li.RC, dats={"F": (np.zeros((n, 3)), dsl.INC_ZERO)},
                         scalars={"u": (np.zeros(1), dsl.INC_ZERO)}, constants=LJ_CONSTANTS)
    ref = oracle.forces(pos, box, oracle.LJ(rc=li.RC))
    assert np.all(np.abs(d["F"] - ref.F) <= 1e-13 * ref.S[:, None])
    assert abs(0.5 * s["u"][0] - ref.pe) <= 1e-12 * np.sum(ref.A)


def test_simple_op_example_against_numpy():
    """Eqs. eqn:simple_op / eqn:simple_op_global over the pairs within the shell cutoff."""
    from oracle import dsl
    pos, box = c1(cells=4)
    n = len(pos)
    a = np.random.default_rng(3).standard_normal((n, 3))
    rcut = 1.6
    d, s = dsl.pair_loop(SIMPLE, pos, box, rcut, dats={"a": (a, dsl.READ), "b": (np.zeros((n, 1)), dsl.INC)},
                         scalars={"S": (np.zeros(1), dsl.INC)}, constants={"dimension": 3})
    dd = pos[:, None, :] - pos[None, :, :]
    dd -= box * np.round(dd / box)
    r2 = (dd ** 2).sum(-1)
    mask = (r2 < rcut * rcut) & ~np.eye(n, dtype=bool)
    q = ((a[:, None, :] - a[None, :, :]) ** 2).sum(-1)
    np.testing.assert_allclose(d["b"][:, 0], (q * mask).sum(1), rtol=1e-12)
    np.testing.assert_allclose(s["S"][0], (q * q * mask).sum(), rtol=1e-12)


def test_access_descriptors():
    """INC adds to the existing values, INC_ZERO starts from zero, READ leaves data alone."""
    from oracle import dsl
    pos, box = c1(cells=4, sigma_d=0.0)
    n = len(pos)
    ones = np.ones((n, 1))
    code = "c.i[0] += 1.0;"
    d_inc, _ = dsl.pair_loop(code, pos, box, 1.3, dats={"c": (ones, dsl.INC)})
    d_zero, _ = dsl.pair_loop(code, pos, box, 1.3, dats={"c": (ones, dsl.INC_ZERO)})
    assert np.array_equal(d_inc["c"], d_zero["c"] + 1.0)
    assert np.all(d_zero["c"] == 12.0)            # perfect-ish fcc: 12 nearest neighbours


def test_velocity_update_particle_loop():
    from oracle import dsl
    rng = np.random.default_rng(5)
    n = 100
    v, F = rng.standard_normal((n, 3)), rng.standard_normal((n, 3))
    d, _ = dsl.particle_loop(VEL_UPDATE, n, dats={"v": (v, dsl.RW), "F": (F, dsl.READ)},
                             constants={"dht_iMASS": 0.0025})
    assert np.array_equal(d["v"], v + F * 0.0025)


def test_kinetic_energy_particle_loop():
    from oracle import dsl
    import oracle
    v = li.velocities(500, 1.44)
    _, s = dsl.particle_loop(KINETIC, 500, dats={"v": (v, dsl.READ)}, scalars={"k": (np.zeros(1), dsl.INC_ZERO)},
                             constants={"mass": 1.0})
    assert abs(s["k"][0] - oracle.kinetic(v)) <= 1e-12 * s["k"][0]


def test_cna_listings_against_cna_oracle():
    """Listings lst:CNA-kernel_I/II produce E_d (direct bonds) and E_d + indirect bonds as in
    Algs. alg:cna_I/II; compared as multisets with the CNA oracle's construction."""
    from oracle import dsl
    from oracle.cna import cna  # noqa: F401  (the construction it follows is re-derived here)
    import oracle
    pos, box = li.hcp(4, 3, 3)
    pos = li.perturb(pos, 0.02)
    n = len(pos)
    rc = 1.2071
    nbmax = 24
    ids = np.arange(n, dtype=np.int64).reshape(-1, 1)
    base = {"id": (ids, dsl.READ)}
    d1, _ = dsl.pair_loop(CNA_I, pos, box, rc, dats={**base, "n_nb": (np.zeros((n, 1), np.int64), dsl.INC_ZERO),
                                                    "n_bond": (np.zeros((n, 1), np.int64), dsl.INC_ZERO),
                                                    "bond": (np.zeros((n, 2 * nbmax * nbmax), np.int64),
                                                             dsl.WRITE)},
                          constants={"rc_sq": rc * rc})
    off, nbr = oracle.neighbours(pos, box, rc, "brute")
    for i in range(n):
        assert d1["n_nb"][i, 0] == off[i + 1] - off[i]
        got = sorted(d1["bond"][i, 1:2 * d1["n_nb"][i, 0]:2].tolist())
        assert got == sorted(nbr[off[i]:off[i + 1]].tolist())
        assert np.all(d1["bond"][i, 0:2 * d1["n_nb"][i, 0]:2] == i)
    d2, _ = dsl.pair_loop(CNA_II, pos, box, rc, dats={**base, "n_nb": (d1["n_nb"], dsl.READ),
                                                    "n_bond": (d1["n_bond"], dsl.INC),
                                                    "bond": (d1["bond"], dsl.RW)},
                          constants={"rc_sq": rc * rc})
    for i in range(0, n, 5):
        nb_i = nbr[off[i]:off[i + 1]]
        expect = [(i, j) for j in nb_i]
        for j in nb_i:
            expect += [(j, k) for k in nbr[off[j]:off[j + 1]] if k != i]
        m = d2["n_bond"][i, 0]
        got = [tuple(d2["bond"][i, 2 * k:2 * k + 2]) for k in range(m)]
        assert sorted(got) == sorted(expect)


def test_pair_set_is_the_strict_cutoff():
    """A pair exactly at the shell cutoff is not visited (reading R4)."""
    from oracle import dsl
    pos = np.array([[1.0, 1.0, 1.0], [2.5, 1.0, 1.0]])
    box = np.array([10.0, 10.0, 10.0])
    code = "c.i[0] += 1.0;"
    d, _ = dsl.pair_loop(code, pos, box, 1.5, dats={"c": (np.zeros((2, 1)), dsl.INC_ZERO)})
    assert np.all(d["c"] == 0.0)
    d, _ = dsl.pair_loop(code, pos, box, 1.5000001, dats={"c": (np.zeros((2, 1)), dsl.INC_ZERO)})
    assert np.all(d["c"] == 1.0)


def test_periodic_image_pairs():
    """Pairs across the periodic boundary use the nearest image."""
    from oracle import dsl
    pos = np.array([[0.2, 5.0, 5.0], [9.9, 5.0, 5.0]])
    box = np.array([10.0, 10.0, 10.0])
    code = "d.i[0] += r.i[0] - r.j[0];"
    d, _ = dsl.pair_loop(code, pos, box, 1.0, dats={"d": (np.zeros((2, 1)), dsl.INC_ZERO)})
    np.testing.assert_allclose(d["d"][:, 0], [0.3, -0.3], atol=1e-12)
