"""System-level pins for the oracle: FCC lattice sums, neighbour sets vs brute force,
Newton's third law, and velocity-Verlet invariants (Alg. alg:VelocityVerlet)."""
import math

import numpy as np
import pytest

import ljinputs as li

RC, DELTA = 2.5, 0.25
RN = RC + DELTA


def fcc_shell_energy(rho, rc, shift):
    """Closed-form truncated lattice sum e = 1/2 sum_{R != 0, |R| < rc} V(|R|) for FCC,
    by enumerating integer points (i,j,k), i+j+k even, scaled by a/2 (independent of the oracle)."""
    a = (4.0 / rho) ** (1.0 / 3.0)
    h = a / 2.0
    kmax = int(math.ceil(rc / h)) + 1
    tot = 0.0
    counts = {}
    for i in range(-kmax, kmax + 1):
        for j in range(-kmax, kmax + 1):
            for k in range(-kmax, kmax + 1):
                if (i + j + k) % 2 or (i == j == k == 0):
                    continue
                r2 = (i * i + j * j + k * k) * h * h
                if r2 < rc * rc:
                    s6 = 1.0 / r2 ** 3
                    tot += 4.0 * (s6 * s6 - s6 + shift)
                    counts[i * i + j * j + k * k] = counts.get(i * i + j * j + k * k, 0) + 1
    return 0.5 * tot, sum(counts.values())


@pytest.fixture(scope="module")
def fcc10():
    return li.fcc(10, 10, 10)


@pytest.mark.parametrize("shift,golden", [
    (0.0, -6.773368053252955),            # SURVEY.md §8(c) pins (closed-form shell sum)
    (0.25, 20.226631946747048),           # paper's +1/4 (Eq. eqn:LJpotential)
    (0.004079222784, -6.332811992580957), # continuous shift (sigma/rc)^6-(sigma/rc)^12
])
def test_fcc_lattice_energy(orc, fcc10, shift, golden):
    pos, box = fcc10
    f = orc.forces(pos, box, orc.LJ(rc=RC, shift=shift))
    e_closed, nnb = fcc_shell_energy(li.RHO, RC, shift)
    assert nnb == 54
    assert f.pe / len(pos) == pytest.approx(e_closed, rel=1e-13)
    assert f.pe / len(pos) == pytest.approx(golden, rel=1e-13)
    np.testing.assert_allclose(f.e, f.e[0], rtol=1e-12)
    # perfect lattice: forces vanish by symmetry
    assert np.abs(f.F).max() < 1e-12


def test_fcc_neighbour_counts(orc, fcc10):
    pos, box = fcc10
    for rn, cnt in ((RC, 54), (RN, 78)):
        off, _ = orc.neighbours(pos, box, rn, "cells")
        assert np.all(np.diff(off) == cnt)


def test_local_density_count(orc):
    """Def. 3 cost note: mean neighbours N_local = 4/3 pi rc^3 rho for a uniform fluid."""
    n, L = 3000, 15.0
    pos = li.uniform_random(n, [L] * 3, seed=5)
    off, _ = orc.neighbours(pos, [L] * 3, RN, "cells")
    expect = 4.0 / 3.0 * math.pi * RN ** 3 * n / L ** 3
    assert np.diff(off).mean() == pytest.approx(expect, rel=0.03)


def _sets(off, nbr):
    return [nbr[off[i]:off[i + 1]].tolist() for i in range(len(off) - 1)]


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_cells_equal_brute_random(orc, seed):
    """O4 == O3 as sets (reading R15: both emit ascending j) on random boxes, 3..5 cells."""
    rng = np.random.default_rng(seed)
    L = rng.uniform(8.3, 14.0, 3)
    pos = li.uniform_random(300, L, seed=seed)
    a = orc.neighbours(pos, L, RN, "brute")
    b = orc.neighbours(pos, L, RN, "cells")
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    # symmetry j in NB(i) <=> i in NB(j) away from ulp-level ties
    s = _sets(*a)
    for i, nb in enumerate(s):
        for j in nb:
            assert i in s[j]


def test_cells_equal_brute_dyadic_ties(orc):
    """Dyadic lattice with many exact ties at rbar_c = 2.75 and rc = 2.5, and seam pairs."""
    L = np.array([9.0, 9.0, 11.0])
    g = np.arange(0, 9.0, 0.25)
    rng = np.random.default_rng(7)
    pos = np.stack([rng.choice(g, 400), rng.choice(g, 400), rng.choice(np.arange(0, 11.0, 0.25), 400)], 1)
    pos = np.unique(pos, axis=0)
    for rn in (RN, RC):
        a = orc.neighbours(pos, L, rn, "brute")
        b = orc.neighbours(pos, L, rn, "cells")
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
        # exact ties are excluded (strict <)
        for i in range(len(pos)):
            for j in a[1][a[0][i]:a[0][i + 1]]:
                d = orc.displacement(pos[i], pos[j], L)
                assert orc.r2(d) < rn * rn


def test_box_too_small(orc):
    with pytest.raises(ValueError):
        orc.neighbours(np.zeros((2, 3)), [8.0, 9.0, 9.0], RN, "cells")


def test_newton_third_law(orc):
    pos, box = li.fcc(6, 6, 6)
    pos = orc.wrap(li.perturb(pos, 0.05), box)
    f = orc.forces(pos, box, orc.LJ())
    tot = f.F.sum(axis=0)
    assert np.all(np.abs(tot) <= 64 * len(pos) * 2.0 ** -53 * f.S.max())
    assert np.abs(tot).max() < 1e-10


def test_kinetic_energy_example(orc):
    """Example 1 / SPEC.md:343: m = 2, v = (1,2,2) -> KE = 9."""
    assert orc.kinetic(np.array([[1.0, 2.0, 2.0]]), mass=2.0) == 9.0


def test_neumaier_sum(orc):
    x = np.array([1.0, 1e100, 1.0, -1e100])
    assert orc.neumaier_sum(x) == 2.0


# ---------------------------------------------------------------- integrator --

def small_liquid(cells=5, t0=1.44, sigma_d=0.05):
    pos, box = li.fcc(cells, cells, cells)
    pos = li.perturb(pos, sigma_d)
    vel = li.velocities(len(pos), t0)
    return pos, vel, box


def test_free_particle(orc):
    """F = 0 (r > rc for all pairs): v unchanged bitwise, x advances by dt*v each step."""
    pos = np.array([[1.0, 1.0, 1.0], [10.0, 10.0, 10.0]])
    vel = np.array([[0.5, -0.25, 0.125], [-1.0, 0.0, 2.0]])
    r = orc.run(pos, vel, [20.0] * 3, 10, dt=0.0625, mode="brute")
    assert np.array_equal(r.vel, vel)
    exp = pos + 10 * 0.0625 * vel
    np.testing.assert_allclose(r.pos, exp % 20.0, rtol=0, atol=1e-14)


def test_two_half_kicks_equal_one(orc):
    """the two half-kicks of one step with constant F add dt/m * F.
    Uniformly accelerated pair far apart: use a single step with a known force."""
    pos = np.array([[1.0, 1.0, 1.0], [2.0, 1.0, 1.0]])   # r = 1: g = 24, F0 = (-24,0,0)
    vel = np.zeros((2, 3))
    dt = 2.0 ** -20
    r = orc.run(pos, vel, [20.0] * 3, 1, dt=dt, mode="brute")
    # v(1) = h F(0) + h F(1) with F(1) ~ F(0) to O(dt^2)
    assert r.vel[0, 0] == pytest.approx(-24.0 * dt, rel=1e-9)
    assert r.vel[1, 0] == pytest.approx(24.0 * dt, rel=1e-9)


def test_momentum_conserved(orc):
    pos, vel, box = small_liquid()
    r = orc.run(pos, vel, box, 200, mode="list", check=1)
    p0 = vel.sum(axis=0)
    assert np.abs(r.vel.sum(axis=0) - p0).max() < 1e-11


def test_reversibility(orc):
    """50 steps forward, negate v, 50 steps -> initial state within 1e-6."""
    pos, vel, box = small_liquid()
    shift = orc.LJ(shift=0.004079222784)
    a = orc.run(pos, vel, box, 50, lj=shift, mode="brute", ns=1000)
    b = orc.run(a.pos, -a.vel, box, 50, lj=shift, mode="brute", ns=1000)
    x0 = orc.wrap(pos, box)
    d = b.pos - x0
    d -= box * np.round(d / box)
    assert np.abs(d).max() < 1e-6
    assert np.abs(b.vel + vel).max() < 1e-6


def test_list_equals_brute_bitwise_safe_policy(orc):
    """With the displacement-checked rebuild (reading R7) the Verlet list is an exact
    accelerator of the brute-force pair loop: identical trajectories bit for bit."""
    pos, vel, box = small_liquid()
    a = orc.run(pos, vel, box, 100, mode="brute", check=1)
    b = orc.run(pos, vel, box, 100, mode="list", check=1)
    assert np.array_equal(a.pos, b.pos) and np.array_equal(a.vel, b.vel)
    assert np.array_equal(a.pe, b.pe) and np.array_equal(a.rebuild_steps, b.rebuild_steps)
    assert len(b.rebuild_steps) >= 3


def test_fixed_schedule(orc):
    pos, vel, box = small_liquid()
    r = orc.run(pos, vel, box, 100, ns=20, check=0)
    assert r.rebuild_steps.tolist() == [20, 40, 60, 80, 100]


def test_nve_drift_and_second_order(orc):
    """Continuous shift (reading R3): |dE|/|E| small over 100 steps, and the energy error of
    VV is O(dt^2): halving dt divides the max deviation by ~4 (a first-order slip would give 2)."""
    pos, vel, box = small_liquid(cells=6, t0=0.72)
    lj = orc.LJ(shift=0.004079222784)
    devs = []
    for dt in (0.004, 0.002):
        n = int(round(0.4 / dt))
        r = orc.run(pos, vel, box, n, lj=lj, dt=dt, mode="list", check=1, energy_every=1)
        E = r.pe + r.ke
        devs.append(np.abs(E - E[0]).max() / abs(E[0]))
    assert devs[0] < 1e-4
    assert 3.0 < devs[0] / devs[1] < 5.0


def test_row_sampled_equals_full(orc):
    """The row-restricted brute force (used for full-size sampled checks) equals the full one."""
    pos, box = li.fcc(5, 5, 6)
    pos = orc.wrap(li.perturb(pos, 0.05), box)
    rows = np.array([0, 7, 123, len(pos) - 1])
    full = orc.forces(pos, box, orc.LJ())
    part = orc.forces_rows(pos, box, rows, orc.LJ())
    assert np.array_equal(part.F, full.F[rows]) and np.array_equal(part.e, full.e[rows])
    off, nbr = orc.neighbours(pos, box, RN, "brute")
    o2, n2 = orc.neighbours_rows(pos, box, RN, rows)
    for r, i in enumerate(rows):
        assert nbr[off[i]:off[i + 1]].tolist() == n2[o2[r]:o2[r + 1]].tolist()
