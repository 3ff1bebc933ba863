"""Pins for the Andersen thermostat oracle (O8; reading R19)."""
import numpy as np
import pytest

import ljinputs as li


# Known-answer vectors of Philox4x32-10 published with Random123 (Salmon et al., SC'11,
# kat_vectors): (counter, key) -> output.
KAT = [
    ((0, 0, 0, 0), (0, 0), (0x6627e8d5, 0xe169c58d, 0xbc57ac4c, 0x9b00dbd8)),
    ((0xffffffff,) * 4, (0xffffffff,) * 2, (0x408f276d, 0x41c83b0e, 0xa20bc7c6, 0x6d5451fd)),
    ((0x243f6a88, 0x85a308d3, 0x13198a2e, 0x03707344), (0xa4093822, 0x299f31d0),
     (0xd16cfe09, 0x94fdcceb, 0x5001e420, 0x24126ea1)),
]


@pytest.mark.parametrize("ctr,key,out", KAT)
def test_philox_known_answers(ctr, key, out):
    import oracle
    assert tuple(int(x) for x in oracle.philox4x32(ctr, key)) == out


def test_nu_zero_changes_nothing():
    import oracle
    v = li.velocities(1000, 1.0)
    v2, k = oracle.andersen(v, seed=5, step=1, nu_dt=0.0, temp=2.0)
    assert k == 0 and np.array_equal(v, v2)


def test_zero_temperature_resamples_to_zero():
    import oracle
    v = li.velocities(1000, 1.0)
    v2, k = oracle.andersen(v, seed=5, step=3, nu_dt=1.0, temp=0.0)
    assert k == 1000 and np.all(v2 == 0.0)


@pytest.mark.parametrize("mass", [1.0, 2.5])
def test_maxwell_boltzmann_moments(mass):
    """nu*dt = 1: every velocity drawn from N(0, T/m): <v> = 0, <v^2> = T/m per component,
    <m v^2 / 2> = 3T/2 per particle, each within 4 standard errors (equipartition)."""
    import oracle
    n, T = 20000, 1.5
    v, k = oracle.andersen(np.zeros((n, 3)), seed=1234, step=7, nu_dt=1.0, temp=T, mass=mass)
    assert k == n
    s2 = T / mass
    se_mean = np.sqrt(s2 / n)
    assert np.all(np.abs(v.mean(axis=0)) < 4 * se_mean)
    var = (v * v).mean(axis=0)
    assert np.all(np.abs(var - s2) < 4 * s2 * np.sqrt(2.0 / n))
    ke = 0.5 * mass * (v * v).sum(axis=1)
    assert abs(ke.mean() - 1.5 * T) < 4 * ke.std() / np.sqrt(n)
    # Gaussian shape: fraction within one standard deviation
    frac = np.mean(np.abs(v / np.sqrt(s2)) < 1.0)
    assert abs(frac - 0.682689492) < 4 * np.sqrt(0.6827 * 0.3173 / (3 * n))


def test_collision_frequency_binomial():
    import oracle
    n, p = 100000, 0.03
    _, k = oracle.andersen(np.ones((n, 3)), seed=99, step=11, nu_dt=p, temp=1.0)
    assert abs(k - n * p) < 4 * np.sqrt(n * p * (1 - p))


def test_draws_are_per_particle_and_step():
    """Counter-based: the draw of (gid, step) is independent of everything else."""
    import oracle
    v1, _ = oracle.andersen(np.zeros((50, 3)), seed=3, step=10, nu_dt=1.0, temp=1.0)
    v2, _ = oracle.andersen(np.zeros((80, 3)), seed=3, step=10, nu_dt=1.0, temp=1.0)
    assert np.array_equal(v1, v2[:50])
    v3, _ = oracle.andersen(np.zeros((50, 3)), seed=3, step=11, nu_dt=1.0, temp=1.0)
    v4, _ = oracle.andersen(np.zeros((50, 3)), seed=4, step=10, nu_dt=1.0, temp=1.0)
    assert not np.any(v1 == v3) and not np.any(v1 == v4)


def test_run_thermostat_off_is_nve():
    import oracle
    pos, vel, box = li.CONFIGS["C1"].build()
    a = oracle.run(pos, vel, box, 5)
    b = oracle.run(pos, vel, box, 5, thermostat=(0.0, 3.0, 77))
    assert np.array_equal(a.vel, b.vel) and np.array_equal(a.pos, b.pos)


def test_run_thermostat_drives_temperature():
    """Strong coupling (nu*dt = 0.5) to T = 0.3 cools the T0 = 1.44 crystal: the sampled
    kinetic temperature ends within 25 % of the target (P:891's quench, short)."""
    import oracle
    pos, vel, box = li.CONFIGS["C1"].build()
    n = len(pos)
    r = oracle.run(pos, vel, box, 60, thermostat=(100.0, 0.3, 2024))
    t_end = 2.0 * r.ke[-1] / (3 * n - 3)
    assert 2.0 * r.ke[0] / (3 * n - 3) > 1.3
    assert abs(t_end - 0.3) < 0.25 * 0.3 + 0.1


def test_run_rejects_bad_probability():
    import oracle
    pos, vel, box = li.CONFIGS["C1"].build()
    with pytest.raises(ValueError):
        oracle.run(pos, vel, box, 1, thermostat=(300.0, 1.0, 1))   # nu*dt = 1.5
