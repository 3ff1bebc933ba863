"""GPU: the rebuild rule, dangerous builds and missed pairs against the oracle (reading R7,
Eq. eqn:extended_cutoff PAPER.md:406-416, the paper's fixed Ns = 20 PAPER.md:728, 741),
and neighbour sets built on the rebuild path at full size."""
import numpy as np
import pytest

import ljinputs as li
from conftest import cuda_available

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_available(), reason="needs a CUDA device")]

DT = 1.0 / 64.0
BOX = np.array([9.0, 9.0, 9.0])
RN = li.RC + li.DELTA


@pytest.fixture(scope="module")
def eng():
    from paper_1704_03329_b200 import ljmd
    ljmd.load()
    return ljmd


def test_safe_threshold_closed_form(eng):
    """One particle (N = 1, an empty list) at |v| = 1, dt = 1/64: rebuilds at 9, 18, 27, 36
    (2 k/64 > 1/4 first at k = 9; k = 8 is exactly delta, not rebuilt) -- the oracle's pin
    in closed form; the flight itself is exact."""
    pos = np.array([[1.0, 4.5, 4.5]])
    vel = np.array([[1.0, 0.0, 0.0]])
    with eng.LJMD(pos, vel, BOX, dt=DT, rebuild_every=1000, rebuild_check=1, energy_every=0) as ctx:
        ctx.step(40)
        assert ctx.rebuild_steps().tolist() == [9, 18, 27, 36]
        np.testing.assert_array_equal(ctx.positions(), [[1.0 + 40 * DT, 4.5, 4.5]])
        assert ctx.stats()["dangerous_builds"] == 0


def test_missed_pairs_closed_form(eng):
    """Head-on approach from r = 3 under the fixed schedule: validation counts 2 particles /
    2 ordered pairs on every step from 17 on (r(k) = 3 - k/32 < 2.5), none before."""
    pos = np.array([[3.0, 4.5, 4.5], [6.0, 4.5, 4.5]])
    vel = np.array([[1.0, 0.0, 0.0], [-1.0, 0.0, 0.0]])
    with eng.LJMD(pos, vel, BOX, dt=DT, rebuild_every=1000, energy_every=0, validate=1) as ctx:
        ctx.step(30)
        ctx.step(10)
        v = ctx.validation()
        k = np.arange(1, 41)
        want = np.where(k >= 17, 2, 0)
        np.testing.assert_array_equal(v[:, 0], k)
        np.testing.assert_array_equal(v[:, 1], want)
        np.testing.assert_array_equal(v[:, 2], want)
        st = ctx.stats()
        assert st["validated_steps"] == 40 and st["missed_pairs"] == 2 * 24
        assert st["missed_particle_steps"] == 2 * 24 and st["max_missed_particles"] == 2
    with eng.LJMD(pos, vel, BOX, dt=DT, rebuild_every=1000, rebuild_check=1, energy_every=0, validate=1) as ctx:
        ctx.step(40)
        assert ctx.rebuild_steps()[0] == 9
        assert not ctx.validation()[:, 1:].any()


@pytest.fixture(scope="module")
def fcc_fixed(orc):
    """C1 perfect FCC at T0 = 1.44 (the verdict's case), 40 steps of the oracle with the
    paper's fixed Ns = 20 and validation on."""
    pos, box = li.fcc(10, 10, 10)
    vel = li.velocities(len(pos), 1.44)
    r = orc.run(pos, vel, box, 40, validate=True, omp=True)
    return pos, vel, box, r


def test_missed_pairs_match_oracle(eng, fcc_fixed):
    """Per-step missed-pair counts of the GPU's validation mode equal the oracle's at every
    step of a 40-step fixed-20 run (18 particles at step 19, the last step the init list
    serves); the counts reset at the rebuilds (steps 20, 40)."""
    pos, vel, box, r = fcc_fixed
    with eng.LJMD(pos, vel, box, validate=1) as ctx:
        ctx.step(40)
        v = ctx.validation()
    assert v[:, 0].tolist() == list(range(1, 41))
    np.testing.assert_array_equal(v[:, 1], r.missed_particles[1:])
    np.testing.assert_array_equal(v[:, 2], r.missed_pairs[1:])
    assert v[18, 1] == 18 and v[19, 1] == 0


def test_dangerous_builds_match_oracle(eng, orc, fcc_fixed):
    """Dangerous builds (2 max|x(s-1) - x(build)| > delta at a rebuild s) and the largest
    such displacement, against the oracle's trajectory: builds at 0 (init, not counted), 20
    and 40; the positions served last are x(19) and x(39)."""
    pos, vel, box, r = fcc_fixed
    x_build0 = orc.wrap(pos, box)
    x19 = orc.run(pos, vel, box, 19, energy_every=0).pos
    x20 = orc.run(pos, vel, box, 20, energy_every=0).pos          # wrapped at the rebuild
    x39 = orc.run(pos, vel, box, 39, energy_every=0).pos
    d1 = np.sqrt(((x19 - x_build0) ** 2).sum(axis=1)).max()
    d2 = np.sqrt(((x39 - x20) ** 2).sum(axis=1)).max()
    want = int(2 * d1 > li.DELTA) + int(2 * d2 > li.DELTA)
    with eng.LJMD(pos, vel, box) as ctx:
        ctx.step(40)
        st = ctx.stats()
    assert st["dangerous_builds"] == want == 2
    assert abs(st["max_build_disp"] - max(d1, d2)) <= 1e-12 * max(d1, d2)


def test_safe_policy_no_missed_no_dangerous(eng, orc):
    """Displacement-checked policy on a melt (C1 perturbed): no missed pair on any step, no
    dangerous build, and the same rebuild steps as the oracle."""
    pos, box = li.fcc(10, 10, 10)
    pos = li.perturb(pos, 0.05)
    vel = li.velocities(len(pos), 1.44)
    with eng.LJMD(pos, vel, box, rebuild_check=1, validate=1) as ctx:
        ctx.step(60)
        v = ctx.validation()
        st = ctx.stats()
        steps = ctx.rebuild_steps()
    assert not v[:, 1:].any()
    assert st["dangerous_builds"] == 0
    r = orc.run(pos, vel, box, 60, check=1, energy_every=0)
    assert steps.tolist() == r.rebuild_steps.tolist()


def test_energy_cached_after_sample_step(eng):
    """ljmd_get_energy right after a step whose last step sampled PE/KE reuses the sample
    (no extra force pass): same values as a recomputation on a fresh context."""
    pos, box = li.fcc(6, 6, 6)
    pos = li.perturb(pos, 0.05)
    vel = li.velocities(len(pos), 1.44)
    with eng.LJMD(pos, vel, box) as ctx:
        ctx.step(20)
        k0 = ctx.stats()["kernel_launches"]
        pe, ke = ctx.energy()
        assert ctx.stats()["kernel_launches"] == k0 + 1      # only the stats readback kernel
        hp, hk = ctx.energy_history()
        assert (pe, ke) == (hp[-1], hk[-1])
        e = ctx.particle_energy()
        x, v = ctx.positions(), ctx.velocities()
        ctx.step(3)                                           # not a sample step at the end
        pe3, ke3 = ctx.energy()
    with eng.LJMD(x, v, box) as c2:
        pe2, ke2 = c2.energy()
        np.testing.assert_allclose(c2.particle_energy(), e, rtol=0, atol=1e-12)
    assert abs(pe2 - pe) <= 1e-10 * abs(pe) and abs(ke2 - ke) <= 1e-12 * abs(ke)
    assert pe3 != pe


@pytest.mark.parametrize("cfg", ["C2", "C5"])
def test_full_size_rebuild_path_neighbours(eng, orc, cfg):
    """Neighbour sets built by the REBUILD path (not init) at full size: C2 after the
    rebuild at step 20 (fixed Ns), C5 after the first displacement-triggered rebuild; 64
    sampled rows equal the oracle's brute force at the build positions, which are the
    positions ljmd_step returns when the rebuild was on its last step."""
    c = li.CONFIGS[cfg]
    pos, vel, box = c.build()
    with eng.LJMD(pos, vel, box, rebuild_check=c.rebuild_check) as ctx:
        if c.rebuild_check:
            k = 0
            while ctx.stats()["n_rebuilds"] == 0:
                ctx.step(1)
                k += 1
                assert k < 40
        else:
            ctx.step(20)
        assert ctx.rebuild_steps()[-1] == ctx.stats()["steps_done"]
        x = ctx.positions()
        off, nbr = ctx.neighbours()
    n = len(x)
    rng = np.random.default_rng(1)
    rows = np.unique(np.concatenate([[0, 1, n - 1, n - 2, n // 2], rng.integers(0, n, 59)]))
    o2, n2 = orc.neighbours_rows(x, box, RN, rows)
    for r, i in enumerate(rows):
        assert sorted(nbr[off[i]:off[i + 1]].tolist()) == n2[o2[r]:o2[r + 1]].tolist()
