"""GPU Andersen thermostat (ljmd_set_thermostat, reading R19) against the oracle's O8:
the same Philox4x32-10 draws keyed by (seed, gid, step), so the collision decisions are
identical and the new velocities agree to a few ulps (libm vs CUDA log/sin/cos)."""
import numpy as np
import pytest

import ljinputs as li

pytestmark = pytest.mark.gpu


def c1(sigma_d=0.05, t0=1.44, cells=10):
    pos, box = li.fcc(cells, cells, cells)
    if sigma_d:
        pos = li.perturb(pos, sigma_d)
    return pos, li.velocities(len(pos), t0), box


def test_full_collision_one_step(orc):
    """nu*dt = 1: after one step every velocity is the oracle's draw for (gid, step 1)."""
    from paper_1704_03329_b200 import LJMD
    pos, vel, box = c1()
    with LJMD(pos, vel, box) as ctx:
        ctx.set_thermostat(1.0 / li.DT, 0.7, seed=314159)
        ctx.step(1)
        v = ctx.velocities()
    ref, k = orc.andersen(np.zeros_like(vel), seed=314159, step=1, nu_dt=1.0, temp=0.7)
    assert k == len(pos)
    np.testing.assert_allclose(v, ref, rtol=1e-14, atol=1e-15)


def test_partial_collisions_decisions_exact(orc):
    """nu*dt = 0.2: exactly the particles the oracle selects change velocity."""
    from paper_1704_03329_b200 import LJMD
    pos, vel, box = c1()
    nu, T, seed = 0.2 / li.DT, 1.0, 2718
    with LJMD(pos, vel, box) as ctx:
        ctx.step(2)
        ctx.set_thermostat(nu, T, seed)
        ctx.step(1)
        v_after = ctx.velocities()
    # expected: the NVE velocities of step 3, replaced by the oracle's collisions of step 3
    with LJMD(pos, vel, box) as ctx:
        ctx.step(3)
        v_nve = ctx.velocities()
    sel_ref, _ = orc.andersen(np.full_like(vel, np.nan), seed=seed, step=3, nu_dt=0.2, temp=T)
    sel = ~np.isnan(sel_ref[:, 0])
    assert 0.1 * len(pos) < sel.sum() < 0.3 * len(pos)
    assert np.array_equal(v_after[~sel], v_nve[~sel])
    np.testing.assert_allclose(v_after[sel], sel_ref[sel], rtol=1e-14, atol=1e-15)


@pytest.mark.parametrize("check", [0, 1])
def test_thermostat_trajectory_vs_oracle(orc, check):
    """C1, 100 steps with collisions every step (nu*dt = 0.05) towards T = 0.5: sampled PE,
    KE within 1e-8 relative of the oracle's thermostatted run, same rebuild steps."""
    from paper_1704_03329_b200 import LJMD
    pos, vel, box = c1(sigma_d=0.0)
    th = (0.05 / li.DT, 0.5, 424242)
    with LJMD(pos, vel, box, rebuild_check=check) as ctx:
        ctx.set_thermostat(*th)
        ctx.step(40)
        ctx.step(60)
        pe, ke = ctx.energy_history()
        rs = ctx.rebuild_steps()
    r = orc.run(pos, vel, box, 100, check=check, mode="list", thermostat=th)
    assert rs.tolist() == r.rebuild_steps.tolist()
    scale = np.abs(r.pe) + np.abs(r.ke)
    assert np.all(np.abs(pe - r.pe) <= 1e-8 * scale)
    assert np.all(np.abs(ke - r.ke) <= 1e-8 * scale)
    assert ke[-1] < 0.8 * ke[0]    # cooling towards T = 0.5 from 1.44


def test_nu_zero_is_nve():
    from paper_1704_03329_b200 import LJMD
    pos, vel, box = c1()
    with LJMD(pos, vel, box) as a, LJMD(pos, vel, box) as b:
        b.set_thermostat(0.0, 5.0, 1)
        a.step(30)
        b.step(30)
        assert np.array_equal(a.velocities(), b.velocities())
        assert np.array_equal(a.positions(), b.positions())


def test_thermostat_decomposition_bitwise():
    """The draws are keyed by gid and step: p = 2 and 3 slabs equal p = 1 bit for bit."""
    from test_gpu_multirank import run_ranks, single
    pos, box = li.fcc(6, 6, 9)
    pos = li.perturb(pos, 0.05)
    vel = li.velocities(len(pos), 1.44)
    th = (0.1 / li.DT, 0.8, 99)
    ref = single(pos, vel, box, 45, thermostat=th, list_order=0)
    for nr in (2, 3):
        got, _ = run_ranks(nr, pos, vel, box, 45, thermostat=th, list_order=0)
        assert np.array_equal(got["V"], ref["V"])
        assert np.array_equal(got["X"], ref["X"])


def test_thermostat_errors():
    from paper_1704_03329_b200 import LJMD, LjmdError
    pos, vel, box = c1()
    with LJMD(pos, vel, box) as ctx:
        with pytest.raises(LjmdError, match="nu"):
            ctx.set_thermostat(1.5 / li.DT, 1.0)
        with pytest.raises(LjmdError):
            ctx.set_thermostat(1.0, -1.0)
