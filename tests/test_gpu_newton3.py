"""Newton-3 half-list variant (ljmd_options.newton3) against the oracle:
the same parity bar as the default path (|dF| <= 1e-10 S_i, |de| <= 1e-10 A_i / 2; 100-step
energies within 1e-8), the half list holding exactly one entry per unordered pair."""
import numpy as np
import pytest

import ljinputs as li

pytestmark = pytest.mark.gpu

TOL = 1e-10


def c1(sigma_d=0.05, t0=1.44, cells=10):
    pos, box = li.fcc(cells, cells, cells)
    if sigma_d:
        pos = li.perturb(pos, sigma_d)
    return pos, li.velocities(len(pos), t0), box


def check(ctx, orc, box):
    x = ctx.positions()
    ref = orc.forces(x, box, orc.LJ(rc=li.RC, shift=0.25))
    F = ctx.forces()
    e = ctx.particle_energy()
    assert np.all(np.abs(F - ref.F) <= TOL * ref.S[:, None] + 1e-300)
    assert np.all(np.abs(e - ref.e) <= TOL * 0.5 * ref.A + 1e-300)
    return ref


@pytest.mark.parametrize("sigma_d", [0.0, 0.05])
def test_init_forces(orc, sigma_d):
    from paper_1704_03329_b200 import LJMD
    pos, vel, box = c1(sigma_d)
    with LJMD(pos, vel, box, newton3=1) as ctx:
        ref = check(ctx, orc, box)
        pe, ke = ctx.energy()
    assert abs(pe - ref.pe) <= 1e-10 * np.sum(0.5 * ref.A)


def test_after_steps_and_rebuilds(orc):
    from paper_1704_03329_b200 import LJMD
    pos, vel, box = c1()
    with LJMD(pos, vel, box, newton3=1) as ctx:
        ctx.step(27)
        check(ctx, orc, box)
        assert ctx.rebuild_steps().tolist() == [20]


@pytest.mark.parametrize("check_policy", [0, 1])
def test_trajectory_energies(orc, check_policy):
    from paper_1704_03329_b200 import LJMD
    pos, vel, box = c1(sigma_d=0.0)
    with LJMD(pos, vel, box, newton3=1, rebuild_check=check_policy) as ctx:
        ctx.step(100)
        pe, ke = ctx.energy_history()
        rs = ctx.rebuild_steps()
    r = orc.run(pos, vel, box, 100, check=check_policy, mode="list")
    assert rs.tolist() == r.rebuild_steps.tolist()
    scale = np.abs(r.pe) + np.abs(r.ke)
    assert np.all(np.abs(pe - r.pe) <= 1e-8 * scale)
    assert np.all(np.abs(ke - r.ke) <= 1e-8 * scale)


def test_matches_full_list_path():
    """Same trajectory as the default (full-list, fused) path to round-off over 40 steps."""
    from paper_1704_03329_b200 import LJMD
    pos, vel, box = c1()
    with LJMD(pos, vel, box) as a, LJMD(pos, vel, box, newton3=1) as b:
        a.step(40)
        b.step(40)
        np.testing.assert_allclose(b.positions(), a.positions(), rtol=0, atol=1e-9)
        np.testing.assert_allclose(b.velocities(), a.velocities(), rtol=0, atol=1e-8)


def test_thermostat_with_newton3(orc):
    from paper_1704_03329_b200 import LJMD
    pos, vel, box = c1(sigma_d=0.0)
    th = (0.05 / li.DT, 0.5, 424242)
    with LJMD(pos, vel, box, newton3=1) as ctx:
        ctx.set_thermostat(*th)
        ctx.step(60)
        pe, ke = ctx.energy_history()
    r = orc.run(pos, vel, box, 60, mode="list", thermostat=th)
    scale = np.abs(r.pe) + np.abs(r.ke)
    assert np.all(np.abs(pe - r.pe) <= 1e-8 * scale)
    assert np.all(np.abs(ke - r.ke) <= 1e-8 * scale)


def test_newton3_rejects_multirank():
    from paper_1704_03329_b200 import LJMD, LjmdError
    pos, vel, box = c1()
    with pytest.raises(LjmdError, match="newton3"):
        LJMD(pos, vel, box, newton3=1, split_self=1)
