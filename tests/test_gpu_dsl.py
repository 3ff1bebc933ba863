"""GPU PairLoop / ParticleLoop front end (paper_1704_03329_b200.dsl, §8(f) NEXT-3) against the
DSL oracle (oracle/dsl.py): the same user kernels, the same access descriptors, compiled with
NVRTC for sm_100a on one side and gcc on the other, with FMA contraction off on both (every
operation rounded as written), so per-pair terms agree bit for bit and only summation
order differs."""
import numpy as np
import pytest

import ljinputs as li
from dsl_kernels import CNA_I, CNA_II, KINETIC, LJ, LJ_CONSTANTS, SIMPLE, VEL_UPDATE

pytestmark = pytest.mark.gpu


def c1(cells=6, sigma_d=0.05, t0=1.44):
    pos, box = li.fcc(cells, cells, cells)
    pos = li.perturb(pos, sigma_d)
    return pos, li.velocities(len(pos), t0), box


def consts(d):
    from paper_1704_03329_b200 import dsl
    return tuple(dsl.Constant(k, v) for k, v in d.items())


@pytest.mark.parametrize("steps", [0, 25])
def test_lj_listing_pairloop(orc, steps):
    """Listing 9 as a PairLoop (shell_cutoff = rc, Listing lst:LJ-loop) equals the oracle's
    pair loop on the same positions (|dF| <= 1e-12 S_i) and the engine's own force kernel
    within the force parity bar."""
    from oracle import dsl as odsl
    from paper_1704_03329_b200 import LJMD, dsl
    pos, vel, box = c1()
    n = len(pos)
    with LJMD(pos, vel, box) as st:
        st.step(steps)
        F = dsl.ParticleDat(st, ncomp=3)
        u = dsl.ScalarArray(st, ncomp=1)
        loop = dsl.PairLoop(dsl.Kernel("lj", LJ, consts(LJ_CONSTANTS)),
                            {"r": dsl.PositionDat(st)(dsl.READ), "F": F(dsl.INC_ZERO), "u": u(dsl.INC_ZERO)},
                            shell_cutoff=li.RC)
        loop.execute()
        Fg, ug = F.data, u.data
        x = st.positions()
        Fe = st.forces()
    d, s = odsl.pair_loop(LJ, x, box, li.RC, dats={"F": (np.zeros((n, 3)), odsl.INC_ZERO)},
                          scalars={"u": (np.zeros(1), odsl.INC_ZERO)}, constants=LJ_CONSTANTS)
    ref = orc.forces(x, box, orc.LJ(rc=li.RC))
    S = ref.S[:, None]
    assert np.all(np.abs(Fg - d["F"]) <= 1e-12 * S)
    assert abs(ug[0] - s["u"][0]) <= 1e-12 * np.sum(ref.A)
    assert np.all(np.abs(Fg - Fe) <= 1e-10 * S)


def test_simple_op_example(orc):
    """Eqs. eqn:simple_op / eqn:simple_op_global (Listing lst:simple-kernel): a READ dat
    read on the j side, an INC dat, an INC ScalarArray used as `S += ...`."""
    from oracle import dsl as odsl
    from paper_1704_03329_b200 import LJMD, dsl
    pos, vel, box = c1(cells=5)
    n = len(pos)
    a0 = np.random.default_rng(11).standard_normal((n, 3))
    with LJMD(pos, vel, box) as st:
        a = dsl.ParticleDat(st, ncomp=3)
        a.data = a0
        b = dsl.ParticleDat(st, ncomp=1, initial_value=1.0)
        S = dsl.ScalarArray(st, ncomp=1, initial_value=2.0)
        loop = dsl.PairLoop(dsl.Kernel("update_b", SIMPLE, (dsl.Constant("dimension", 3),)),
                            {"r": dsl.PositionDat(st)(dsl.READ), "a": a(dsl.READ), "b": b(dsl.INC), "S": S(dsl.INC)},
                            shell_cutoff=1.6)
        loop.execute()
        bg, Sg, x = b.data, S.data, st.positions()
        assert np.array_equal(a.data, a0)
    d, s = odsl.pair_loop(SIMPLE, x, box, 1.6, dats={"a": (a0, odsl.READ), "b": (np.ones((n, 1)), odsl.INC)},
                          scalars={"S": (np.full(1, 2.0), odsl.INC)}, constants={"dimension": 3})
    np.testing.assert_allclose(bg, d["b"], rtol=1e-13)
    np.testing.assert_allclose(Sg, s["S"], rtol=1e-13)


def test_particle_loops_velocity_update_and_kinetic(orc):
    """Listing lst:velocity_update on the engine's velocities (RW) and forces (READ): bitwise
    v + F dt/(2m); Example 1's kinetic energy as a global INC."""
    from oracle import dsl as odsl
    from paper_1704_03329_b200 import LJMD, dsl
    pos, vel, box = c1()
    n = len(pos)
    with LJMD(pos, vel, box) as st:
        v0, F0 = st.velocities(), st.forces()
        up = dsl.ParticleLoop(dsl.Kernel("vel", VEL_UPDATE, (dsl.Constant("dht_iMASS", 0.0025),)),
                              {"v": dsl.velocities(st)(dsl.RW), "F": dsl.forces(st)(dsl.READ)})
        up.execute()
        v1 = st.velocities()
        k = dsl.ScalarArray(st)
        ke = dsl.ParticleLoop(dsl.Kernel("ke", KINETIC, (dsl.Constant("mass", 1.0),)),
                              {"v": dsl.velocities(st)(dsl.READ), "k": k(dsl.INC_ZERO)})
        ke.execute()
        kg = k.data[0]
    d, _ = odsl.particle_loop(VEL_UPDATE, n, dats={"v": (v0, odsl.RW), "F": (F0, odsl.READ)},
                              constants={"dht_iMASS": 0.0025})
    assert np.array_equal(v1, d["v"])
    assert abs(kg - orc.kinetic(v1)) <= 1e-12 * kg


def test_cna_listings_pairloops(orc):
    """Listings lst:CNA-kernel_I/II as pair loops: int64 dats, the engine's global ids on
    both sides, a wide WRITE/RW dat (direct global access) read on the j side (R20)."""
    from oracle import dsl as odsl
    from paper_1704_03329_b200 import LJMD, dsl
    pos, box = li.fcc(5, 5, 5)
    pos = li.perturb(pos, 0.03)
    n = len(pos)
    rc = (li.fcc_lattice_constant() * (1 / np.sqrt(2) + 1)) / 2
    W = 2 * 24 * 24
    with LJMD(pos, np.zeros_like(pos), box) as st:
        ids = dsl.global_ids(st)
        n_nb = dsl.ParticleDat(st, dtype=np.int64)
        n_bond = dsl.ParticleDat(st, dtype=np.int64)
        bond = dsl.ParticleDat(st, ncomp=W, dtype=np.int64)
        k1 = dsl.PairLoop(dsl.Kernel("cna1", CNA_I, (dsl.Constant("rc_sq", rc * rc),)),
                          {"r": dsl.PositionDat(st)(dsl.READ), "id": ids(dsl.READ), "n_nb": n_nb(dsl.INC_ZERO),
                           "n_bond": n_bond(dsl.INC_ZERO), "bond": bond(dsl.WRITE)}, shell_cutoff=rc)
        k1.execute()
        k2 = dsl.PairLoop(dsl.Kernel("cna2", CNA_II, (dsl.Constant("rc_sq", rc * rc),)),
                          {"r": dsl.PositionDat(st)(dsl.READ), "id": ids(dsl.READ), "n_nb": n_nb(dsl.READ),
                           "n_bond": n_bond(dsl.INC), "bond": bond(dsl.RW)}, shell_cutoff=rc)
        k2.execute()
        g_nb, g_b, g_bond, x = n_nb.data, n_bond.data, bond.data, st.positions()
    gids = np.arange(n, dtype=np.int64).reshape(-1, 1)
    base = {"id": (gids, odsl.READ)}
    d1, _ = odsl.pair_loop(CNA_I, x, box, rc, dats={**base, "n_nb": (np.zeros((n, 1), np.int64), odsl.INC_ZERO),
                                                  "n_bond": (np.zeros((n, 1), np.int64), odsl.INC_ZERO),
                                                  "bond": (np.zeros((n, W), np.int64), odsl.WRITE)},
                           constants={"rc_sq": rc * rc})
    d2, _ = odsl.pair_loop(CNA_II, x, box, rc, dats={**base, "n_nb": (d1["n_nb"], odsl.READ),
                                                   "n_bond": (d1["n_bond"], odsl.INC), "bond": (d1["bond"], odsl.RW)},
                           constants={"rc_sq": rc * rc})
    assert np.array_equal(g_nb, d1["n_nb"]) and np.array_equal(g_b, d2["n_bond"])
    for i in range(n):
        m, k = g_b[i, 0], g_nb[i, 0]
        got = g_bond[i, :2 * m].reshape(-1, 2)
        ref = d2["bond"][i, :2 * m].reshape(-1, 2)
        assert sorted(map(tuple, got[:k])) == sorted(map(tuple, ref[:k]))
        assert sorted(map(tuple, got)) == sorted(map(tuple, ref))


def test_dats_follow_particles_across_rebuilds_and_set_state(orc):
    from paper_1704_03329_b200 import LJMD, dsl
    pos, vel, box = c1(cells=5)
    n = len(pos)
    tag = np.arange(n, dtype=np.int64) * 7 + 3
    with LJMD(pos, vel, box) as st:
        a = dsl.ParticleDat(st, dtype=np.int64)
        a.data = tag.reshape(-1, 1)
        st.step(45)                    # two rebuilds: the engine reorders its particles
        assert np.array_equal(a.data[:, 0], tag)
        st.set_state(pos, vel)
        assert np.array_equal(a.data[:, 0], tag)
        # a particle loop sees each particle's own row: copy the gid next to the tag
        g = dsl.ParticleDat(st, ncomp=2, dtype=np.int64)
        dsl.ParticleLoop(dsl.Kernel("cp", "g.i[0] = a.i[0]; g.i[1] = id.i[0];"),
                         {"a": a(dsl.READ), "g": g(dsl.WRITE), "id": dsl.global_ids(st)(dsl.READ)}).execute()
        out = g.data
    assert np.array_equal(out[:, 0], tag) and np.array_equal(out[:, 1], np.arange(n))


def test_generated_source_and_errors():
    from paper_1704_03329_b200 import LJMD, LjmdError, dsl
    pos, vel, box = c1(cells=5)
    with LJMD(pos, vel, box) as st:
        b = dsl.ParticleDat(st)
        loop = dsl.ParticleLoop(dsl.Kernel("k", "b.i[0] = 2.0;"), {"b": b(dsl.WRITE)})
        assert "b.i[0] = 2.0;" in loop.source and "extern \"C\" __global__" in loop.source
        loop.execute()
        assert np.all(b.data == 2.0)
        with pytest.raises(LjmdError, match="shell_cutoff"):
            dsl.PairLoop(dsl.Kernel("k", "b.i[0] += 1.0;"), {"b": b(dsl.INC)}, shell_cutoff=3.0)
    with LJMD(pos, vel, box) as st:
        b = dsl.ParticleDat(st)
        with pytest.raises(LjmdError, match="does not compile"):
            dsl.ParticleLoop(dsl.Kernel("bad", "b.i[0] = undefined_name;"), {"b": b(dsl.WRITE)})
    with LJMD(pos, vel, box) as st:
        with pytest.raises(LjmdError, match="READ only"):
            dsl.ParticleLoop(dsl.Kernel("k", "F.i[0] = 0.0;"), {"F": dsl.forces(st)(dsl.WRITE)})
    with LJMD(pos, vel, box) as st:
        S = dsl.ScalarArray(st)
        with pytest.raises(LjmdError, match="ScalarArray"):
            dsl.ParticleLoop(dsl.Kernel("k", "S[0] = 1.0;"), {"S": S(dsl.WRITE)})
