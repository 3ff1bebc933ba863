"""Multi-rank z-slab decomposition on ONE GPU through the in-process loopback transport
(several contexts of this process, one per host thread, exchanging halo planes, migrants
and reductions with device copies) -- the same device code path NCCL drives on 1-8 GPUs.

Decomposition invariance: slab boundaries lie on global cell planes,
ghosts are x_j + s*L rounded once, every list is emitted in (stencil row, slot) order and
cells are sorted by (x, gid), so each particle sees the same neighbours in the same order:
positions, velocities and forces are BITWISE equal to the single-rank run.
"""
import threading
import uuid

import numpy as np
import pytest

import ljinputs as li

pytestmark = pytest.mark.gpu


def run_ranks(nranks, pos, vel, box, nsteps, thermostat=None, **kw):
    from paper_1704_03329_b200 import ljmd
    gid = ljmd.local_group_id(uuid.uuid4().hex)
    out = [None] * nranks
    err = [None] * nranks

    def work(r):
        try:
            with ljmd.LJMD(pos, vel, box, rank=r, nranks=nranks, nccl_id=gid, **kw) as ctx:
                if thermostat is not None:
                    ctx.set_thermostat(*thermostat)
                ctx.step(nsteps)
                F = np.full((len(pos), 3), np.nan)
                X = np.full((len(pos), 3), np.nan)
                V = np.full((len(pos), 3), np.nan)
                ctx._ck(ctx._lib.ljmd_get_forces(ctx._h, ljmd._dp(F)))
                ctx._ck(ctx._lib.ljmd_get_positions(ctx._h, ljmd._dp(X), 0))
                ctx._ck(ctx._lib.ljmd_get_velocities(ctx._h, ljmd._dp(V)))
                pe, ke = ctx.energy()
                out[r] = dict(F=F, X=X, V=V, pe=pe, ke=ke, hist=ctx.energy_history(), st=ctx.stats(),
                              rs=ctx.rebuild_steps())
        except Exception as e:  # noqa: BLE001
            err[r] = e

    th = [threading.Thread(target=work, args=(r,)) for r in range(nranks)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    assert not any(t.is_alive() for t in th), "rank thread hung"
    for e in err:
        if e is not None:
            raise e
    merged = {}
    for k in ("F", "X", "V"):
        a = np.full((len(pos), 3), np.nan)
        for o in out:
            m = ~np.isnan(o[k][:, 0])
            assert np.all(np.isnan(a[m, 0])), "a particle owned by two ranks"
            a[m] = o[k][m]
        assert not np.isnan(a).any(), "a particle owned by no rank"
        merged[k] = a
    return merged, out


def single(pos, vel, box, nsteps, thermostat=None, **kw):
    from paper_1704_03329_b200 import ljmd
    with ljmd.LJMD(pos, vel, box, **kw) as ctx:
        if thermostat is not None:
            ctx.set_thermostat(*thermostat)
        ctx.step(nsteps)
        return dict(F=ctx.forces(), X=ctx.positions(), V=ctx.velocities(), e=ctx.energy(),
                    hist=ctx.energy_history(), rs=ctx.rebuild_steps())


@pytest.mark.parametrize("nranks", [2, 3])
def test_decomposition_bitwise(nranks):
    """C1-like liquid (6 x 6 x 9 FCC cells -> 9 z planes): p = 2 (both neighbours the same
    rank) and p = 3, 45 steps (two rebuilds with migration) equal p = 1 bit for bit."""
    pos, box = li.fcc(6, 6, 9)
    pos = li.perturb(pos, 0.05)
    vel = li.velocities(len(pos), 1.44)
    ref = single(pos, vel, box, 45, list_order=0)
    got, per = run_ranks(nranks, pos, vel, box, 45, list_order=0)
    assert np.array_equal(got["X"], ref["X"])
    assert np.array_equal(got["V"], ref["V"])
    assert np.array_equal(got["F"], ref["F"])
    # global energies: same terms, reduction order differs across ranks
    for o in per:
        assert o["pe"] == pytest.approx(ref["e"][0], rel=1e-12)
        assert o["ke"] == pytest.approx(ref["e"][1], rel=1e-12)
        np.testing.assert_allclose(o["hist"][0], ref["hist"][0], rtol=1e-12)
        assert o["rs"].tolist() == ref["rs"].tolist()
    assert sum(o["st"]["n_owned"] for o in per) == len(pos)


@pytest.mark.parametrize("nranks,check", [(2, 0), (3, 0), (2, 1)])
def test_decomposition_overlapped_halo_bitwise(nranks, check):
    """Slabs thick enough for the overlapped halo path (>= 3 tile layers per rank: 6 x 6 x 24
    FCC cells -> 14 z planes): the boundary planes travel on the second stream in the
    receiver's ghost-plane layout while the interior tiles compute, the two boundary tile
    layers run as one launch after it.  45 steps (two rebuilds with migration; also under
    the displacement-checked policy) equal p = 1 bit for bit."""
    pos, box = li.fcc(6, 6, 24)
    pos = li.perturb(pos, 0.05)
    vel = li.velocities(len(pos), 1.44)
    ref = single(pos, vel, box, 45, list_order=0, rebuild_check=check)
    got, per = run_ranks(nranks, pos, vel, box, 45, list_order=0, rebuild_check=check)
    assert np.array_equal(got["X"], ref["X"])
    assert np.array_equal(got["V"], ref["V"])
    assert np.array_equal(got["F"], ref["F"])
    for o in per:
        assert o["rs"].tolist() == ref["rs"].tolist()


def test_decomposition_default_order():
    """With the (default) bank-aware neighbour order the per-particle summation order
    depends on the tiling, so p = 2 agrees with p = 1 to rounding, not bitwise."""
    pos, box = li.fcc(6, 6, 8)
    pos = li.perturb(pos, 0.05)
    vel = li.velocities(len(pos), 1.44)
    ref = single(pos, vel, box, 10)
    got, _ = run_ranks(2, pos, vel, box, 10)
    np.testing.assert_allclose(got["X"], ref["X"], rtol=0, atol=1e-12)
    np.testing.assert_allclose(got["F"], ref["F"], rtol=0, atol=1e-9)


def test_decomposition_against_oracle(orc):
    """p = 2 after 21 steps: forces of every particle vs the oracle's brute force."""
    pos, box = li.fcc(6, 6, 8)
    pos = li.perturb(pos, 0.05)
    vel = li.velocities(len(pos), 1.44)
    got, _ = run_ranks(2, pos, vel, box, 21)
    ref = orc.forces(got["X"], box, orc.LJ(rc=li.RC, shift=0.25))
    assert np.all(np.abs(got["F"] - ref.F) <= 1e-10 * ref.S[:, None])


def test_decomposition_safe_policy():
    """Displacement-checked rebuilds need a global max (all-reduce) each step."""
    pos, box = li.fcc(6, 6, 8)
    pos = li.perturb(pos, 0.05)
    vel = li.velocities(len(pos), 2.5)
    ref = single(pos, vel, box, 40, rebuild_check=1, list_order=0)
    got, per = run_ranks(2, pos, vel, box, 40, rebuild_check=1, list_order=0)
    assert np.array_equal(got["X"], ref["X"])
    for o in per:
        assert o["rs"].tolist() == ref["rs"].tolist()


@pytest.mark.parametrize("transport", ["nccl", "local"])
def test_split_self_transport(transport):
    """nranks = 1 with split_self: the slab-exchange path (plane counts, halo planes, gids,
    all-reduces) runs through the real transport -- NCCL self send/recv on one GPU, or the
    loopback -- and reproduces the plain single-rank run bitwise."""
    from paper_1704_03329_b200 import ljmd
    pos, box = li.fcc(6, 6, 7)
    pos = li.perturb(pos, 0.05)
    vel = li.velocities(len(pos), 1.44)
    ref = single(pos, vel, box, 30, list_order=0)
    nid = ljmd.nccl_unique_id() if transport == "nccl" else ljmd.local_group_id(uuid.uuid4().hex)
    with ljmd.LJMD(pos, vel, box, split_self=1, nccl_id=nid, list_order=0) as ctx:
        ctx.step(30)
        assert np.array_equal(ctx.positions(), ref["X"])
        assert np.array_equal(ctx.forces(), ref["F"])
        pe, ke = ctx.energy()
        assert pe == pytest.approx(ref["e"][0], rel=1e-13) and ke == pytest.approx(ref["e"][1], rel=1e-13)
