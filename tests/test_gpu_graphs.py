"""GPU: ljmd_step as a captured CUDA graph (device-side rebuild decision and capacity checks,
DESIGN.md §10) against the eager path, which takes the same decisions on the host: the
same kernels in the same order on the same data, so the trajectories agree bit for bit."""
import numpy as np
import pytest

import ljinputs as li
from conftest import cuda_available

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_available(), reason="needs a CUDA device")]


@pytest.fixture(scope="module")
def eng():
    from paper_1704_03329_b200 import ljmd
    ljmd.load()
    return ljmd


def state(cells=8, sigma_d=0.05, t0=1.44):
    pos, box = li.fcc(cells, cells, cells)
    return li.perturb(pos, sigma_d), li.velocities(len(pos), t0), box


def run(eng, pos, vel, box, calls, **kw):
    with eng.LJMD(pos, vel, box, **kw) as ctx:
        for n in calls:
            ctx.step(n)
        out = dict(x=ctx.positions(), v=ctx.velocities(), F=ctx.forces(), e=ctx.energy_history(),
                   reb=ctx.rebuild_steps(), st=ctx.stats())
    return out


def same(a, b):
    assert np.array_equal(a["x"], b["x"]) and np.array_equal(a["v"], b["v"]) and np.array_equal(a["F"], b["F"])
    assert np.array_equal(a["e"][0], b["e"][0]) and np.array_equal(a["e"][1], b["e"][1])
    assert a["reb"].tolist() == b["reb"].tolist()


@pytest.mark.parametrize("check", [0, 1])
def test_graph_equals_eager(eng, check):
    """Both rebuild policies, calls of several lengths (graphs captured per shape and
    replayed): positions, velocities, forces, the energy history and the rebuild steps are
    bitwise those of the eager path."""
    pos, vel, box = state()
    calls = [20, 20, 7, 13, 20, 1, 19]
    g = run(eng, pos, vel, box, calls, rebuild_check=check, graphs=1)
    e = run(eng, pos, vel, box, calls, rebuild_check=check, graphs=0)
    same(g, e)
    assert g["st"]["graph_calls"] == len(calls) and e["st"]["graph_calls"] == 0
    assert g["st"]["dangerous_builds"] == e["st"]["dangerous_builds"]
    assert len(g["reb"]) >= (2 if check == 0 else 4)


def test_graph_capacity_abort_resumes(eng):
    """Capacities shrunk to the initial state's needs (tight_caps): the first rebuild inside
    a captured sequence that needs more (slots, staging or list width) aborts on the device;
    the host resumes eagerly at that step with regrown buffers.  The trajectory is the eager
    one bit for bit."""
    pos, vel, box = state(sigma_d=0.0, t0=2.0)   # perfect FCC melting: the layout grows
    calls = [20, 20, 20]
    g = run(eng, pos, vel, box, calls, graphs=1, tight_caps=1)
    e = run(eng, pos, vel, box, calls, graphs=0)
    same(g, e)
    assert g["st"]["graph_aborts"] >= 1 and g["st"]["regrows"] >= 1


def test_graph_parity_with_oracle(eng, orc):
    """A 40-step graph-mode run (two captured calls, one rebuild each) against the oracle's
    trajectory with the same schedule: energies within the 100-step bar."""
    pos, vel, box = state(cells=10)
    with eng.LJMD(pos, vel, box, graphs=1) as ctx:
        ctx.step(20)
        ctx.step(20)
        pe, ke = ctx.energy_history()
        assert ctx.stats()["graph_calls"] == 2
    r = orc.run(pos, vel, box, 40)
    np.testing.assert_allclose(pe, r.pe, rtol=1e-8)
    np.testing.assert_allclose(ke, r.ke, rtol=1e-8)


@pytest.mark.parametrize("check,cells", [(0, 8), (1, 8), (1, 32)])
def test_deferred_settlement_equals_synchronous(eng, monkeypatch, check, cells):
    """Graph calls return once queued; the host settles a call after queueing the next one
    (or at the next getter).  Against LJMD_DEFER=0 (one host wait per call) and the eager
    path: the same trajectory, energies and rebuild steps bit for bit, with getters
    interleaved between the calls -- under both rebuild policies; 32^3 cells is large enough
    for one force CTA per tile, where the displacement-checked policy's list order (bank-aware
    or build order, from the rebuild intervals two calls back) changes between calls."""
    pos, vel, box = state(cells=cells)
    calls = [20, 20, 20, 3, 17, 20, 40, 1] if cells == 8 else [20, 20, 20, 7, 13, 20]

    def run_mixed(**kw):
        kw["rebuild_check"] = check
        hist = []
        with eng.LJMD(pos, vel, box, **kw) as ctx:
            for k, n in enumerate(calls):
                ctx.step(n)
                if k % 3 == 2:
                    hist.append(ctx.energy())
                    hist.append(ctx.stats()["steps_done"])
            out = dict(x=ctx.positions(), v=ctx.velocities(), F=ctx.forces(), e=ctx.energy_history(),
                       reb=ctx.rebuild_steps(), st=ctx.stats())
        return out, hist

    monkeypatch.setenv("LJMD_DEFER", "0")
    s, hs = run_mixed(graphs=1)
    e, he = run_mixed(graphs=0)
    monkeypatch.setenv("LJMD_DEFER", "1")
    d, hd = run_mixed(graphs=1)
    same(d, s)
    same(d, e)
    assert hd == hs == he
    assert d["st"]["steps_done"] == sum(calls) and d["st"]["graph_calls"] == len(calls)


def test_deferred_abort_with_queued_calls(eng):
    """A capacity abort in a call that already has the next one queued behind it: the queued
    call runs as no-ops on the device (k_call_begin keeps the abort record), the host resumes
    the aborted call eagerly and re-runs the queued one -- the eager trajectory bit for bit."""
    pos, vel, box = state(sigma_d=0.0, t0=2.0)
    calls = [20, 20, 20, 20]
    g = run(eng, pos, vel, box, calls, graphs=1, tight_caps=1)
    e = run(eng, pos, vel, box, calls, graphs=0)
    same(g, e)
    assert g["st"]["graph_aborts"] >= 1 and g["st"]["steps_done"] == sum(calls)


def test_list_order_change_between_calls(eng):
    """Under the displacement check the bank-aware list order is chosen per call from the
    rebuild intervals (two calls back): a hot melt (rebuilds every few steps: build order)
    followed by a cold state of the same particles (long intervals: bank-aware order) changes
    the choice between calls without a rebuild in between.  Every force launch must read the
    last build's list (the pass re-sequences it in place): graph (deferred) and eager runs agree
    bit for bit and the energies stay finite."""
    pos, vel, box = state(cells=32, sigma_d=0.05, t0=1.44)
    cold = li.velocities(len(pos), 0.05)

    def run(**kw):
        with eng.LJMD(pos, vel, box, rebuild_check=1, **kw) as ctx:
            for _ in range(3):
                ctx.step(20)
            ctx.set_state(ctx.positions(), cold)
            for _ in range(6):
                ctx.step(20)
            return dict(x=ctx.positions(), v=ctx.velocities(), F=ctx.forces(), e=ctx.energy_history(),
                        reb=ctx.rebuild_steps(), st=ctx.stats())

    g = run(graphs=1)
    e = run(graphs=0)
    same(g, e)
    assert np.isfinite(g["e"][0]).all() and np.isfinite(g["e"][1]).all()
    assert np.isfinite(g["F"]).all()


def test_speculative_eager_rebuild(eng, monkeypatch):
    """The eager rebuild runs the captured rebuild's kernels with device-side capacity checks
    and one host wait; a shortfall (tight_caps) falls back to the host-checked sequence, which
    regrows it.  Bitwise the host-checked rebuild's trajectory (LJMD_SPEC_REBUILD=0)."""
    pos, vel, box = state(sigma_d=0.0, t0=2.0)   # perfect FCC melting: the layout grows
    calls = [20, 20, 20]
    s = run(eng, pos, vel, box, calls, graphs=0, tight_caps=1)
    monkeypatch.setenv("LJMD_SPEC_REBUILD", "0")
    h = run(eng, pos, vel, box, calls, graphs=0, tight_caps=1)
    same(s, h)
    assert s["st"]["regrows"] >= 1
