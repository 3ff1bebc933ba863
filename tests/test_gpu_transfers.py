"""Overlapped host transfers (ljmd_stage_state, ljmd_set_state(NULL, NULL),
ljmd_get_positions_async, ljmd_wait_transfers): a staged state gives bitwise the same
trajectory as the synchronous ljmd_set_state, queued states are consumed in order, and
the asynchronous positions equal ljmd_get_positions; forces still match the oracle."""
import numpy as np
import pytest

import ljinputs as li

pytestmark = pytest.mark.gpu


def pinned(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).pin_memory()


@pytest.fixture(scope="module")
def states():
    pos, box = li.fcc(6, 6, 6)
    vel = li.velocities(len(pos), 1.44)
    return [(li.perturb(pos, s), vel * (1 + 0.1 * k), box) for k, s in enumerate((0.02, 0.05, 0.08))]


def run_sync(st, steps):
    from paper_1704_03329_b200 import LJMD
    pos, vel, box = st
    with LJMD(pos, vel, box, rc=li.RC, dt=li.DT, device=0) as ctx:
        ctx.step(steps)
        return ctx.positions(), ctx.velocities(), ctx.forces(), ctx.energy()


def test_staged_equals_synchronous(states, orc):
    from paper_1704_03329_b200 import LJMD
    import torch
    pos0, vel0, box = states[0]
    hp = [pinned(s[0]) for s in states]
    hv = [pinned(s[1]) for s in states]
    ho = [torch.zeros((len(pos0), 3), dtype=torch.float64).pin_memory() for _ in states]
    ref = [run_sync(s, 25) for s in states]
    with LJMD(pos0, vel0, box, rc=li.RC, dt=li.DT, device=0) as ctx:
        ctx.stage_state_ptr(hp[0].data_ptr(), hv[0].data_ptr())
        ctx.stage_state_ptr(hp[1].data_ptr(), hv[1].data_ptr())   # two queued ahead
        for k in range(len(states)):
            ctx.set_staged_state()
            if k + 2 < len(states):
                ctx.stage_state_ptr(hp[k + 2].data_ptr(), hv[k + 2].data_ptr())
            ctx.step(25)
            ctx.positions_async_ptr(ho[k].data_ptr())
            x, v, F, (pe, ke) = ref[k]
            assert np.array_equal(ctx.velocities(), v)
            assert np.array_equal(ctx.forces(), F)
            assert ctx.energy() == (pe, ke)
        ctx.wait_transfers()
        for k in range(len(states)):
            assert np.array_equal(ho[k].numpy(), ref[k][0]), f"state {k}"
        # forces at the final positions against the oracle's brute force
        xw = orc.wrap(ho[-1].numpy(), box)
        r = orc.forces(xw, box, orc.LJ(rc=li.RC, shift=0.25))
        assert np.all(np.abs(ref[-1][2] - r.F) <= 1e-10 * r.S[:, None])


def test_staged_errors(states):
    from paper_1704_03329_b200 import LJMD, ljmd
    pos0, vel0, box = states[0]
    hp, hv = pinned(pos0), pinned(vel0)
    with LJMD(pos0, vel0, box, rc=li.RC, dt=li.DT, device=0) as ctx:
        with pytest.raises(ljmd.LjmdError, match="no staged state"):
            ctx.set_staged_state()
    with LJMD(pos0, vel0, box, rc=li.RC, dt=li.DT, device=0) as ctx:
        ctx.stage_state_ptr(hp.data_ptr(), hv.data_ptr())
        ctx.stage_state_ptr(hp.data_ptr(), hv.data_ptr())
        with pytest.raises(ljmd.LjmdError, match="already queued"):
            ctx.stage_state_ptr(hp.data_ptr(), hv.data_ptr())


def test_staged_needs_single_rank(states):
    from paper_1704_03329_b200 import LJMD, ljmd
    pos0, vel0, box = states[0]
    hp, hv = pinned(pos0), pinned(vel0)
    import uuid
    with LJMD(pos0, vel0, box, rc=li.RC, dt=li.DT, device=0, split_self=1,
              nccl_id=ljmd.local_group_id(uuid.uuid4().hex)) as ctx:
        with pytest.raises(ljmd.LjmdError, match="single rank"):
            ctx.stage_state_ptr(hp.data_ptr(), hv.data_ptr())


def test_set_profile(states):
    """ljmd_set_profile switches the per-launch force timing on and off between steps."""
    from paper_1704_03329_b200 import LJMD, ljmd
    pos0, vel0, box = states[0]
    with LJMD(pos0, vel0, box, rc=li.RC, dt=li.DT, device=0) as ctx:
        ctx.step(5)
        s0 = ctx.stats()
        assert s0["force_launches"] == 0 and s0["force_ms"] == 0.0
        ctx.set_profile(True)
        ctx.step(5)
        s1 = ctx.stats()
        assert s1["force_launches"] == 5 and s1["force_ms"] > 0.0
        ctx.set_profile(False)
        ctx.step(5)
        assert ctx.stats()["force_launches"] == 5
        assert ctx._lib.ljmd_set_profile(ctx._h, 2) == -1    # LJMD_E_ARG
