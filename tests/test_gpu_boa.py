"""GPU bond-order analysis (ljmd_boa, §8(f) NEXT-2) against the oracle (oracle/boa.py) and
Tab. tab:Q4Q6 of the paper."""
import numpy as np
import pytest

import ljinputs as li

pytestmark = pytest.mark.gpu

TAB = {"fcc": (0.191, 0.0, 0.575), "hcp": (0.097, 0.252, 0.485), "bcc": (0.036, 0.0, 0.511)}


def lattice(kind):
    if kind == "fcc":
        pos, box = li.fcc(4, 4, 4, rho=4.0 / np.sqrt(2.0) ** 3)
        return pos, box, 1.2
    if kind == "hcp":
        pos, box = li.hcp(6, 4, 4)
        return pos, box, 1.2
    pos, box = li.bcc(5, 5, 5)
    return pos, box, 1.4


@pytest.mark.parametrize("kind", ["fcc", "hcp", "bcc"])
def test_boa_lattices(kind):
    from oracle.boa import boa
    from paper_1704_03329_b200 import LJMD
    pos, box, rcut = lattice(kind)
    with LJMD(pos, np.zeros_like(pos), box, rc=1.5, delta=0.25) as ctx:
        for ell, ref in zip((4, 5, 6), TAB[kind]):
            Q, nnb = ctx.boa(ell, rcut)
            assert np.all(nnb == (14 if kind == "bcc" else 12))
            np.testing.assert_allclose(Q, ref, atol=5.5e-4)
            Qo, _ = boa(pos, box, ell, rcut)
            np.testing.assert_allclose(Q, Qo, rtol=1e-10, atol=1e-12)


@pytest.mark.parametrize("ell", [0, 1, 4, 6, 8, 12])
def test_boa_liquid_vs_oracle(ell):
    """Perturbed FCC at the benchmark density after 25 MD steps (one rebuild), rcut = rc."""
    from oracle.boa import boa
    from paper_1704_03329_b200 import LJMD
    pos, box = li.fcc(6, 6, 6)
    pos = li.perturb(pos, 0.05)
    vel = li.velocities(len(pos), 1.44)
    with LJMD(pos, vel, box) as ctx:
        ctx.step(25)
        x = ctx.positions()
        Q, nnb = ctx.boa(ell, li.RC)
    Qo, no = boa(x, box, ell, li.RC)
    assert np.array_equal(nnb, no)
    np.testing.assert_allclose(Q, Qo, rtol=1e-10, atol=1e-13)


def test_boa_errors():
    from paper_1704_03329_b200 import LJMD, LjmdError
    pos, box, _ = lattice("fcc")
    with LJMD(pos, np.zeros_like(pos), box, rc=1.5) as ctx:
        with pytest.raises(LjmdError, match="rcut"):
            ctx.boa(6, 1.6)
    with LJMD(pos, np.zeros_like(pos), box, rc=1.5) as ctx:
        with pytest.raises(LjmdError, match="ell"):
            ctx.boa(13, 1.2)
