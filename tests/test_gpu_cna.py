"""GPU common-neighbour analysis (ljmd_cna, §8(f) NEXT-4) against the oracle (oracle/cna.py,
Algs. alg:cna_I-III, alg:max_cluster_size) and the lattice signatures."""
import numpy as np
import pytest

import ljinputs as li

pytestmark = pytest.mark.gpu

EXPECT = {
    "fcc": {(4, 2, 1): 12},
    "hcp": {(4, 2, 1): 6, (4, 2, 2): 6},
    "bcc": {(6, 6, 6): 8, (4, 4, 4): 6},
}
CLASS = {"fcc": 1, "hcp": 2, "bcc": 3}


def lattice(kind):
    if kind == "fcc":
        pos, box = li.fcc(4, 4, 4, rho=4.0 / np.sqrt(2.0) ** 3)
        return pos, box, 1.2071
    if kind == "hcp":
        pos, box = li.hcp(6, 4, 4)
        return pos, box, 1.2071
    pos, box = li.bcc(5, 5, 5)
    return pos, box, 1.39


def oracle_arrays(pos, box, rcut):
    from oracle.cna import cna
    res = cna(pos, box, rcut)
    n = len(pos)
    nnb = np.zeros(n, dtype=np.int64)
    tr = np.zeros((n, 24, 3), dtype=np.int32)
    for i in range(n):
        nnb[i] = len(res[i])
        for k, (_, t) in enumerate(res[i]):
            tr[i, k] = t
    return nnb, tr


def classify(nnb, tr):
    """Class from the triplets (Stukowski 2012 Tab. 1 signatures), for the oracle side."""
    out = np.zeros(len(nnb), dtype=np.int32)
    for i in range(len(nnb)):
        sig = {}
        for t in map(tuple, tr[i, :nnb[i]]):
            sig[t] = sig.get(t, 0) + 1
        for kind, ref in EXPECT.items():
            if sig == ref:
                out[i] = CLASS[kind]
    return out


@pytest.mark.parametrize("kind", ["fcc", "hcp", "bcc"])
def test_cna_lattices(kind):
    from paper_1704_03329_b200 import LJMD
    pos, box, rcut = lattice(kind)
    with LJMD(pos, np.zeros_like(pos), box, rc=1.5, delta=0.25) as ctx:
        cls, nnb, tr = ctx.cna(rcut, triplets=True)
    assert np.all(cls == CLASS[kind])
    on, otr = oracle_arrays(pos, box, rcut)
    assert np.array_equal(nnb, on)
    assert np.array_equal(tr, otr)


@pytest.mark.parametrize("sigma_d,rcut", [(0.03, 1.2071), (0.08, 1.2071), (0.12, 1.3)])
def test_cna_perturbed_crystal(sigma_d, rcut):
    """Thermally disordered fcc: a mix of fcc and 'other' particles, triplets exact vs oracle."""
    from paper_1704_03329_b200 import LJMD
    pos, box = li.fcc(4, 4, 4, rho=4.0 / np.sqrt(2.0) ** 3)
    pos = li.perturb(pos, sigma_d)
    with LJMD(pos, np.zeros_like(pos), box, rc=1.5, delta=0.25) as ctx:
        x = ctx.positions()
        cls, nnb, tr = ctx.cna(rcut, triplets=True)
    on, otr = oracle_arrays(x, box, rcut)
    assert np.array_equal(nnb, on)
    assert np.array_equal(tr, otr)
    assert np.array_equal(cls, classify(on, otr))


def test_cna_liquid_after_md():
    """LJ liquid at the benchmark density after 25 MD steps (one rebuild), rcut = 1.5 sigma
    (first minimum of g(r)); bonded neighbours taken from the engine's Verlet list."""
    from paper_1704_03329_b200 import LJMD
    pos, box = li.fcc(5, 5, 5)
    pos = li.perturb(pos, 0.05)
    vel = li.velocities(len(pos), 1.44)
    with LJMD(pos, vel, box) as ctx:
        ctx.step(25)
        x = ctx.positions()
        cls, nnb, tr = ctx.cna(1.5, triplets=True)
    on, otr = oracle_arrays(x, box, 1.5)
    assert np.array_equal(nnb, on)
    assert np.array_equal(tr, otr)
    assert np.array_equal(cls, classify(on, otr))


def test_cna_large_fcc_all_fcc():
    """At the benchmark size every particle of the ideal crystal is fcc (property check)."""
    from paper_1704_03329_b200 import LJMD
    pos, box = li.fcc(32, 32, 32)
    a = li.fcc_lattice_constant()
    rcut = a * (1.0 / np.sqrt(2.0) + 1.0) / 2.0
    with LJMD(pos, np.zeros_like(pos), box) as ctx:
        cls, nnb = ctx.cna(rcut)
    assert np.all(nnb == 12) and np.all(cls == 1)


def test_cna_errors():
    from paper_1704_03329_b200 import LJMD, LjmdError
    pos, box, _ = lattice("fcc")
    with LJMD(pos, np.zeros_like(pos), box, rc=1.5) as ctx:
        with pytest.raises(LjmdError, match="rcut"):
            ctx.cna(1.6)
    # more than 24 bonds: a dense cluster with rcut = rc
    pos, box = li.fcc(5, 5, 5, rho=3.0)   # 12 + 6 + 24 neighbours inside 1.5
    with LJMD(pos, np.zeros_like(pos), box, rc=1.5, delta=0.25) as ctx:
        with pytest.raises(LjmdError, match="bonded"):
            ctx.cna(1.5)
