"""Pins for the common-neighbour-analysis oracle (oracle/cna.py)."""
import numpy as np
import pytest

import ljinputs as li


def lattice(kind):
    if kind == "fcc":
        pos, box = li.fcc(3, 3, 3, rho=4.0 / np.sqrt(2.0) ** 3)   # nearest neighbour 1
        return pos, box, 1.2071                                     # (1 + sqrt 2) / 2
    if kind == "hcp":
        pos, box = li.hcp(4, 3, 3)
        return pos, box, 1.2071
    pos, box = li.bcc(4, 4, 4)
    return pos, box, 1.39     # between the 2nd (1.155) and 3rd (1.633) shells: 14 neighbours


EXPECT = {
    "fcc": {(4, 2, 1): 12},                      # Stukowski 2012 Tab. 1 (the paper's ref.)
    "hcp": {(4, 2, 1): 6, (4, 2, 2): 6},
    "bcc": {(6, 6, 6): 8, (4, 4, 4): 6},         # Stukowski 2012 Tab. 1
}


@pytest.mark.parametrize("kind", ["fcc", "hcp", "bcc"])
def test_lattice_signatures(kind):
    from oracle.cna import cna, signature
    pos, box, rc = lattice(kind)
    res = cna(pos, box, rc)
    for i in range(0, len(pos), 7):
        assert signature(res[i]) == EXPECT[kind], (kind, i, signature(res[i]))


def test_max_cluster_size():
    from oracle.cna import max_cluster_size
    assert max_cluster_size([]) == 0
    assert max_cluster_size([(1, 0), (3, 2)]) == 1                  # fcc-like: two separate bonds
    assert max_cluster_size([(1, 0), (2, 1), (5, 4)]) == 2          # hcp-like chain of two
    assert max_cluster_size([(1, 0), (2, 1), (3, 2), (3, 0), (9, 8)]) == 4   # a ring of four


def test_relabelling_invariance():
    """Triplets depend on geometry only: permuting particle order permutes the result."""
    from oracle.cna import cna
    pos, box, rc = lattice("hcp")
    pos = li.perturb(pos, 0.02)
    perm = np.random.default_rng(4).permutation(len(pos))
    a = cna(pos, box, rc)
    b = cna(pos[perm], box, rc)
    inv = np.argsort(perm)
    for i in range(0, len(pos), 11):
        ta = sorted(t for _, t in a[i])
        tb = sorted(t for _, t in b[int(inv[i])])
        assert ta == tb
