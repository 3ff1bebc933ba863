"""Bond-order analysis oracle (§8(f) NEXT-2) -- TEST INFRASTRUCTURE ONLY.

Steinhardt order parameters exactly as Sec. 4.1 defines them:
  q_lm(i) = (1/|N(i)|) sum_{j in N(i)} Y_l^m(r_hat_ij),  r_hat_ij = (r_i - r_j)/|r_i - r_j|
                                                          (Eq. eqn:qellm)
  Q_l(i)  = sqrt( 4 pi / (2l + 1) sum_{m=-l..l} |q_lm(i)|^2 )   (Eq. eqn:Qell)
with N(i) = { j != i : |r_i - r_j| < rcut } (minimum image, the oracle's O2 displacement and
strict cutoff, readings R4/R9), computed in the order of Algorithms alg:sph_I (pair loop)
and alg:sph_II (particle loop).  Y_l^m is scipy.special.sph_harm_y (a library primitive
used as a step, fp64); |N(i)| = 0 gives Q_l = 0.

Pinned by tests/test_oracle_boa.py: Tab. tab:Q4Q6 for perfect fcc, hcp
and bcc; the addition theorem (one neighbour -> Q_l = 1); Q_odd = 0 for centrosymmetric
environments.
"""
from __future__ import annotations

import numpy as np
from scipy.special import sph_harm_y

from . import displacement, neighbours


def boa(pos, box, ell: int, rcut: float):
    """Returns (Q_l[n], |N(i)|[n])."""
    pos = np.ascontiguousarray(pos, dtype=np.float64).reshape(-1, 3)
    box = np.asarray(box, dtype=np.float64)
    n = pos.shape[0]
    off, nbr = neighbours(pos, box, rcut, "brute")
    Q = np.zeros(n)
    nnb = np.diff(off)
    for i in range(n):                                   # Algorithm alg:sph_I: pairs (i, j)
        if nnb[i] == 0:
            continue
        d = np.array([displacement(pos[i], pos[j], box) for j in nbr[off[i]:off[i + 1]]])
        r = np.sqrt(np.sum(d * d, axis=1))
        u = d / r[:, None]                               # r_hat_ij
        theta = np.arccos(np.clip(u[:, 2], -1.0, 1.0))
        phi = np.arctan2(u[:, 1], u[:, 0])
        acc = 0.0
        for m in range(-ell, ell + 1):
            q = np.sum(sph_harm_y(ell, m, theta, phi)) / nnb[i]   # q_lm, Eq. eqn:qellm
            acc += abs(q) ** 2
        Q[i] = np.sqrt(4.0 * np.pi / (2 * ell + 1) * acc)         # Algorithm alg:sph_II
    return Q, nnb
