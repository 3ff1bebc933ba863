"""Common-neighbour analysis oracle (§8(f) NEXT-4) -- TEST INFRASTRUCTURE ONLY.

Follows Sec. 4.2 step by step, plain Python, for small systems:

  Alg. alg:cna_I: direct bonds  E_d(i) = {(G(i), G(j)) : |r_i - r_j| < rc}
  Alg. alg:cna_II: indirect bonds: for every bonded j, the direct bonds of j
                               that do not end at i
  Alg. alg:cna_III: for every bonded pair (i, j): common neighbours
                               C = {v : v = E(i)_{2k+1} = E(j)_{2l+1}}, common-neighbour bonds
                               E = {(v, w) in E(i) : v, w in C} as unordered pairs,
                               triplet (n_nb, n_b, n_lcb) = (|C|, |E|, maxClusterSize(E))
  Alg. alg:max_cluster_size: edges of the largest connected component,
                               breadth-first, removing visited edges.

Distances use the oracle's minimum-image displacement and canonical r^2 with a strict
cutoff (readings R4, R9).  Triplets of particle i are returned in ascending neighbour gid.
Pinned by tests/test_oracle_cna.py: the hcp signature 6 x (4,2,1) + 6 x (4,2,2),
fcc 12 x (4,2,1) and bcc 8 x (6,6,6) + 6 x (4,4,4) (Stukowski 2012 Tab. 1, the paper's
ref.), invariance under relabelling.
"""
from __future__ import annotations

import numpy as np

from . import neighbours


def max_cluster_size(edges):
    """Alg. alg:max_cluster_size: number of edges in the largest connected component."""
    E = set(edges)
    s_max = 0
    while E:
        s = 0
        v1, _ = next(iter(E))
        Q = {v1}
        while Q:
            v = Q.pop()
            P = {e for e in E if v in e}
            Q |= {w for e in P for w in e if w != v}
            s += len(P)
            E -= P
        s_max = max(s, s_max)
    return s_max


def cna(pos, box, rcut):
    """Returns {gid i: [(gid j, (n_nb, n_b, n_lcb)) for bonded j, ascending j]}."""
    pos = np.ascontiguousarray(pos, dtype=np.float64).reshape(-1, 3)
    off, nbr = neighbours(pos, box, rcut, "brute")        # pairs with r < rc
    n = pos.shape[0]
    G = np.arange(n)
    # Alg. alg:cna_I: direct bonds (G(i), G(j))
    E = {i: [(int(G[i]), int(G[j])) for j in nbr[off[i]:off[i + 1]]] for i in range(n)}
    n_nb = {i: len(E[i]) for i in range(n)}
    # Alg. alg:cna_II: indirect bonds from every bonded j (computed from the direct bonds)
    Ein = {}
    for i in range(n):
        ind = []
        for j in nbr[off[i]:off[i + 1]]:
            for k in range(n_nb[j]):
                if E[j][k][1] != G[i]:
                    ind.append(E[j][k])
        Ein[i] = E[i] + ind
    # Alg. alg:cna_III
    out = {}
    for i in range(n):
        trip = []
        for j in sorted(nbr[off[i]:off[i + 1]].tolist()):
            C = {E[i][k][1] for k in range(n_nb[i])} & {E[j][l][1] for l in range(n_nb[j])}
            bonds = set()
            for k in range(n_nb[i], len(Ein[i])):
                v, w = Ein[i][k]
                if v in C and w in C:
                    if w > v:
                        v, w = w, v
                    bonds.add((v, w))
            trip.append((j, (len(C), len(bonds), max_cluster_size(bonds))))
        out[i] = trip
    return out


def signature(trips):
    """Counts of triplets for one particle."""
    sig = {}
    for _, t in trips:
        sig[t] = sig.get(t, 0) + 1
    return sig
