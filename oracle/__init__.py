"""CPU oracle for the LJ PairLoop hot path of arXiv 1704.03329 -- TEST INFRASTRUCTURE.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
legs may import this package.  The product path (paper_1704_03329_b200) never
imports it and shares no code with it.

Thin ctypes wrapper over ljmd_oracle.c (plain fp64 C, -O2 -ffp-contract=off);
every arithmetic step lives in that file, with its PAPER.md citation.
Pins: tests/test_oracle_*.py (closed forms, golden fixtures, brute force).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "ljmd_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_LIB_OMP = os.path.join(_HERE, "liboracle_omp.so")   # same source, -fopenmp (all-core timing leg)
_lib = None
_lib_omp = None

_D = ctypes.POINTER(ctypes.c_double)
_I = ctypes.POINTER(ctypes.c_int64)


def build(force: bool = False) -> str:
    """Compile the oracle (gcc, -O2 -ffp-contract=off), plain and OpenMP.  Returns the
    plain .so path."""
    for lib, extra in ((_LIB, []), (_LIB_OMP, ["-fopenmp"])):
        if force or not os.path.exists(lib) or os.path.getmtime(lib) < os.path.getmtime(_SRC):
            tmp = lib + f".tmp{os.getpid()}"
            subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-std=c11",
                                   "-fPIC", "-shared", *extra, "-o", tmp, _SRC, "-lm"])
            os.replace(tmp, lib)
    return _LIB


class _LJ(ctypes.Structure):
    _fields_ = [("rc", ctypes.c_double), ("eps", ctypes.c_double),
                ("sigma", ctypes.c_double), ("shift", ctypes.c_double)]


class _Params(ctypes.Structure):
    _fields_ = [("lj", _LJ), ("dt", ctypes.c_double), ("mass", ctypes.c_double),
                ("delta", ctypes.c_double), ("ns", ctypes.c_int64), ("check", ctypes.c_int64),
                ("mode", ctypes.c_int64), ("energy_every", ctypes.c_int64),
                ("nu_dt", ctypes.c_double), ("temp", ctypes.c_double), ("seed", ctypes.c_uint64)]


def _load(omp: bool = False):
    global _lib, _lib_omp
    if omp and _lib_omp is not None:
        return _lib_omp
    if not omp and _lib is not None:
        return _lib
    if True:
        build()
        lib = ctypes.CDLL(_LIB_OMP if omp else _LIB)
        lib.orc_wrap.restype = ctypes.c_int64
        lib.orc_wrap.argtypes = [ctypes.c_int64, _D, _D]
        lib.orc_displacement.restype = None
        lib.orc_displacement.argtypes = [_D, _D, _D, _D]
        lib.orc_r2.restype = ctypes.c_double
        lib.orc_r2.argtypes = [_D]
        for f in (lib.orc_neigh_brute, lib.orc_neigh_cells):
            f.restype = ctypes.c_int64
            f.argtypes = [ctypes.c_int64, _D, _D, ctypes.c_double, _I, _I]
        lib.orc_cell_dims.restype = ctypes.c_int
        lib.orc_cell_dims.argtypes = [_D, ctypes.c_double, _I]
        lib.orc_forces.restype = ctypes.c_double
        lib.orc_forces.argtypes = [ctypes.c_int64, _D, _D, ctypes.POINTER(_LJ), _I, _I, _D, _D, _D, _D]
        lib.orc_sum.restype = ctypes.c_double
        lib.orc_sum.argtypes = [_D, ctypes.c_int64]
        lib.orc_kinetic.restype = ctypes.c_double
        lib.orc_kinetic.argtypes = [ctypes.c_int64, _D, ctypes.c_double]
        lib.orc_neigh_rows.restype = ctypes.c_int64
        lib.orc_neigh_rows.argtypes = [ctypes.c_int64, _D, _D, ctypes.c_double, _I, ctypes.c_int64, _I, _I]
        lib.orc_forces_rows.restype = None
        lib.orc_forces_rows.argtypes = [ctypes.c_int64, _D, _D, ctypes.POINTER(_LJ), _I, ctypes.c_int64,
                                        _D, _D, _D, _D]
        lib.orc_run.restype = ctypes.c_int64
        lib.orc_run.argtypes = [ctypes.c_int64, _D, _D, _D, ctypes.POINTER(_Params), ctypes.c_int64,
                                _D, _D, _D, _I, ctypes.c_int64, _I, _I]
        lib.orc_missed.restype = None
        lib.orc_missed.argtypes = [ctypes.c_int64, _D, _D, ctypes.c_double, _I, _I, _I, _I]
        lib.orc_threads.restype = ctypes.c_int
        lib.orc_threads.argtypes = [ctypes.c_int]
        U32 = ctypes.POINTER(ctypes.c_uint32)
        lib.orc_philox4x32.restype = None
        lib.orc_philox4x32.argtypes = [U32, U32, U32]
        lib.orc_andersen.restype = ctypes.c_int64
        lib.orc_andersen.argtypes = [ctypes.c_int64, _D, ctypes.c_uint64, ctypes.c_int64, ctypes.c_double,
                                     ctypes.c_double, ctypes.c_double]
        if omp:
            _lib_omp = lib
        else:
            _lib = lib
    return lib


def threads(k: int = 0) -> int:
    """Threads of the OpenMP build (k > 0 sets them); results do not depend on it."""
    return _load(omp=True).orc_threads(int(k))


def _dp(a):
    return a.ctypes.data_as(_D) if a is not None else None


def _ip(a):
    return a.ctypes.data_as(_I) if a is not None else None


def _f64(a, shape=None):
    a = np.ascontiguousarray(a, dtype=np.float64)
    if shape is not None:
        a = a.reshape(shape)
    return a


@dataclass
class LJ:
    rc: float = 2.5
    eps: float = 1.0
    sigma: float = 1.0
    shift: float = 0.25

    def c(self):
        return _LJ(self.rc, self.eps, self.sigma, self.shift)


def wrap(pos, box):
    """O1: returns wrapped copy; raises ValueError naming a non-finite particle."""
    p = _f64(pos, (-1, 3)).copy()
    b = _f64(box)
    bad = _load().orc_wrap(p.shape[0], _dp(p), _dp(b))
    if bad >= 0:
        raise ValueError(f"non-finite position at particle {bad}")
    return p


def displacement(xi, xj, box):
    d = np.zeros(3)
    _load().orc_displacement(_dp(_f64(xi)), _dp(_f64(xj)), _dp(_f64(box)), _dp(d))
    return d


def r2(d):
    return _load().orc_r2(_dp(_f64(d)))


def cell_dims(box, rn):
    nc = np.zeros(3, dtype=np.int64)
    if _load().orc_cell_dims(_dp(_f64(box)), float(rn), _ip(nc)) != 0:
        raise ValueError("box too small: fewer than 3 cells of width >= rbar_c")
    return nc


def neighbours(pos, box, rn, method="brute", omp=False):
    """O3 (brute) / O4 (cells): CSR (offsets[n+1], nbr[...]) with each NB(i) ascending.
    omp: the OpenMP build of the same source (rows in parallel, identical results)."""
    p = _f64(pos, (-1, 3))
    b = _f64(box)
    n = p.shape[0]
    off = np.zeros(n + 1, dtype=np.int64)
    f = _load(omp).orc_neigh_brute if method == "brute" else _load(omp).orc_neigh_cells
    tot = f(n, _dp(p), _dp(b), float(rn), _ip(off), None)
    if tot < 0:
        raise ValueError("box too small: fewer than 3 cells of width >= rbar_c")
    nbr = np.zeros(max(tot, 1), dtype=np.int64)
    f(n, _dp(p), _dp(b), float(rn), _ip(off), _ip(nbr))
    return off, nbr[:tot]


@dataclass
class Forces:
    F: np.ndarray
    e: np.ndarray
    S: np.ndarray
    A: np.ndarray
    pe: float


def forces(pos, box, lj: LJ = LJ(), nlist=None, omp=False):
    """O5: per-particle forces, energies e_i = 1/2 sum_j V, tolerance scales S_i, A_i.
    omp: the OpenMP build of the same source (rows in parallel, identical results)."""
    p = _f64(pos, (-1, 3))
    b = _f64(box)
    n = p.shape[0]
    F = np.zeros((n, 3))
    e = np.zeros(n)
    S = np.zeros(n)
    A = np.zeros(n)
    c = lj.c()
    off, nbr = (None, None) if nlist is None else (np.ascontiguousarray(nlist[0], dtype=np.int64),
                                                   np.ascontiguousarray(nlist[1], dtype=np.int64))
    pe = _load(omp).orc_forces(n, _dp(p), _dp(b), ctypes.byref(c), _ip(off), _ip(nbr),
                            _dp(F), _dp(e), _dp(S), _dp(A))
    return Forces(F, e, S, A, pe)


def neighbours_rows(pos, box, rn, rows):
    """O3 restricted to rows (sampled checks at full size): CSR over the given rows."""
    p = _f64(pos, (-1, 3))
    b = _f64(box)
    idx = np.ascontiguousarray(rows, dtype=np.int64)
    off = np.zeros(idx.shape[0] + 1, dtype=np.int64)
    lib = _load()
    tot = lib.orc_neigh_rows(p.shape[0], _dp(p), _dp(b), float(rn), _ip(idx), idx.shape[0], _ip(off), None)
    nbr = np.zeros(max(tot, 1), dtype=np.int64)
    lib.orc_neigh_rows(p.shape[0], _dp(p), _dp(b), float(rn), _ip(idx), idx.shape[0], _ip(off), _ip(nbr))
    return off, nbr[:tot]


def forces_rows(pos, box, rows, lj: LJ = LJ()):
    """O5 brute force restricted to rows: Forces over the given rows (pe = sum of their e_i)."""
    p = _f64(pos, (-1, 3))
    b = _f64(box)
    idx = np.ascontiguousarray(rows, dtype=np.int64)
    m = idx.shape[0]
    F, e, S, A = np.zeros((m, 3)), np.zeros(m), np.zeros(m), np.zeros(m)
    c = lj.c()
    _load().orc_forces_rows(p.shape[0], _dp(p), _dp(b), ctypes.byref(c), _ip(idx), m,
                            _dp(F), _dp(e), _dp(S), _dp(A))
    return Forces(F, e, S, A, float(e.sum()))


def philox4x32(ctr, key):
    """O8: Philox4x32-10 block (4 x uint32 counter, 2 x uint32 key) -> 4 x uint32."""
    c = np.ascontiguousarray(ctr, dtype=np.uint32)
    k = np.ascontiguousarray(key, dtype=np.uint32)
    o = np.zeros(4, dtype=np.uint32)
    U32 = ctypes.POINTER(ctypes.c_uint32)
    _load().orc_philox4x32(c.ctypes.data_as(U32), k.ctypes.data_as(U32), o.ctypes.data_as(U32))
    return o


def andersen(vel, seed, step, nu_dt, temp, mass=1.0):
    """O8: one Andersen pass (reading R19) on a copy of vel; returns (vel', n_resampled)."""
    v = _f64(vel, (-1, 3)).copy()
    k = _load().orc_andersen(v.shape[0], _dp(v), seed, step, nu_dt, temp, mass)
    return v, int(k)


def neumaier_sum(x):
    x = _f64(x).ravel()
    return _load().orc_sum(_dp(x), x.shape[0])


def kinetic(vel, mass=1.0):
    v = _f64(vel, (-1, 3))
    return _load().orc_kinetic(v.shape[0], _dp(v), float(mass))


@dataclass
class Run:
    pos: np.ndarray
    vel: np.ndarray
    F: np.ndarray
    pe: np.ndarray
    ke: np.ndarray
    rebuild_steps: np.ndarray
    missed_particles: np.ndarray = None   # validate: per step (index = step; 0 = init)
    missed_pairs: np.ndarray = None


def missed(pos, box, rc, nlist):
    """Missed pairs of the list nlist = (offsets, nbr) at positions pos: (particles with at
    least one pair r < rc not in their list, such ordered pairs), brute force."""
    p = _f64(pos, (-1, 3))
    off = np.ascontiguousarray(nlist[0], dtype=np.int64)
    nb = np.ascontiguousarray(nlist[1], dtype=np.int64)
    a, b = ctypes.c_int64(), ctypes.c_int64()
    _load().orc_missed(p.shape[0], _dp(p), _dp(_f64(box)), float(rc), _ip(off), _ip(nb), ctypes.byref(a),
                       ctypes.byref(b))
    return a.value, b.value


def run(pos, vel, box, nsteps, lj: LJ = LJ(), dt=0.005, mass=1.0, delta=0.25, ns=20,
        check=0, mode="list", energy_every=10, thermostat=None, validate=False, omp=False):
    """O6/O7: velocity-Verlet trajectory with the paper's rebuild schedule.
    thermostat = (nu, T, seed): O8 Andersen collisions after every step.
    validate: missed pairs of the list at every step (orc_missed; list mode).
    omp: the OpenMP build of the same source (identical results; bench timing leg)."""
    p = _f64(pos, (-1, 3)).copy()
    v = _f64(vel, (-1, 3)).copy()
    b = _f64(box)
    n = p.shape[0]
    F = np.zeros((n, 3))
    ns_samp = (nsteps // energy_every if energy_every > 0 else 0) + 1
    pe = np.zeros(ns_samp)
    ke = np.zeros(ns_samp)
    cap = nsteps + 1
    rs = np.zeros(cap, dtype=np.int64)
    nu, temp, seed = thermostat if thermostat is not None else (0.0, 0.0, 0)
    if nu * dt > 1.0 or nu < 0.0 or temp < 0.0:
        raise ValueError("Andersen thermostat needs 0 <= nu*dt <= 1 and T >= 0")
    prm = _Params(lj.c(), dt, mass, delta, ns, check, 1 if mode == "list" else 0, energy_every,
                  nu * dt, temp, seed)
    mp = np.zeros(nsteps + 1, dtype=np.int64) if validate else None
    mq = np.zeros(nsteps + 1, dtype=np.int64) if validate else None
    nreb = _load(omp).orc_run(n, _dp(p), _dp(v), _dp(b), ctypes.byref(prm), nsteps,
                              _dp(F), _dp(pe), _dp(ke), _ip(rs), cap, _ip(mp), _ip(mq))
    if nreb < 0:
        raise ValueError("box too small: fewer than 3 cells of width >= rbar_c")
    return Run(p, v, F, pe, ke, rs[:nreb], mp, mq)
