"""PairLoop / ParticleLoop front end -- the paper's embedded DSL (Sec. 2.2-2.4)
on the B200 engine.  Argument marshalling only: the kernels are compiled by libljmd.so
(NVRTC, sm_100a) and run on the device; there is no Python or CPU execution path.

Classes follow Tabs. tab:DSL_data / tab:DSL_looping / tab:DSL_access:

    state = LJMD(pos, vel, box)                        # the State: positions, velocities, lists
    a = ParticleDat(state, ncomp=3)                    # per-particle data, caller order
    S = ScalarArray(state, ncomp=1)                    # global data
    k = Kernel("update_b", code, (Constant("dimension", 3),))
    loop = PairLoop(k, {"r": state_positions(state)(READ), "a": a(READ), "b": b(INC),
                        "S": S(INC)}, shell_cutoff=1.5)
    loop.execute()

A PairLoop visits every ordered pair with |r_i - r_j| < shell_cutoff <= rc (reading R20),
through the engine's neighbour list.  Single rank.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from typing import Dict, Sequence, Tuple

import numpy as np

from .ljmd import LJMD, _I

READ, WRITE, RW, INC, INC_ZERO = 0, 1, 2, 3, 4


class access:  # noqa: N801  (the paper's spelling: access.READ, ...)
    READ, WRITE, RW, INC, INC_ZERO = READ, WRITE, RW, INC, INC_ZERO


_DTYPES = {np.dtype(np.float64): 0, np.dtype(np.int32): 1, np.dtype(np.int64): 2}
_NP = {0: np.float64, 1: np.int32, 2: np.int64}


@dataclass(frozen=True)
class Constant:
    """Numerical constant substituted into the kernel source (Tab. tab:DSL_data)."""
    label: str
    value: float

    def define(self) -> str:
        v = self.value
        if isinstance(v, (bool, np.bool_)):
            v = int(v)
        if isinstance(v, (int, np.integer)):
            return f"{self.label}={int(v)}"
        return f"{self.label}={float(v)!r}"


@dataclass
class Kernel:
    label: str
    code: str
    constants: Sequence[Constant] = field(default_factory=tuple)


class _Bindable:
    handle: int
    state: LJMD

    def __call__(self, acc: int) -> Tuple["_Bindable", int]:
        return (self, int(acc))


class ParticleDat(_Bindable):
    """ncomp values of dtype per particle, owned by the engine context (device memory)."""

    def __init__(self, state: LJMD, ncomp: int = 1, dtype=np.float64, initial_value=0, npart=None,
                 _global: bool = False):
        self.state = state
        self.ncomp = int(ncomp)
        self.dtype = np.dtype(dtype)
        if self.dtype not in _DTYPES:
            raise TypeError(f"dtype {self.dtype} not supported (float64, int32, int64)")
        self._global = _global
        if npart is not None and not _global and int(npart) != state.n:
            raise ValueError("npart must equal the number of particles of the state")
        h = ctypes.c_int64()
        state._ck(state._lib.ljmd_dat_create(state._h, self.ncomp, _DTYPES[self.dtype], 1 if _global else 0,
                                             ctypes.byref(h)))
        self.handle = h.value
        if initial_value:
            self.data = np.full(self.shape, initial_value, dtype=self.dtype)

    @property
    def shape(self):
        return (self.ncomp,) if self._global else (self.state.n, self.ncomp)

    @property
    def data(self) -> np.ndarray:
        out = np.zeros(self.shape, dtype=self.dtype)
        self.state._ck(self.state._lib.ljmd_dat_get(self.state._h, self.handle, out.ctypes.data_as(ctypes.c_void_p)))
        return out

    @data.setter
    def data(self, values):
        a = np.ascontiguousarray(np.broadcast_to(np.asarray(values, dtype=self.dtype), self.shape))
        self.state._ck(self.state._lib.ljmd_dat_set(self.state._h, self.handle, a.ctypes.data_as(ctypes.c_void_p)))

    def free(self):
        if self.state._h is not None and self.handle >= 0:
            self.state._ck(self.state._lib.ljmd_dat_free(self.state._h, self.handle))
            self.handle = -100


class ScalarArray(ParticleDat):
    """Global property with ncomp components (Tab. tab:DSL_data)."""

    def __init__(self, state: LJMD, ncomp: int = 1, dtype=np.float64, initial_value=0):
        super().__init__(state, ncomp, dtype, initial_value, _global=True)


class EngineDat(_Bindable):
    """Engine-owned particle data: positions (the PositionDat), velocities, forces, gids,
    per-particle energies."""

    def __init__(self, state: LJMD, handle: int):
        self.state = state
        self.handle = handle


def PositionDat(state: LJMD) -> EngineDat:  # noqa: N802
    return EngineDat(state, -1)


def velocities(state: LJMD) -> EngineDat:
    return EngineDat(state, -2)


def forces(state: LJMD) -> EngineDat:
    return EngineDat(state, -3)


def global_ids(state: LJMD) -> EngineDat:
    return EngineDat(state, -4)


def particle_energies(state: LJMD) -> EngineDat:
    return EngineDat(state, -5)


class _Loop:
    _kind = 0

    def __init__(self, kernel: Kernel, dat_dict: Dict[str, Tuple[_Bindable, int]], shell_cutoff: float = 0.0,
                 fmad: bool = False):
        if not dat_dict:
            raise ValueError("a loop needs at least one dat")
        states = {id(d.state) for d, _ in dat_dict.values()}
        if len(states) != 1:
            raise ValueError("all dats of a loop must belong to one state")
        self.state = next(iter(dat_dict.values()))[0].state
        self.kernel = kernel
        labels = list(dat_dict)
        n = len(labels)
        c_labels = (ctypes.c_char_p * n)(*[lb.encode() for lb in labels])
        handles = np.array([dat_dict[lb][0].handle for lb in labels], dtype=np.int64)
        acc = np.array([dat_dict[lb][1] for lb in labels], dtype=np.int64)
        consts = "\n".join(c.define() for c in kernel.constants).encode()
        h = ctypes.c_int64()
        st = self.state
        st._ck(st._lib.ljmd_loop_create(st._h, self._kind, kernel.label.encode(), kernel.code.encode(), consts,
                                        float(shell_cutoff), n, c_labels, handles.ctypes.data_as(_I),
                                        acc.ctypes.data_as(_I), 1 if fmad else 0, ctypes.byref(h)))
        self.handle = h.value
        self._keep = (c_labels, handles, acc)

    def execute(self):
        self.state._ck(self.state._lib.ljmd_loop_execute(self.state._h, self.handle))

    @property
    def source(self) -> str:
        st = self.state
        n = ctypes.c_int64()
        st._ck(st._lib.ljmd_loop_source(st._h, self.handle, None, 0, ctypes.byref(n)))
        buf = ctypes.create_string_buffer(n.value + 1)
        st._ck(st._lib.ljmd_loop_source(st._h, self.handle, buf, n.value + 1, ctypes.byref(n)))
        return buf.value.decode()

    def free(self):
        if self.state._h is not None and self.handle >= 0:
            self.state._ck(self.state._lib.ljmd_loop_free(self.state._h, self.handle))
            self.handle = -1


class ParticleLoop(_Loop):
    """Execute a kernel for all particles (Def. 1)."""
    _kind = 0

    def __init__(self, kernel: Kernel, dat_dict, fmad: bool = False):
        super().__init__(kernel, dat_dict, 0.0, fmad)


class PairLoop(_Loop):
    """Execute a kernel for all ordered pairs within shell_cutoff (Def. 3)."""
    _kind = 1

    def __init__(self, kernel: Kernel, dat_dict, shell_cutoff: float, fmad: bool = False):
        super().__init__(kernel, dat_dict, shell_cutoff, fmad)


__all__ = ["READ", "WRITE", "RW", "INC", "INC_ZERO", "access", "Constant", "Kernel", "ParticleDat", "ScalarArray",
           "EngineDat", "PositionDat", "velocities", "forces", "global_ids", "particle_energies", "ParticleLoop",
           "PairLoop"]
