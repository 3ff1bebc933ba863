"""ctypes binding of libljmd.so (include/ljmd.h) -- argument marshalling only.

Every step of the LJ PairLoop path runs in the sm_100a kernels of libljmd.so; there is
no Python or CPU fallback.  If the library is missing or no CUDA device is present the
calls raise instead of computing anything.

Function names mirror the C ABI (ljmd_init, ljmd_step, ...); `LJMD` is a thin owner of a
context handle with the same calls as methods.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libljmd.so")

_D = ctypes.POINTER(ctypes.c_double)
_I = ctypes.POINTER(ctypes.c_int64)

STATUS = {0: "LJMD_OK", -1: "LJMD_E_ARG", -2: "LJMD_E_BOX", -3: "LJMD_E_NONFINITE",
          -4: "LJMD_E_OVERLAP", -5: "LJMD_E_CAPACITY", -6: "LJMD_E_CUDA", -7: "LJMD_E_NCCL",
          -8: "LJMD_E_STATE"}

EXPORTS = ("ljmd_default_options", "ljmd_init", "ljmd_set_state", "ljmd_step", "ljmd_get_forces",
           "ljmd_get_positions", "ljmd_get_velocities", "ljmd_get_particle_energy", "ljmd_get_energy",
           "ljmd_get_energy_history", "ljmd_get_neighbours", "ljmd_get_rebuild_steps", "ljmd_get_stats",
           "ljmd_get_validation",
           "ljmd_last_error", "ljmd_destroy", "ljmd_version", "ljmd_plan_cells", "ljmd_plan_slab",
           "ljmd_measure_fp64_peak", "ljmd_nccl_unique_id", "ljmd_boa", "ljmd_cna", "ljmd_set_thermostat", "ljmd_set_profile",
           "ljmd_stage_state", "ljmd_get_positions_async", "ljmd_wait_transfers",
           "ljmd_dat_create", "ljmd_dat_set", "ljmd_dat_get", "ljmd_dat_free", "ljmd_loop_create",
           "ljmd_loop_execute", "ljmd_loop_source", "ljmd_loop_free")


class LjmdError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class Options(ctypes.Structure):
    _fields_ = [("delta", ctypes.c_double), ("rebuild_every", ctypes.c_int64),
                ("rebuild_check", ctypes.c_int64), ("mass", ctypes.c_double),
                ("energy_shift", ctypes.c_double), ("energy_every", ctypes.c_int64),
                ("device", ctypes.c_int64), ("nbr_capacity", ctypes.c_int64),
                ("rank", ctypes.c_int64), ("nranks", ctypes.c_int64),
                ("nccl_id", ctypes.c_void_p), ("stream", ctypes.c_void_p),
                ("profile", ctypes.c_int64), ("list_order", ctypes.c_int64),
                ("split_self", ctypes.c_int64), ("newton3", ctypes.c_int64),
                ("validate", ctypes.c_int64), ("graphs", ctypes.c_int64), ("tight_caps", ctypes.c_int64)]


class Stats(ctypes.Structure):
    _fields_ = [("steps_done", ctypes.c_int64), ("n_rebuilds", ctypes.c_int64),
                ("n_owned", ctypes.c_int64), ("n_ghost", ctypes.c_int64),
                ("nbr_capacity", ctypes.c_int64), ("max_neighbours", ctypes.c_int64),
                ("total_neighbours", ctypes.c_int64), ("n_cells", ctypes.c_int64 * 3),
                ("regrows", ctypes.c_int64), ("force_launches", ctypes.c_int64),
                ("force_ms", ctypes.c_double), ("energy_samples", ctypes.c_int64),
                ("kernel_launches", ctypes.c_int64), ("dangerous_builds", ctypes.c_int64),
                ("max_build_disp", ctypes.c_double), ("validated_steps", ctypes.c_int64),
                ("missed_pairs", ctypes.c_int64), ("missed_particle_steps", ctypes.c_int64),
                ("max_missed_particles", ctypes.c_int64), ("graph_calls", ctypes.c_int64),
                ("graph_aborts", ctypes.c_int64), ("graphs_cached", ctypes.c_int64)]

    def as_dict(self):
        d = {k: getattr(self, k) for k, _ in self._fields_}
        d["n_cells"] = list(self.n_cells)
        return d


_lib = None


def load(path: str = None):
    """Load libljmd.so (raises if it has not been built: no fallback path exists).
    LJMD_LIB overrides the path (A/B builds of the same sources)."""
    global _lib
    if _lib is not None:
        return _lib
    path = path or os.environ.get("LJMD_LIB", LIB_PATH)
    if not os.path.exists(path):
        raise RuntimeError(f"libljmd.so not built at {path}; run __graft_entry__.build()")
    lib = ctypes.CDLL(path)
    vp = ctypes.c_void_p
    sig = {
        "ljmd_default_options": ([ctypes.POINTER(Options)], ctypes.c_int),
        "ljmd_init": ([ctypes.POINTER(vp), ctypes.c_int64, _D, _D, _D, ctypes.c_double, ctypes.c_double,
                       ctypes.c_double, ctypes.c_double, ctypes.POINTER(Options)], ctypes.c_int),
        "ljmd_set_state": ([vp, _D, _D], ctypes.c_int),
        "ljmd_stage_state": ([vp, _D, _D], ctypes.c_int),
        "ljmd_get_positions_async": ([vp, _D], ctypes.c_int),
        "ljmd_wait_transfers": ([vp], ctypes.c_int),
        "ljmd_step": ([vp, ctypes.c_int64], ctypes.c_int),
        "ljmd_get_forces": ([vp, _D], ctypes.c_int),
        "ljmd_get_positions": ([vp, _D, ctypes.c_int64], ctypes.c_int),
        "ljmd_get_velocities": ([vp, _D], ctypes.c_int),
        "ljmd_get_particle_energy": ([vp, _D], ctypes.c_int),
        "ljmd_get_energy": ([vp, _D, _D], ctypes.c_int),
        "ljmd_get_energy_history": ([vp, _D, _D, ctypes.c_int64, _I], ctypes.c_int),
        "ljmd_get_neighbours": ([vp, _I, _I, ctypes.c_int64], ctypes.c_int),
        "ljmd_get_rebuild_steps": ([vp, _I, ctypes.c_int64, _I], ctypes.c_int),
        "ljmd_get_stats": ([vp, ctypes.POINTER(Stats)], ctypes.c_int),
        "ljmd_get_validation": ([vp, _I, ctypes.c_int64, _I], ctypes.c_int),
        "ljmd_last_error": ([vp], ctypes.c_char_p),
        "ljmd_destroy": ([vp], None),
        "ljmd_version": ([], ctypes.c_char_p),
        "ljmd_plan_cells": ([_D, ctypes.c_double, _I], ctypes.c_int),
        "ljmd_plan_slab": ([ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, _I, _I], ctypes.c_int),
        "ljmd_measure_fp64_peak": ([ctypes.c_int64, _D], ctypes.c_int),
        "ljmd_nccl_unique_id": ([ctypes.c_void_p], ctypes.c_int),
        "ljmd_boa": ([vp, ctypes.c_int64, ctypes.c_double, _D, _I], ctypes.c_int),
        "ljmd_set_thermostat": ([vp, ctypes.c_double, ctypes.c_double, ctypes.c_uint64], ctypes.c_int),
        "ljmd_set_profile": ([vp, ctypes.c_int64], ctypes.c_int),
        "ljmd_cna": ([vp, ctypes.c_double, ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int32), _I],
                     ctypes.c_int),
        "ljmd_dat_create": ([vp, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, _I], ctypes.c_int),
        "ljmd_dat_set": ([vp, ctypes.c_int64, ctypes.c_void_p], ctypes.c_int),
        "ljmd_dat_get": ([vp, ctypes.c_int64, ctypes.c_void_p], ctypes.c_int),
        "ljmd_dat_free": ([vp, ctypes.c_int64], ctypes.c_int),
        "ljmd_loop_create": ([vp, ctypes.c_int64, ctypes.c_char_p, ctypes.c_char_p, ctypes.c_char_p, ctypes.c_double,
                              ctypes.c_int64, ctypes.POINTER(ctypes.c_char_p), _I, _I, ctypes.c_int64, _I],
                             ctypes.c_int),
        "ljmd_loop_execute": ([vp, ctypes.c_int64], ctypes.c_int),
        "ljmd_loop_source": ([vp, ctypes.c_int64, ctypes.c_char_p, ctypes.c_int64, _I], ctypes.c_int),
        "ljmd_loop_free": ([vp, ctypes.c_int64], ctypes.c_int),
    }
    for name, (args, res) in sig.items():
        if not hasattr(lib, name) and "LJMD_LIB" in os.environ:
            continue   # an older A/B build of the library (measurement runs only)
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = res
    _lib = lib
    return lib


def _dp(a):
    return a.ctypes.data_as(_D)


def _rows(a, n=None):
    a = np.ascontiguousarray(a, dtype=np.float64).reshape(-1, 3)
    if n is not None and a.shape[0] != n:
        raise ValueError(f"expected {n} rows, got {a.shape[0]}")
    return a


def default_options(**kw) -> Options:
    o = Options()
    load().ljmd_default_options(ctypes.byref(o))
    for k, v in kw.items():
        if not hasattr(o, k):
            raise KeyError(k)
        setattr(o, k, v)
    return o


def plan_cells(box, rbar_c):
    nc = np.zeros(3, dtype=np.int64)
    b = np.ascontiguousarray(box, dtype=np.float64)
    s = load().ljmd_plan_cells(_dp(b), float(rbar_c), nc.ctypes.data_as(_I))
    if s != 0:
        raise LjmdError(s, "box too small for 3 cells of width >= rbar_c")
    return nc


def plan_slab(ncz, nranks, rank):
    z0, z1 = ctypes.c_int64(), ctypes.c_int64()
    s = load().ljmd_plan_slab(ncz, nranks, rank, ctypes.byref(z0), ctypes.byref(z1))
    if s != 0:
        raise LjmdError(s, "bad slab split")
    return z0.value, z1.value


def measure_fp64_peak(device: int = -1) -> float:
    """FP64 FMA throughput of the device in TFLOP/s (DFMA-chain probe kernel)."""
    t = ctypes.c_double()
    s = load().ljmd_measure_fp64_peak(device, ctypes.byref(t))
    if s != 0:
        raise LjmdError(s, load().ljmd_last_error(None).decode())
    return t.value


def nccl_unique_id() -> bytes:
    """128-byte ncclUniqueId (rank 0 creates it; broadcast it to the other ranks)."""
    buf = ctypes.create_string_buffer(128)
    s = load().ljmd_nccl_unique_id(buf)
    if s != 0:
        raise LjmdError(s, load().ljmd_last_error(None).decode())
    return buf.raw


def local_group_id(key: str) -> bytes:
    """Id of an in-process loopback group (several contexts of this process, one GPU)."""
    b = ("LJMDLOCAL:" + key).encode()
    if len(b) > 127:
        raise ValueError("key too long")
    return b + b"\0" * (128 - len(b))


def shm_group_id(key: str) -> bytes:
    """Id of a host-staged multi-PROCESS group on one GPU (NCCL refuses two ranks per device):
    every rank passes the same key."""
    b = ("LJMDSHM:" + key).encode()
    if len(b) > 127:
        raise ValueError("key too long")
    return b + b"\0" * (128 - len(b))


def version() -> str:
    return load().ljmd_version().decode()


class LJMD:
    """One engine context (one rank / GPU).  Mirrors ljmd_init / ljmd_step / getters."""

    def __init__(self, pos, vel, box, rc=2.5, epsilon=1.0, sigma=1.0, dt=0.005, options=None, **kw):
        lib = load()
        pos = _rows(pos)
        self.n = pos.shape[0]
        vel = _rows(vel, self.n)
        box = np.ascontiguousarray(box, dtype=np.float64).reshape(3)
        nccl_id = kw.pop("nccl_id", None)
        opt = options if options is not None else default_options(**kw)
        if nccl_id is not None:
            self._id_buf = ctypes.create_string_buffer(bytes(nccl_id), 128)
            opt.nccl_id = ctypes.cast(self._id_buf, ctypes.c_void_p)
        h = ctypes.c_void_p()
        s = lib.ljmd_init(ctypes.byref(h), self.n, _dp(pos), _dp(vel), _dp(box), float(rc), float(epsilon),
                          float(sigma), float(dt), ctypes.byref(opt))
        if s != 0:
            raise LjmdError(s, lib.ljmd_last_error(None).decode())
        self._h = h
        self._lib = lib
        self.box = box
        self.options = opt

    # -- lifecycle
    def close(self):
        if getattr(self, "_h", None):
            self._lib.ljmd_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def _ck(self, s):
        if s != 0:
            raise LjmdError(s, self._lib.ljmd_last_error(self._h).decode())

    # -- calls
    def set_state(self, pos, vel):
        p, v = _rows(pos, self.n), _rows(vel, self.n)
        self._ck(self._lib.ljmd_set_state(self._h, _dp(p), _dp(v)))

    def set_state_ptr(self, pos_ptr: int, vel_ptr: int):
        """Same as set_state, from raw host pointers (e.g. pinned torch tensors)."""
        self._ck(self._lib.ljmd_set_state(self._h, ctypes.cast(pos_ptr, _D), ctypes.cast(vel_ptr, _D)))

    def stage_state_ptr(self, pos_ptr: int, vel_ptr: int):
        """Queue an overlapped host->device copy of the next state (page-locked host arrays,
        [n][3] fp64); consumed by set_staged_state.  The arrays must stay unchanged until then."""
        self._ck(self._lib.ljmd_stage_state(self._h, ctypes.cast(pos_ptr, _D), ctypes.cast(vel_ptr, _D)))

    def set_staged_state(self):
        """ljmd_set_state(NULL, NULL): load the oldest state queued by stage_state_ptr."""
        self._ck(self._lib.ljmd_set_state(self._h, None, None))

    def positions_async_ptr(self, ptr: int):
        """Queue an overlapped device->host copy of the positions (caller order) into a
        page-locked [n][3] fp64 buffer; complete after wait_transfers()."""
        self._ck(self._lib.ljmd_get_positions_async(self._h, ctypes.cast(ptr, _D)))

    def wait_transfers(self):
        self._ck(self._lib.ljmd_wait_transfers(self._h))

    def step(self, nsteps: int):
        self._ck(self._lib.ljmd_step(self._h, int(nsteps)))

    def forces(self):
        out = np.zeros((self.n, 3))
        self._ck(self._lib.ljmd_get_forces(self._h, _dp(out)))
        return out

    def positions(self, wrapped: bool = False):
        out = np.zeros((self.n, 3))
        self._ck(self._lib.ljmd_get_positions(self._h, _dp(out), 1 if wrapped else 0))
        return out

    def positions_into_ptr(self, ptr: int, wrapped: bool = False):
        self._ck(self._lib.ljmd_get_positions(self._h, ctypes.cast(ptr, _D), 1 if wrapped else 0))

    def velocities(self):
        out = np.zeros((self.n, 3))
        self._ck(self._lib.ljmd_get_velocities(self._h, _dp(out)))
        return out

    def particle_energy(self):
        out = np.zeros(self.n)
        self._ck(self._lib.ljmd_get_particle_energy(self._h, _dp(out)))
        return out

    def energy(self):
        pe, ke = ctypes.c_double(), ctypes.c_double()
        self._ck(self._lib.ljmd_get_energy(self._h, ctypes.byref(pe), ctypes.byref(ke)))
        return pe.value, ke.value

    def energy_history(self):
        cnt = ctypes.c_int64()
        self._ck(self._lib.ljmd_get_energy_history(self._h, None, None, 0, ctypes.byref(cnt)))
        pe, ke = np.zeros(cnt.value), np.zeros(cnt.value)
        self._ck(self._lib.ljmd_get_energy_history(self._h, _dp(pe), _dp(ke), cnt.value, ctypes.byref(cnt)))
        return pe, ke

    def neighbours(self):
        off = np.zeros(self.n + 1, dtype=np.int64)
        self._ck(self._lib.ljmd_get_neighbours(self._h, off.ctypes.data_as(_I), None, 0))
        g = np.zeros(max(int(off[-1]), 1), dtype=np.int64)
        self._ck(self._lib.ljmd_get_neighbours(self._h, off.ctypes.data_as(_I), g.ctypes.data_as(_I),
                                               g.shape[0]))
        return off, g[:off[-1]]

    def boa(self, ell: int, rcut: float):
        """Bond-order parameter Q_ell per particle and |N(i)| (Sec. 4.1 of the paper)."""
        Q = np.zeros(self.n)
        nnb = np.zeros(self.n, dtype=np.int64)
        self._ck(self._lib.ljmd_boa(self._h, int(ell), float(rcut), _dp(Q), nnb.ctypes.data_as(_I)))
        return Q, nnb

    def set_thermostat(self, nu: float, temperature: float, seed: int = 0):
        """Andersen thermostat: collision frequency nu (probability nu*dt per step),
        target temperature T, Philox seed; nu = 0 restores NVE."""
        self._ck(self._lib.ljmd_set_thermostat(self._h, float(nu), float(temperature), int(seed)))

    def set_profile(self, on: bool):
        """Per-launch CUDA-event timing of the force kernel on/off (ljmd_get_stats force_ms)."""
        self._ck(self._lib.ljmd_set_profile(self._h, 1 if on else 0))

    def cna(self, rcut: float, triplets: bool = False):
        """Common-neighbour analysis (Sec. 4.2): class per particle (0 other, 1 fcc, 2 hcp,
        3 bcc), bonds per particle, and optionally the (n_nb, n_b, n_lcb) triplets
        [n, 24, 3] of each bond in ascending neighbour gid."""
        P32 = ctypes.POINTER(ctypes.c_int32)
        cls = np.zeros(self.n, dtype=np.int32)
        nnb = np.zeros(self.n, dtype=np.int64)
        tr = np.zeros((self.n, 24), dtype=np.int32) if triplets else None
        self._ck(self._lib.ljmd_cna(self._h, float(rcut), cls.ctypes.data_as(P32),
                                    tr.ctypes.data_as(P32) if tr is not None else None,
                                    nnb.ctypes.data_as(_I)))
        if tr is None:
            return cls, nnb
        t3 = np.stack([tr & 0xff, (tr >> 8) & 0xff, (tr >> 16) & 0xff], axis=-1)
        return cls, nnb, t3

    def rebuild_steps(self):
        cnt = ctypes.c_int64()
        self._ck(self._lib.ljmd_get_rebuild_steps(self._h, None, 0, ctypes.byref(cnt)))
        out = np.zeros(cnt.value, dtype=np.int64)
        self._ck(self._lib.ljmd_get_rebuild_steps(self._h, out.ctypes.data_as(_I), cnt.value,
                                                  ctypes.byref(cnt)))
        return out

    def validation(self):
        """Validation mode: [k, 3] int64 rows (step, particles with a missed pair, missed
        ordered pairs) for every validated step since init / set_state."""
        cnt = ctypes.c_int64()
        self._ck(self._lib.ljmd_get_validation(self._h, None, 0, ctypes.byref(cnt)))
        out = np.zeros((cnt.value, 3), dtype=np.int64)
        self._ck(self._lib.ljmd_get_validation(self._h, out.ctypes.data_as(_I), cnt.value, ctypes.byref(cnt)))
        return out

    def stats(self):
        s = Stats()
        self._ck(self._lib.ljmd_get_stats(self._h, ctypes.byref(s)))
        return s.as_dict()


# C-ABI-named conveniences
def ljmd_init(pos, vel, box, rc, epsilon, sigma, dt, options=None, **kw) -> LJMD:
    return LJMD(pos, vel, box, rc, epsilon, sigma, dt, options, **kw)


def ljmd_step(ctx: LJMD, nsteps: int):
    ctx.step(nsteps)


def ljmd_get_forces(ctx: LJMD):
    return ctx.forces()


def ljmd_get_energy(ctx: LJMD):
    return ctx.energy()


def ljmd_destroy(ctx: LJMD):
    ctx.close()
