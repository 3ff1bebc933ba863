"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NONE of the method's arithmetic (no pair displacement, no LJ
potential or force, no integrator, no cell/neighbour logic).  It only builds the
initial conditions the paper's benchmark describes:

* FCC crystal at number density rho = 0.8442 (Tab. 7.2T1),
  lattice constant a = (4/rho)^(1/3); global index
  gid = ((cz*ny + cy)*nx + cx)*4 + b.
* Gaussian velocities from numpy PCG64 (seed 87287), mean removed, rescaled to
  exactly T0 with dof = 3N-3 and k_B = 1 (reading R13).
* Gaussian position perturbations from PCG64 (seed 1704).

The paper gives N, rho, rc, rbar_c and the rebuild cadence but no temperature,
time step or lattice; the remaining values are the readings
listed in DESIGN.md.
"""
from __future__ import annotations

import dataclasses
from typing import Tuple

import numpy as np

RHO = 0.8442          # Tab. 7.2T1
RC = 2.5              # Tab. 7.2T1
DELTA = 0.25          # rbar_c - rc = 0.1 rc
NS = 20               # rebuild every 20 steps
DT = 0.005            # reading R12 (LJ units, not stated in the paper)
SEED_VEL = 87287
SEED_PERTURB = 1704

FCC_BASIS = np.array([[0.0, 0.0, 0.0],
                      [0.5, 0.5, 0.0],
                      [0.5, 0.0, 0.5],
                      [0.0, 0.5, 0.5]])


def fcc_lattice_constant(rho: float = RHO) -> float:
    return (4.0 / rho) ** (1.0 / 3.0)


def fcc(nx: int, ny: int, nz: int, rho: float = RHO) -> Tuple[np.ndarray, np.ndarray]:
    """Perfect FCC crystal: returns (pos[N,3] float64, box[3] float64)."""
    a = fcc_lattice_constant(rho)
    cz, cy, cx = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    cells = np.stack([cx.ravel(), cy.ravel(), cz.ravel()], axis=1).astype(np.float64)
    pos = (cells[:, None, :] + FCC_BASIS[None, :, :]).reshape(-1, 3) * a
    box = np.array([nx * a, ny * a, nz * a], dtype=np.float64)
    return np.ascontiguousarray(pos), box


def velocities(n: int, t0: float, seed: int = SEED_VEL, mass: float = 1.0) -> np.ndarray:
    """Maxwell velocities: N(0,1) per component, zero momentum, exact T0 (dof 3N-3)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    v = rng.standard_normal((n, 3))
    v -= v.mean(axis=0, keepdims=True)
    if n > 1 and t0 > 0.0:
        t_now = mass * float(np.sum(v * v)) / (3 * n - 3)
        v *= np.sqrt(t0 / t_now)
    else:
        v[:] = 0.0
    return np.ascontiguousarray(v)


def perturb(pos: np.ndarray, sigma_d: float, seed: int = SEED_PERTURB) -> np.ndarray:
    rng = np.random.Generator(np.random.PCG64(seed))
    return np.ascontiguousarray(pos + sigma_d * rng.standard_normal(pos.shape))


def uniform_random(n: int, box, seed: int, min_sep: float = 0.0) -> np.ndarray:
    """Uniform random positions in [0,L) (optionally with a minimum separation, O(N^2), tiny n only)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    box = np.asarray(box, dtype=np.float64)
    if min_sep <= 0.0:
        return np.ascontiguousarray(rng.random((n, 3)) * box)
    out = []
    while len(out) < n:
        p = rng.random(3) * box
        ok = True
        for q in out:
            d = p - q
            d -= box * np.round(d / box)
            if float(d @ d) < min_sep * min_sep:
                ok = False
                break
        if ok:
            out.append(p)
    return np.ascontiguousarray(np.array(out))


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    cells: Tuple[int, int, int]
    t0: float
    sigma_d: float = 0.0
    energy_shift: float = 0.25
    rebuild_check: int = 0
    md_steps: int = 100

    @property
    def n(self) -> int:
        return 4 * self.cells[0] * self.cells[1] * self.cells[2]

    def build(self, t0: float | None = None):
        pos, box = fcc(*self.cells)
        if self.sigma_d > 0.0:
            pos = perturb(pos, self.sigma_d)
        vel = velocities(pos.shape[0], self.t0 if t0 is None else t0)
        return pos, vel, box


# BASELINE.json configs
CONFIGS = {
    "C1": Config("C1", (10, 10, 10), 1.44, md_steps=100),
    "C2": Config("C2", (64, 64, 64), 1.44, md_steps=1000),
    "C3": Config("C3", (128, 128, 128), 1.44, md_steps=1000),
    "C4": Config("C4", (64, 64, 128), 1.44, md_steps=1000),
    "C5": Config("C5", (80, 80, 80), 1.5, sigma_d=0.05, rebuild_check=1, md_steps=1000),
}


def weak_config(n_gpus: int) -> Config:
    """Weak scaling at 1,048,576 particles per GPU: 64 x 64 x (64*n) FCC cells (z-slabs)."""
    return Config(f"C2x{n_gpus}", (64, 64, 64 * n_gpus), 1.44, md_steps=1000)


def hcp(nx: int, ny: int, nz: int, d: float = 1.0):
    """Ideal hcp (c/a = sqrt(8/3)) with nearest-neighbour distance d, orthohexagonal cell
    (d, sqrt(3) d, sqrt(8/3) d) holding 4 atoms; returns (pos, box)."""
    basis = np.array([[0.0, 0.0, 0.0], [0.5, 0.5, 0.0], [0.0, 1.0 / 3.0, 0.5], [0.5, 5.0 / 6.0, 0.5]])
    cell = np.array([d, np.sqrt(3.0) * d, np.sqrt(8.0 / 3.0) * d])
    cz, cy, cx = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    cells = np.stack([cx.ravel(), cy.ravel(), cz.ravel()], axis=1).astype(np.float64)
    pos = ((cells[:, None, :] + basis[None, :, :]) * cell).reshape(-1, 3)
    return np.ascontiguousarray(pos), cell * np.array([nx, ny, nz], dtype=np.float64)


def bcc(nx: int, ny: int, nz: int, d: float = 1.0):
    """bcc with nearest-neighbour distance d (cube edge 2 d / sqrt(3)); returns (pos, box)."""
    a = 2.0 * d / np.sqrt(3.0)
    basis = np.array([[0.0, 0.0, 0.0], [0.5, 0.5, 0.5]])
    cz, cy, cx = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    cells = np.stack([cx.ravel(), cy.ravel(), cz.ravel()], axis=1).astype(np.float64)
    pos = ((cells[:, None, :] + basis[None, :, :]) * a).reshape(-1, 3)
    return np.ascontiguousarray(pos), np.array([nx, ny, nz], dtype=np.float64) * a
