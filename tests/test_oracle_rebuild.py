"""Pins of the oracle's rebuild rule (O7) and its missed-pair count (validation), CPU only.

Reading R7: the safe policy rebuilds when 2 max_i |x_i - x_i(build)| > delta
(Eq. eqn:extended_cutoff); the paper's benchmark rebuilds every Ns = 20
steps regardless.  The cases below are free flights with dyadic
numbers, so every displacement is exact and the expected steps follow in closed form.
"""
import numpy as np

import ljinputs as li

DT = 1.0 / 64.0          # dyadic: x(k) = x0 + k v dt exactly
BOX = np.array([9.0, 9.0, 9.0])   # 3 cells of width 3 >= rbar_c = 2.75


def free_particle(nsteps, check, ns=1000, delta=0.25, v=1.0):
    pos = np.array([[1.0, 4.5, 4.5]])
    vel = np.array([[v, 0.0, 0.0]])
    return pos, vel


def test_safe_threshold_closed_form(orc):
    """One particle at |v| = 1: displacement k/64 after k steps, 2 k/64 > 1/4 first at k = 9
    (k = 8 gives exactly delta: strict >, no rebuild); each rebuild restarts the count:
    rebuilds at 9, 18, 27, 36.  A factor-2 slip (|dx| > delta, or 4|dx| > delta) would give
    17, 34 or 5, 10, ...; a non-strict test 8, 16, ..."""
    pos, vel = free_particle(40, 1)
    r = orc.run(pos, vel, BOX, 40, dt=DT, ns=1000, check=1, energy_every=0)
    assert r.rebuild_steps.tolist() == [9, 18, 27, 36]
    np.testing.assert_array_equal(r.pos, [[1.0 + 40 * DT, 4.5, 4.5]])   # F = 0: exact flight


def test_safe_threshold_max_not_relative(orc):
    """Two particles flying apart at +-v: the rule takes each particle's own displacement
    (max_i), not the pair's relative one -- the same 9, 18, 27, 36."""
    pos = np.array([[1.0, 1.0, 1.0], [1.0, 5.5, 5.5]])
    vel = np.array([[1.0, 0.0, 0.0], [-1.0, 0.0, 0.0]])
    r = orc.run(pos, vel, BOX, 40, dt=DT, ns=1000, check=1, energy_every=0)
    assert r.rebuild_steps.tolist() == [9, 18, 27, 36]


def test_fixed_schedule_ignores_displacement(orc):
    pos, vel = free_particle(40, 0)
    r = orc.run(pos, vel, BOX, 40, dt=DT, ns=15, check=0, energy_every=0)
    assert r.rebuild_steps.tolist() == [15, 30]


def head_on():
    # r(0) = 3 > rbar_c: not listed at init; closing speed 2 -> r(k) = 3 - k/32
    pos = np.array([[3.0, 4.5, 4.5], [6.0, 4.5, 4.5]])
    vel = np.array([[1.0, 0.0, 0.0], [-1.0, 0.0, 0.0]])
    return pos, vel


def test_missed_pairs_closed_form(orc):
    """Two particles approaching head-on from r = 3 under the fixed schedule (no rebuild in
    40 steps): r(k) = 3 - k/32 < rc = 2.5 first at k = 17, and the list built at r = 3 never
    serves the pair, so steps 17..40 miss it (2 particles, 2 ordered pairs); the free
    flight is exact because the list is empty."""
    pos, vel = head_on()
    r = orc.run(pos, vel, BOX, 40, dt=DT, ns=1000, check=0, energy_every=0, validate=True)
    k = np.arange(41)
    want = np.where(k >= 17, 2, 0)
    np.testing.assert_array_equal(r.missed_particles, want)
    np.testing.assert_array_equal(r.missed_pairs, want)
    np.testing.assert_array_equal(r.pos[:, 0], [3.0 + 40 * DT, 6.0 - 40 * DT])


def test_missed_pairs_safe_policy_head_on(orc):
    """The same approach under the safe policy: rebuilt at k = 9 (r = 2.71875 < rbar_c, now
    listed), no step misses the pair (the skin argument)."""
    pos, vel = head_on()
    r = orc.run(pos, vel, BOX, 40, dt=DT, ns=1000, check=1, energy_every=0, validate=True)
    assert r.rebuild_steps[0] == 9
    assert not r.missed_particles.any() and not r.missed_pairs.any()


def test_missed_equals_force_error_count(orc):
    """Cross-check of the count against the force it stands for: perfect FCC at T0 = 1.44
    under the paper's fixed Ns = 20 (C1).  At step 19 (the last served by the init list) the
    particles with a missed pair are exactly those whose list force differs from the
    brute-force force by more than the 1e-10 S_i bar -- computed here from O4 + O5 with and
    without the list, not from orc_missed."""
    pos, box = li.fcc(10, 10, 10)
    vel = li.velocities(len(pos), 1.44)
    r = orc.run(pos, vel, box, 19, validate=True, omp=True)
    assert r.rebuild_steps.size == 0
    L0 = orc.neighbours(orc.wrap(pos, box), box, li.RC + li.DELTA, "cells")
    lj = orc.LJ(rc=li.RC, shift=0.25)
    fl = orc.forces(r.pos, box, lj, nlist=L0)
    fb = orc.forces(r.pos, box, lj)
    off = np.any(np.abs(fl.F - fb.F) > 1e-10 * fb.S[:, None], axis=1)
    assert int(off.sum()) == r.missed_particles[19] > 0
    assert orc.missed(r.pos, box, li.RC, L0) == (r.missed_particles[19], r.missed_pairs[19])


def test_safe_policy_never_misses(orc):
    """The theorem behind reading R7 on a melt (C1 perturbed, T0 = 1.44): 60 steps under the
    displacement-checked policy miss nothing."""
    pos, box = li.fcc(10, 10, 10)
    pos = li.perturb(pos, 0.05)
    vel = li.velocities(len(pos), 1.44)
    r = orc.run(pos, vel, box, 60, check=1, validate=True, omp=True)
    assert r.rebuild_steps.size >= 3
    assert not r.missed_particles.any()


def test_openmp_build_identical(orc):
    """The OpenMP build (bench.py's all-core leg) computes bit for bit what the plain one does."""
    pos, box = li.fcc(6, 6, 6)
    pos = li.perturb(pos, 0.05)
    vel = li.velocities(len(pos), 1.44)
    a = orc.run(pos, vel, box, 25, omp=False)
    b = orc.run(pos, vel, box, 25, omp=True)
    assert np.array_equal(a.pos, b.pos) and np.array_equal(a.vel, b.vel)
    assert np.array_equal(a.pe, b.pe) and np.array_equal(a.ke, b.ke)
    assert orc.threads() >= 1
