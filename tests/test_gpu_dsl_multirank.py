"""DSL loops on several z-slab ranks (one GPU, in-process loopback transport -- the device path
NCCL drives on 1-8 GPUs): particle data migrates with its particles, the data a pair loop
reads on the j side is exchanged into the halo before the loop, ScalarArray INC
is all-reduced.  With the build-order lists (list_order = 0) every particle sees the same
neighbours in the same order on any number of ranks, so per-particle results are bitwise
equal to one rank."""
import threading
import uuid

import numpy as np
import pytest

import ljinputs as li
from dsl_kernels import CNA_I, CNA_II, LJ, LJ_CONSTANTS, SIMPLE

pytestmark = pytest.mark.gpu

MISSING = -(2 ** 40)


def system():
    pos, box = li.fcc(6, 6, 9)
    pos = li.perturb(pos, 0.05)
    return pos, li.velocities(len(pos), 1.44), box


def run(nranks, body, pos, vel, box):
    """body(ctx) -> {name: array over all particles, non-owned rows left at MISSING/NaN}."""
    from paper_1704_03329_b200 import ljmd
    if nranks == 1:
        with ljmd.LJMD(pos, vel, box, list_order=0) as ctx:
            return body(ctx)
    gid = ljmd.local_group_id(uuid.uuid4().hex)
    out, err = [None] * nranks, [None] * nranks

    def work(r):
        try:
            with ljmd.LJMD(pos, vel, box, rank=r, nranks=nranks, nccl_id=gid, list_order=0) as ctx:
                out[r] = body(ctx)
        except Exception as e:  # noqa: BLE001
            err[r] = e

    th = [threading.Thread(target=work, args=(r,)) for r in range(nranks)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    assert not any(t.is_alive() for t in th)
    for e in err:
        if e is not None:
            raise e
    merged = {}
    for k, v0 in out[0].items():
        if k.startswith("scalar"):
            for o in out[1:]:
                np.testing.assert_array_equal(o[k], v0)   # every rank holds the reduced value
            merged[k] = v0
            continue
        acc = np.full_like(v0, MISSING if v0.dtype.kind == "i" else np.nan)
        for o in out:
            own = o[k] != MISSING if v0.dtype.kind == "i" else ~np.isnan(o[k])
            own = own.reshape(len(own), -1).all(axis=1)
            acc[own] = o[k][own]
        merged[k] = acc
    return merged


def dat_rows(dat, kind):
    """dat.data with the rows this rank does not own marked (ljmd_dat_get leaves them)."""
    from paper_1704_03329_b200.ljmd import _I  # noqa: F401
    import ctypes
    buf = np.full(dat.shape, MISSING if kind == "i" else np.nan, dtype=dat.dtype)
    dat.state._ck(dat.state._lib.ljmd_dat_get(dat.state._h, dat.handle, buf.ctypes.data_as(ctypes.c_void_p)))
    return buf


@pytest.mark.parametrize("nranks", [2, 3])
def test_lj_and_simple_op_decomposition(nranks):
    from paper_1704_03329_b200 import dsl
    pos, vel, box = system()
    a0 = np.random.default_rng(2).standard_normal((len(pos), 3))

    def body(st):
        st.step(25)                                 # one rebuild with migration
        F, u = dsl.ParticleDat(st, ncomp=3), dsl.ScalarArray(st)
        dsl.PairLoop(dsl.Kernel("lj", LJ, tuple(dsl.Constant(k, v) for k, v in LJ_CONSTANTS.items())),
                     {"r": dsl.PositionDat(st)(dsl.READ), "F": F(dsl.INC_ZERO), "u": u(dsl.INC_ZERO)},
                     shell_cutoff=li.RC).execute()
        a = dsl.ParticleDat(st, ncomp=3)
        a.data = a0
        b, S = dsl.ParticleDat(st), dsl.ScalarArray(st)
        dsl.PairLoop(dsl.Kernel("s", SIMPLE, (dsl.Constant("dimension", 3),)),
                     {"r": dsl.PositionDat(st)(dsl.READ), "a": a(dsl.READ), "b": b(dsl.INC_ZERO),
                      "S": S(dsl.INC_ZERO)}, shell_cutoff=1.6).execute()
        v = dsl.ParticleDat(st, ncomp=3)            # the engine's velocities read on the j side
        dsl.PairLoop(dsl.Kernel("vj", "w.i[0] += v.j[0]; w.i[1] += v.j[1]; w.i[2] += v.j[2];"),
                     {"r": dsl.PositionDat(st)(dsl.READ), "v": dsl.velocities(st)(dsl.READ), "w": v(dsl.INC_ZERO)},
                     shell_cutoff=1.6).execute()
        return {"F": dat_rows(F, "f"), "b": dat_rows(b, "f"), "w": dat_rows(v, "f"),
                "scalar_u": u.data, "scalar_S": S.data}

    ref = run(1, body, pos, vel, box)
    got = run(nranks, body, pos, vel, box)
    for k in ("F", "b", "w"):
        assert not np.isnan(got[k]).any(), k
        assert np.array_equal(got[k], ref[k]), k
    np.testing.assert_allclose(got["scalar_u"], ref["scalar_u"], rtol=1e-12)
    np.testing.assert_allclose(got["scalar_S"], ref["scalar_S"], rtol=1e-12)


@pytest.mark.parametrize("nranks", [2, 3])
def test_cna_kernels_and_migration(nranks):
    """Integer data set from the host, carried through two rebuilds with migration, then
    the CNA kernels (j-side reads of an RW dat and of the global ids) on every rank."""
    from paper_1704_03329_b200 import dsl
    pos, vel, box = system()
    n = len(pos)
    rc = (li.fcc_lattice_constant() * (1 / np.sqrt(2) + 1)) / 2
    W = 2 * 24 * 24
    tag0 = (np.arange(n, dtype=np.int64) * 13 + 5).reshape(-1, 1)

    def body(st):
        tag = dsl.ParticleDat(st, dtype=np.int64)
        tag.data = tag0
        st.step(45)                                 # two rebuilds: rows migrate with particles
        ids = dsl.global_ids(st)
        n_nb, n_bond = dsl.ParticleDat(st, dtype=np.int64), dsl.ParticleDat(st, dtype=np.int64)
        bond = dsl.ParticleDat(st, ncomp=W, dtype=np.int64)
        rcs = (dsl.Constant("rc_sq", rc * rc),)
        dsl.PairLoop(dsl.Kernel("c1", CNA_I, rcs),
                     {"r": dsl.PositionDat(st)(dsl.READ), "id": ids(dsl.READ), "n_nb": n_nb(dsl.INC_ZERO),
                      "n_bond": n_bond(dsl.INC_ZERO), "bond": bond(dsl.WRITE)}, shell_cutoff=rc).execute()
        dsl.PairLoop(dsl.Kernel("c2", CNA_II, rcs),
                     {"r": dsl.PositionDat(st)(dsl.READ), "id": ids(dsl.READ), "n_nb": n_nb(dsl.READ),
                      "n_bond": n_bond(dsl.INC), "bond": bond(dsl.RW)}, shell_cutoff=rc).execute()
        s = dsl.ParticleDat(st, dtype=np.int64)     # sum of the neighbours' tags (j-side halo)
        cnt = dsl.ScalarArray(st, dtype=np.int64)
        dsl.PairLoop(dsl.Kernel("t", "s.i[0] += tag.j[0]; cnt[0] += 1;"),
                     {"r": dsl.PositionDat(st)(dsl.READ), "tag": tag(dsl.READ), "s": s(dsl.INC_ZERO),
                      "cnt": cnt(dsl.INC_ZERO)}, shell_cutoff=rc).execute()
        return {"tag": dat_rows(tag, "i"), "n_nb": dat_rows(n_nb, "i"), "n_bond": dat_rows(n_bond, "i"),
                "bond": dat_rows(bond, "i"), "s": dat_rows(s, "i"), "scalar_cnt": cnt.data}

    ref = run(1, body, pos, vel, box)
    got = run(nranks, body, pos, vel, box)
    assert np.array_equal(got["tag"], tag0)
    for k in ("n_nb", "n_bond", "bond", "s"):
        assert np.array_equal(got[k], ref[k]), k
    assert got["scalar_cnt"][0] == ref["scalar_cnt"][0] == int(ref["n_nb"].sum())


@pytest.mark.parametrize("transport", ["nccl", "local"])
def test_dsl_halo_through_transport(transport):
    """split_self: one rank running the several-rank DSL path (data halo through the
    transport -- NCCL self send/recv on one GPU, or the loopback -- and the ScalarArray
    all-reduce), equal to the plain single-rank loop."""
    from paper_1704_03329_b200 import dsl, ljmd
    pos, vel, box = system()
    a0 = np.random.default_rng(9).standard_normal((len(pos), 3))

    def body(st):
        st.step(25)
        a = dsl.ParticleDat(st, ncomp=3)
        a.data = a0
        b, S = dsl.ParticleDat(st), dsl.ScalarArray(st)
        dsl.PairLoop(dsl.Kernel("s", SIMPLE, (dsl.Constant("dimension", 3),)),
                     {"r": dsl.PositionDat(st)(dsl.READ), "a": a(dsl.READ), "b": b(dsl.INC_ZERO),
                      "S": S(dsl.INC_ZERO)}, shell_cutoff=1.6).execute()
        return b.data, S.data

    with ljmd.LJMD(pos, vel, box, list_order=0) as st:
        rb, rS = body(st)
    nid = ljmd.nccl_unique_id() if transport == "nccl" else ljmd.local_group_id(uuid.uuid4().hex)
    with ljmd.LJMD(pos, vel, box, split_self=1, nccl_id=nid, list_order=0) as st:
        gb, gS = body(st)
    assert np.array_equal(gb, rb)
    np.testing.assert_allclose(gS, rS, rtol=1e-13)
