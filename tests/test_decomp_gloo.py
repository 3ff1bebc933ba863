"""CPU (gloo, world_size 2 and 3) check of the z-slab decomposition protocol the engine runs
over NCCL: slab plan from libljmd's host planner, migration of
particles that left the slab, exchange of the boundary cell planes in the engine's order
(send to the upper, then the lower neighbour; receive from the lower, then the upper one --
the order that also pairs correctly when both neighbours are the same rank), and the force
on every owned particle from (owned + received planes) equal to the global oracle's.

The device implementation of the same protocol is exercised on one GPU through the loopback
transport in tests/test_gpu_multirank.py (bitwise p = 1 vs p = 2, 3).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import ljinputs as li

RN = li.RC + li.DELTA


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _plane(z, w, ncz, L):
    z = z - L * np.floor(z / L)
    return np.clip(np.floor(z / w).astype(int), 0, ncz - 1)


def _xchg(to_hi, to_lo, lo, hi):
    """Engine order: send (upper, lower), receive (from lower, from upper); tags keep the two
    directions apart for gloo exactly as the posting order does for NCCL."""
    def send(arr, peer, tag):
        n = torch.tensor([arr.shape[0]], dtype=torch.int64)
        return [dist.isend(n, peer, tag=tag), dist.isend(torch.from_numpy(np.ascontiguousarray(arr)), peer,
                                                          tag=tag + 10)]
    reqs = send(to_hi, hi, 0) + send(to_lo, lo, 1)
    n_lo, n_hi = torch.zeros(1, dtype=torch.int64), torch.zeros(1, dtype=torch.int64)
    dist.recv(n_lo, lo, tag=0)       # what the lower rank sent to its upper neighbour
    dist.recv(n_hi, hi, tag=1)
    a_lo = torch.zeros((int(n_lo), to_hi.shape[1]), dtype=torch.float64)
    a_hi = torch.zeros((int(n_hi), to_lo.shape[1]), dtype=torch.float64)
    dist.recv(a_lo, lo, tag=10)
    dist.recv(a_hi, hi, tag=11)
    for r in reqs:
        r.wait()
    return a_lo.numpy(), a_hi.numpy()


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from paper_1704_03329_b200 import plan_cells, plan_slab
        pos0, box = li.fcc(6, 6, 12)
        pos0 = li.perturb(pos0, 0.05)
        n = len(pos0)
        nc = plan_cells(box, RN)
        w = box[2] / nc[2]
        z0, z1 = plan_slab(int(nc[2]), world, rank)
        lo, hi = (rank - 1) % world, (rank + 1) % world
        # initial ownership, then every particle drifts (some across slab boundaries)
        p0 = _plane(pos0[:, 2], w, nc[2], box[2])
        mine = np.nonzero((p0 >= z0) & (p0 < z1))[0]
        rng = np.random.default_rng(9)
        moved = pos0 + rng.normal(0.0, 0.4, pos0.shape)
        rows = np.concatenate([moved, np.arange(n)[:, None]], axis=1)[mine]     # x, y, z, gid
        # migration: leavers go to the adjacent slab only
        pl = _plane(rows[:, 2], w, nc[2], box[2])
        down = pl == (z0 - 1) % nc[2]
        up = (pl == z1 % nc[2]) & ~down
        stay = ~(down | up)
        assert np.all((pl[stay] >= z0) & (pl[stay] < z1))
        got_lo, got_hi = _xchg(rows[up], rows[down], lo, hi)
        own = np.concatenate([rows[stay], got_lo, got_hi])
        # ownership after migration is exactly the slab
        pl = _plane(own[:, 2], w, nc[2], box[2])
        assert np.all((pl >= z0) & (pl < z1))
        # halo planes: top plane -> upper neighbour's lower ghost, bottom -> lower's upper
        top, bot = own[pl == z1 - 1], own[pl == z0]
        g_lo, g_hi = _xchg(top, bot, lo, hi)
        local = np.concatenate([own, g_lo, g_hi])
        f_loc = oracle.forces_rows(local[:, :3], box, np.arange(len(own)), oracle.LJ())
        f_ref = oracle.forces_rows(moved, box, own[:, 3].astype(np.int64), oracle.LJ())
        ok = bool(np.allclose(f_loc.F, f_ref.F, rtol=0, atol=1e-12 * (1 + f_ref.S.max())))
        ok_e = bool(np.allclose(f_loc.e, f_ref.e, rtol=1e-12, atol=1e-14))
        q.put((rank, sorted(own[:, 3].astype(int).tolist()), ok, ok_e))
    except Exception as e:  # noqa: BLE001
        q.put((rank, repr(e), False, False))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_slab_protocol_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    owned = []
    for rank, gids, ok, ok_e in res:
        assert isinstance(gids, list), gids
        assert ok and ok_e, f"rank {rank}: local forces differ from the global oracle"
        owned += gids
    n = 4 * 6 * 6 * 12
    assert sorted(owned) == list(range(n)), "every particle owned exactly once"
