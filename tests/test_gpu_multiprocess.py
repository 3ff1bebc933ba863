"""Ranks as separate PROCESSES -- the launch shape of bench.py under torchrun (one process
per GPU, z-slab decomposition).

One GPU: NCCL refuses two ranks on one device, so the processes exchange through the
engine's host-staged multi-process transport (`LJMDSHM`); everything else -- slab
planning, migration, halo planes, the all-reduces of the displacement check and the
energies, the host loop of every rank -- is the code path the NCCL run takes.
* two and three processes reproduce the single-rank run bit for bit (build-order lists);
* bench.py under torch.distributed.run (2 ranks, default legs) prints one valid JSON line.
Two or more GPUs: bench.py over NCCL, one rank per GPU (skipped on one GPU, and says so)."""
import json
import os
import socket
import subprocess
import sys
import uuid

import numpy as np
import pytest
import torch

import ljinputs as li

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def run_processes(nranks, dims, steps, check, tmp_path):
    key = uuid.uuid4().hex
    outs = [str(tmp_path / f"r{r}.npz") for r in range(nranks)]
    procs = [subprocess.Popen([sys.executable, os.path.join(ROOT, "tests", "mp_rank.py"), str(r), str(nranks), key,
                               outs[r], *map(str, dims), str(steps), str(check)],
                              stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
             for r in range(nranks)]
    logs = []
    try:
        for p in procs:
            logs.append(p.communicate(timeout=300)[0])
    finally:
        for p in procs:
            if p.poll() is None:
                p.kill()
    for p, log in zip(procs, logs):
        assert p.returncode == 0, log[-3000:]
    return [dict(np.load(o)) for o in outs]


@pytest.mark.parametrize("nranks,dims,check", [(2, (6, 6, 9), 0), (3, (6, 6, 24), 0), (2, (6, 6, 24), 1)])
def test_processes_bitwise(nranks, dims, check, tmp_path):
    from paper_1704_03329_b200 import ljmd
    pos, box = li.fcc(*dims)
    pos = li.perturb(pos, 0.05)
    vel = li.velocities(len(pos), 1.44)
    steps = 45   # two rebuilds with migration
    with ljmd.LJMD(pos, vel, box, list_order=0, rebuild_check=check) as ctx:
        ctx.step(steps)
        ref = dict(F=ctx.forces(), X=ctx.positions(), V=ctx.velocities(), e=ctx.energy(), rs=ctx.rebuild_steps())
    per = run_processes(nranks, dims, steps, check, tmp_path)
    assert sum(int(o["n_owned"]) for o in per) == len(pos)
    for k in ("X", "V", "F"):
        a = np.full((len(pos), 3), np.nan)
        for o in per:
            m = ~np.isnan(o[k][:, 0])
            assert np.all(np.isnan(a[m, 0])), "a particle owned by two ranks"
            a[m] = o[k][m]
        assert np.array_equal(a, ref[k]), k
    for o in per:
        assert float(o["pe"]) == pytest.approx(ref["e"][0], rel=1e-12)
        assert float(o["ke"]) == pytest.approx(ref["e"][1], rel=1e-12)
        assert o["rs"].tolist() == ref["rs"].tolist()


def run_bench(nproc, extra_env, args, timeout=900):
    env = dict(os.environ, **extra_env)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()), os.path.join(ROOT, "bench.py"),
           "--gpus", str(nproc), *args]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, env=env, cwd=ROOT)
    assert r.returncode == 0, (r.stdout + r.stderr)[-4000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-3000:]   # rank 0 alone prints
    return json.loads(lines[0])


def test_bench_torchrun_two_processes_one_gpu():
    """The driver's N > 1 launch (torch.distributed.run, default legs) with both ranks on GPU 0."""
    d = run_bench(2, {"LJMD_BENCH_DEVICE": "0"}, ["--steps", "2", "--warmup", "3"])   # C2x2, as the driver
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["steps"] == 2
    assert d["transport"].startswith("shm") and d["e2e"]["value"] > 0
    assert d["roofline"]["achieved"] > 0 and d["config"]["parallelism"] == "z-slab x2"
    assert d["config"]["workload"] == "C2x2" and d["config"]["n_particles"] == 2 * 1048576


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="one GPU visible: the NCCL multi-process run needs >= 2 "
                                                           "(its host flow is covered on one GPU above)")
def test_bench_torchrun_nccl_multi_gpu():
    n = min(torch.cuda.device_count(), 8)
    d = run_bench(n, {}, ["--steps", "2", "--warmup", "3"])
    assert d["n_gpus"] == n and d["value"] > 0 and d["transport"] == "nccl"
