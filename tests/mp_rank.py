"""One rank of tests/test_gpu_multiprocess.py (a separate process, as under torchrun):
python tests/mp_rank.py RANK NRANKS KEY OUT.npz NX NY NZ STEPS CHECK
Runs the z-slab engine on GPU 0 through the host-staged multi-process transport and saves
this rank's owned F, X, V (NaN rows elsewhere), the energies and the rebuild steps."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import ljinputs as li
from paper_1704_03329_b200 import ljmd

rank, nranks, key, out = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3], sys.argv[4]
nx, ny, nz, steps, check = (int(v) for v in sys.argv[5:10])
pos, box = li.fcc(nx, ny, nz)
pos = li.perturb(pos, 0.05)
vel = li.velocities(len(pos), 1.44)
with ljmd.LJMD(pos, vel, box, rank=rank, nranks=nranks, nccl_id=ljmd.shm_group_id(key), list_order=0,
               rebuild_check=check, device=0) as ctx:
    ctx.step(steps)
    res = {}
    for k, fn in (("F", ctx._lib.ljmd_get_forces), ("V", ctx._lib.ljmd_get_velocities)):
        a = np.full((len(pos), 3), np.nan)
        ctx._ck(fn(ctx._h, ljmd._dp(a)))
        res[k] = a
    X = np.full((len(pos), 3), np.nan)
    ctx._ck(ctx._lib.ljmd_get_positions(ctx._h, ljmd._dp(X), 0))
    pe, ke = ctx.energy()
    np.savez(out, X=X, **res, pe=pe, ke=ke, rs=ctx.rebuild_steps(), n_owned=ctx.stats()["n_owned"],
             transport=ctx.stats().get("transport", ""))
print("rank", rank, "done")
