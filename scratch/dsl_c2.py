import sys, time, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import ljinputs as li
from paper_1704_03329_b200 import LJMD, dsl
sys.path.insert(0, "tests")
from dsl_kernels import LJ, LJ_CONSTANTS
pos, vel, box = li.CONFIGS["C2"].build()
with LJMD(pos, vel, box) as st:
    st.step(20)
    F = dsl.ParticleDat(st, ncomp=3); u = dsl.ScalarArray(st)
    loop = dsl.PairLoop(dsl.Kernel("lj", LJ, tuple(dsl.Constant(k, v) for k, v in LJ_CONSTANTS.items())),
                        {"r": dsl.PositionDat(st)(dsl.READ), "F": F(dsl.INC_ZERO), "u": u(dsl.INC_ZERO)}, shell_cutoff=li.RC)
    loop.execute(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(10): loop.execute()
    torch.cuda.synchronize()
    print("wall ms per execute", (time.perf_counter() - t0) / 10 * 1e3)
    Fg = F.data; Fe = st.forces()
    print("max |dF|", np.abs(Fg - Fe).max(), "max |F|", np.abs(Fe).max(), "u", u.data)
    pe, ke = st.energy()
    print("pe", pe, "u/2", u.data[0] / 2)
