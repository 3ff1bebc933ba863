import sys, time, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import ljinputs as li
from paper_1704_03329_b200 import ljmd, LJMD
pos, vel, box = li.CONFIGS["C2"].build()
n = len(pos)
for mode in ("own", "torch"):
    if mode == "torch":
        s = torch.cuda.Stream(); torch.cuda.set_stream(s); h = s.cuda_stream
    else:
        h = None
    opts = ljmd.default_options(device=0, stream=h, profile=1)
    ctx = LJMD(pos, vel, box, options=opts)
    hp = torch.from_numpy(pos.copy()).pin_memory(); hv = torch.from_numpy(vel.copy()).pin_memory()
    ho = torch.empty((n, 3), dtype=torch.float64).pin_memory()
    for it in range(3):
        t = [time.perf_counter()]
        ctx.set_state_ptr(hp.data_ptr(), hv.data_ptr()); torch.cuda.synchronize(); t.append(time.perf_counter())
        ctx.step(20); torch.cuda.synchronize(); t.append(time.perf_counter())
        ctx.positions_into_ptr(ho.data_ptr()); t.append(time.perf_counter())
        ctx.energy(); t.append(time.perf_counter())
        print(mode, it, ["%.1f" % ((b - a) * 1e3) for a, b in zip(t, t[1:])], flush=True)
    ctx.close()
