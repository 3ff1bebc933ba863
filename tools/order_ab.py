"""ljmd_step(20) cycles timed with CUDA events for list_order 0 / 1 on a config (graph mode):
python tools/order_ab.py [config]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import ljinputs as li
from paper_1704_03329_b200 import LJMD, ljmd

cfg = li.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C1"]
pos, vel, box = cfg.build()
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
for order in (0, 1, 0, 1):
    o = ljmd.default_options(device=0, stream=s.cuda_stream, list_order=order, rebuild_check=cfg.rebuild_check)
    with LJMD(pos, vel, box, rc=li.RC, dt=li.DT, options=o) as ctx:
        for _ in range(5):
            ctx.step(20)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        k = 30
        for _ in range(k):
            ctx.step(20)
        e1.record(s)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / k
        print(f"{cfg.name} list_order={order}: {ms * 1e3 / 20:.2f} us per MD step, {len(pos) * 20 / (ms * 1e-3):.3e} PTS/s")
