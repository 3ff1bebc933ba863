"""ncu target: C2 init + 45 MD steps (two rebuilds) with the library in LJMD_LIB."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ljinputs as li
from paper_1704_03329_b200 import LJMD
pos, box = li.fcc(64, 64, 64)
vel = li.velocities(len(pos), 1.44)
with LJMD(pos, vel, box, rc=li.RC, dt=li.DT, device=0) as ctx:
    ctx.step(45)
