"""compute-sanitizer target: small systems through init, steps with rebuilds on the graph and
the eager paths (both rebuild policies), a capacity abort resumed eagerly, validation mode,
the analyses, and a dilute box (C1-sized)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import ljinputs as li
from paper_1704_03329_b200 import LJMD

pos, box = li.fcc(6, 6, 6)
pos = li.perturb(pos, 0.05)
vel = li.velocities(len(pos), 1.44)
for check in (0, 1):
    for graphs in (1, 0):
        with LJMD(pos, vel, box, rc=li.RC, dt=li.DT, device=0, rebuild_check=check, graphs=graphs) as ctx:
            ctx.step(25)
            ctx.step(20)
            ctx.forces(); ctx.energy(); ctx.positions()
            ctx.boa(6, 1.5)
            ctx.cna(1.5)
with LJMD(li.fcc(6, 6, 6)[0], li.velocities(len(pos), 2.0), box, device=0, tight_caps=1) as ctx:
    ctx.step(40)
with LJMD(pos, vel, box, device=0, validate=1) as ctx:
    ctx.step(21)
box2 = np.array([22.0, 24.5, 27.0])
p2 = li.uniform_random(200, box2, seed=13, min_sep=0.9)
with LJMD(p2, li.velocities(len(p2), 1.0), box2, rc=li.RC, dt=li.DT, device=0) as ctx:
    ctx.step(25)
    ctx.forces()
print("sanitize drive done")
