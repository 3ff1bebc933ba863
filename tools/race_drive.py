"""racecheck target: the sanitize drive's stepping part on one path (argv[1]: graphs 0/1)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ljinputs as li
from paper_1704_03329_b200 import LJMD
g = int(sys.argv[1])
pos, box = li.fcc(6, 6, 6)
pos = li.perturb(pos, 0.05)
vel = li.velocities(len(pos), 1.44)
for check in (0, 1):
    with LJMD(pos, vel, box, device=0, rebuild_check=check, graphs=g) as ctx:
        ctx.step(25)
        ctx.step(20)
print("race drive done", g)
