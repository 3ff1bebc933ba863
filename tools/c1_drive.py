"""ncu target: C1 init + 40 MD steps (two rebuilds)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ljinputs as li
from paper_1704_03329_b200 import LJMD
pos, vel, box = li.CONFIGS["C1"].build()
with LJMD(pos, vel, box) as md:
    md.step(40)
