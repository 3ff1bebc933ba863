"""ncu target: C2 init (one list build), optionally list_order from argv[1]."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ljinputs as li
from paper_1704_03329_b200 import LJMD
lo = int(sys.argv[1]) if len(sys.argv) > 1 else 1
pos, vel, box = li.CONFIGS["C2"].build()
with LJMD(pos, vel, box, list_order=lo) as md:
    md.step(20)
